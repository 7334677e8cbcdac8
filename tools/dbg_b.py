import numpy as np, os, sys
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), 'trace_mega.py')).read().split("t = sess.trace_step(G)")[0])
t = sess.trace_step(G).astype(np.int64).reshape(L + 1, G, 16)
for l in [1, 5, 9, 13, 17, 20]:
    r = t[l].astype(np.float64)
    d = lambda k: (r[:, k] - r[:, 11]) / 1965.0
    B = (r[:, 4] - r[:, 3]) / 1e3
    print(f"L{l}: warp0 ctx {d(12).mean():.2f}  warp0 user+park {d(13).mean():.2f}  all warps parked {d(14).mean():.2f}/{d(14).max():.2f}  fold factors {d(15).mean():.2f}  B total {B.mean():.2f}/{B.max():.2f}")
