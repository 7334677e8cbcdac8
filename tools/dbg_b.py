import numpy as np, os, sys
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), 'trace_mega.py')).read().split("t = sess.trace_step(G)")[0])
t = sess.trace_step(G).astype(np.int64).reshape(L + 1, G, 16)
for l in [1, 5, 15, 20]:
    r = t[l]
    base = r[:, 3]
    d = lambda k: np.where(r[:, k] > 0, (r[:, k] - base) / 1e3, np.nan)
    print(f"L{l}: " + "  ".join(f"[{k}] {np.nanmean(d(k)):.2f}/{np.nanmax(d(k)):.2f}" for k in range(11, 16)) + f"  B end {np.nanmean(d(4)):.2f}")
