import numpy as np, os, sys
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), 'trace_mega.py')).read().split("t = sess.trace_step(G)")[0])
t = sess.trace_step(G).astype(np.int64).reshape(L + 1, G, 16)
for l in [1, 5, 15, 20]:
    r = t[l].astype(np.float64)
    base = r[:, 10]
    d = lambda k: (r[:, k] - base) / 1965.0
    print(f"L{l}: xr {d(11).mean():.2f}  acq1 {d(12).mean():.2f}  st1 {d(13).mean():.2f}  acq2 {d(14).mean():.2f}   issue(stage1) {d(15).mean():.2f} (min {d(15).min():.2f} max {d(15).max():.2f})")
