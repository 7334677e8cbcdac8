import numpy as np, os, sys
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), 'trace_mega.py')).read().split("t = sess.trace_step(G)")[0])
t = sess.trace_step(G).astype(np.int64).reshape(L + 1, G, 16)
k = t[L]
print("stages observed per CTA", k[:, 6].mean(), "mean issue->complete us", (k[:, 7] / np.maximum(k[:, 6], 1)).mean() / 1965)
h = k[:, 8:14].sum(0)
print("histogram <1,1-2,2-4,4-8,8-16,>16 us:", h, np.round(h / h.sum(), 3))
