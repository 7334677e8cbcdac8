import numpy as np, os, sys
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), 'trace_mega.py')).read().split("t = sess.trace_step(G)")[0])
t = sess.trace_step(G).astype(np.int64).reshape(L + 1, G, 16)
for l in [1, 5, 13, 20]:
    r = t[l].astype(np.float64)
    first = (r[:, 13] - r[:, 12]) / 1965.0
    second = (r[:, 14] - r[:, 13]) / 1965.0
    print(f"L{l}: factor code 1st run {first.mean()*1000:.0f} ns (max {first.max()*1000:.0f}), 2nd run {second.mean()*1000:.0f} ns (max {second.max()*1000:.0f})")
