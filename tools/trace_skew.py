"""Per-CTA skew of each phase: which CTAs are slow, and how often."""
import numpy as np, os, sys
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), 'trace_mega.py')).read().split("t = sess.trace_step(G)")[0])
res = []
for rep in range(3):
    t = sess.trace_step(G).astype(np.int64).reshape(L + 1, G, 16)
    res.append(t)
names = ["x wait", "A", "qkv wait", "B", "merge", "C", "R"]
for t in res[-1:]:
    seg = np.stack([np.diff(t[l, :, :8], axis=1) / 1e3 for l in range(L)])  # [L][G][7]
    base, extra = G // H, G % H
    heads_n = np.array([base + 1 if (c < extra * (base + 1)) else base for c in range(G)])
    for i, n in enumerate(names):
        v = seg[:, :, i]
        m4 = v[:, heads_n == base].mean(); m5 = v[:, heads_n == base + 1].mean()
        p90 = np.percentile(v, 90); mx = v.max()
        slow = np.argsort(v.mean(0))[-5:][::-1]
        print(f"{n:9s} mean {v.mean():5.2f}  p90 {p90:5.2f}  max {mx:6.2f}  |  {base}-CTA heads {m4:5.2f}  {base+1}-CTA heads {m5:5.2f} | slowest CTAs {slow.tolist()}")
    lay = (t[:L, :, 7].max(1) - t[:L, :, 0].min(1)) / 1e3
    print("layer times:", np.round(lay, 1))
