"""Per-CTA skew of the attention phase vs its plan (pieces, user rows)."""
import numpy as np, os, sys
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), 'trace_mega.py')).read().split("t = sess.trace_step(G)")[0])
t = sess.trace_step(G).astype(np.int64).reshape(L + 1, G, 16)
ulen = 16 + 3
UNIT = 16
cu = S // UNIT; uu = (ulen + 1 + UNIT - 1) // UNIT; per = cu + uu; TU = H * per
npieces = []; users = []
for c in range(G):
    a0, b0 = c * TU // G, (c + 1) * TU // G
    hs = set(u // per for u in range(a0, b0))
    npieces.append(len(hs))
    users.append(sum(1 for u in range(a0, b0) if u % per >= cu))
npieces = np.array(npieces); users = np.array(users)
Bt = np.stack([(t[l, :, 4] - t[l, :, 3]) / 1e3 for l in range(L)])  # [L][G]
At = np.stack([(t[l, :, 2] - t[l, :, 1]) / 1e3 for l in range(L)])
print("B time by (pieces, user units): mean over layers")
for np_ in (1, 2):
    for uu_ in sorted(set(users)):
        m = (npieces == np_) & (users == uu_)
        if m.any():
            print(f"  pieces={np_} user_units={uu_}: n={m.sum():3d}  B mean {Bt[:, m].mean():.2f}  max {Bt[:, m].max():.2f}   A mean {At[:, m].mean():.2f}")
print("B per-CTA mean (first 40 CTAs):", np.round(Bt.mean(0)[:40], 1))
print("A per-CTA mean (first 40 CTAs):", np.round(At.mean(0)[:40], 1))
