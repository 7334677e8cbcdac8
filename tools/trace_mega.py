"""Phase timeline of one persistent decode step (diagnostics): per layer, the
mean/max over CTAs of each phase's duration and of the waits for its inputs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_14085_b200 import edgekv as ek
L, H, d, S, DEEP = 22, 32, 64, 2048, 11
ctx = ek.Context(0)
G = torch.cuda.get_device_properties(0).multi_processor_count
m = ek.EdgeModel(ctx, L, H, d, S + 256); m.synthesize(1)
kvc = ek.AssembledContext(m, S, [16] * (L - DEEP) + [8] * DEEP, group=d); kvc.synthesize(2)
sess = ek.Session(m, kvc, 128)
sess.forward(torch.zeros((16, H * d), device="cuda"))
sess.decode(3)
t = sess.trace_step(G).astype(np.int64)
G = t.size // (16 * (L + 1))  # the kernel's grid (a multiple of the head count)
t = t.reshape(L + 1, G, 16)
st = t[:L, :, :8]
start = t[L, :, 0]
t0 = start.min()
print(f"CTA start spread {(start.max() - start.min()) / 1e3:.2f} us; step {(st[-1, :, 7].max() - t0) / 1e3:.1f} us")
pr = t[L]
print(f"producer: stages/CTA {pr[:, 3].mean():.0f}, busy {(pr[:, 2] - pr[:, 1]).mean() / 1e3:.1f} us, "
      f"waiting for free slots {pr[:, 4].mean() / pr[:, 5].mean() * 100:.1f}% of its cycles")
names = ["x wait", "A qkv", "qkv wait", "B attn", "merge", "C outproj", "R reduce"]
tot = np.zeros(7)
rw = np.zeros(3)
for l in range(L):
    seg = np.diff(st[l], axis=1) / 1e3  # [G][7]
    tot += seg.mean(0)
    rw += t[l, :, 8:11].mean(0) / 8 / 1.9e3  # per-warp us at ~1.9 GHz
    if l < 3 or l >= L - 2:
        print(f"L{l:2d} " + " | ".join(f"{n} {seg[:, i].mean():5.2f}/{seg[:, i].max():5.2f}" for i, n in enumerate(names))
              + f" | layer {(st[l, :, 7].max() - st[l, :, 0].min()) / 1e3:6.2f}"
              + " | ring wait/warp A,B,C " + " ".join(f"{v / 8 / 1.9e3:.2f}" for v in t[l, :, 8:11].mean(0)))
print("sum over layers of per-CTA mean (us):", {n: round(v, 1) for n, v in zip(names, tot)})
print("sum over layers of per-warp ring wait (us) A,B,C:", np.round(rw, 1))
if os.environ.get("DBG"):
    for l in [1, 5, 15]:
        for cta in [0, 40, 100]:
            row = t[l, cta]
            base = row[1]
            print("dbg L", l, "cta", cta, [round((row[k] - base) / 1e3, 2) if row[k] else None for k in [2, 11, 12, 13, 14, 15]])
