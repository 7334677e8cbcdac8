"""Per-barrier timeline of one persistent decode step (diagnostics)."""
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
t = sess.trace_step(G).astype(np.int64).reshape(-1)
start = t[6 * L * G:6 * L * G + G]
bars = t[:6 * L * G].reshape(3 * L, 2, G)
t0 = start.min()
print("start spread us", (start.max() - start.min()) / 1e3)
prev_rel = start
names = ["P1 qkv", "P2 attn", "P3 out"]
tot = {n: 0.0 for n in names}
for b in range(3 * L):
    arr, rel = bars[b, 0], bars[b, 1]
    work = (arr - prev_rel) / 1e3          # per-CTA phase work time
    sync = (rel - arr) / 1e3
    if b < 9 or b >= 3 * L - 3:
        print(f"L{b//3:2d} {names[b%3]:7s} work mean {work.mean():7.2f} max {work.max():7.2f} (cta {work.argmax():3d}) | "
              f"barrier wait mean {sync.mean():6.2f} | last arrival->release {(rel.min()-arr.max())/1e3:6.2f}")
    tot[names[b % 3]] += (rel.max() - prev_rel.min()) / 1e3
    prev_rel = rel
print("phase totals us", {k: round(v, 1) for k, v in tot.items()}, "step us", (bars[-1, 1].max() - t0) / 1e3)

sub = t[(6 * L + 1) * G:].reshape(G, 32).astype(np.int64)
names = {0: "P1 start", 1: "x staged", 3: "qkv done", 10: "P2 start", 11: "q staged", 12: "rows done",
         13: "partials+atomics", 14: "merge", 20: "P3 start", 21: "concat staged", 22: "out proj done"}
for cta in [0, 18, 70, 120]:
    row = sub[cta]
    out = []
    prev = None
    for k in sorted(names):
        if row[k] > 0:
            if prev is not None:
                out.append(f"{names[k]} +{(row[k] - prev) / 1e3:.2f}")
            prev = row[k]
    print("cta", cta, "| ".join(out), "| ring-wait cycles (sum over warps) P1/P2/P3:", row[28:31])
