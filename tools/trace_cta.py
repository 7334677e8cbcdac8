"""Per-CTA view of one traced decode step (diagnostics): for every CTA the mean over layers
of each phase's duration and its lateness at the layer's end, to see whether the same CTAs /
heads are slow every layer (placement) or the skew moves around (noise)."""
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
reps = []
for rep in range(4):
    t = sess.trace_step(G).astype(np.int64)
    G2 = t.size // (16 * (L + 1))
    reps.append(t.reshape(L + 1, G2, 16))
names = ["xwait", "A", "qkvwait", "B", "merge", "C", "R"]
for ri, t in enumerate(reps):
    st = t[:L, :, :8].astype(np.float64)
    seg = np.diff(st, axis=2) / 1e3  # [L][G][7]
    cend = st[:, :, 6]                # C done per layer/CTA
    late = (cend - cend.min(axis=1, keepdims=True)) / 1e3
    per = seg.mean(axis=0)            # [G][7]
    lat = late.mean(axis=0)
    order = np.argsort(-lat)
    print(f"rep {ri}: slowest C-end CTAs (mean lateness us): " +
          ", ".join(f"{c}:{lat[c]:.2f}" for c in order[:8]) + f" | median {np.median(lat):.2f}")
    print("   B mean per CTA: min %.2f med %.2f max %.2f (cta %d); A: min %.2f max %.2f (cta %d)" % (
        per[:, 3].min(), np.median(per[:, 3]), per[:, 3].max(), per[:, 3].argmax(),
        per[:, 1].min(), per[:, 1].max(), per[:, 1].argmax()))
# correlation of lateness across reps
lats = []
for t in reps:
    st = t[:L, :, :8].astype(np.float64); ce = st[:, :, 6]
    lats.append(((ce - ce.min(axis=1, keepdims=True)) / 1e3).mean(axis=0))
lats = np.array(lats)
print("lateness correlation across reps:", np.round(np.corrcoef(lats), 2).tolist())
