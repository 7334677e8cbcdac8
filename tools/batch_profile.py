"""Per-kernel CUDA-event times of one batched decode row (ekv_batch_profile_row) at the
C2 shapes, averaged over a few rows, for B sessions (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_14085_b200 import edgekv as ek
L, H, d, S, U, DEEP = 22, 32, 64, 2048, 16, 11
ctx = ek.Context(0)
h = H * d
for B in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "128,512").split(",")]:
    model = ek.EdgeModel(ctx, L, H, d, S + 64); model.synthesize(1234)
    kvc = ek.AssembledContext(model, S, [16] * (L - DEEP) + [8] * DEEP, group=d); kvc.synthesize(99)
    b = ek.SessionBatch(model, kvc, B, U + 20)
    b.forward(torch.empty((B, U, h), device="cuda").uniform_(-1, 1)); b.decode(2)
    p = np.mean([b.profile_row() for _ in range(5)], axis=0)
    names = ["qkv", "ctx attn", "user+merge", "out proj", "splitK sum"]
    per = {n: [] for n in names}
    for l in range(L):
        for i, n in enumerate(names):
            per[n].append(p[1 + 5 * l + i])
    tot = p.sum()
    print(f"B={B}: row {tot * 1e3:.0f} us; " + ", ".join(
        f"{n} {np.mean(v[:11]) * 1e3:.1f}/{np.mean(v[11:]) * 1e3:.1f} us (local/deep)" for n, v in per.items()),
        f"info {b.info()}")
    del b, kvc, model
