"""Time the user-prompt prefill (graph-path kernels, R <= 8 rows per chunk) at the C2 shapes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_14085_b200 import edgekv as ek
L, H, d, S, DEEP = 22, 32, 64, int(os.environ.get("S", 2048)), 11
ctx = ek.Context(0)
model = ek.EdgeModel(ctx, L, H, d, S + 200); model.synthesize(seed=1234)
kvc = ek.AssembledContext(model, S, [16] * (L - DEEP) + [8] * DEEP, group=d); kvc.synthesize(seed=99)
sess = ek.Session(model, kvc, 100)
for U in (1, 8, 16):
    emb = torch.empty((U, H * d), device="cuda").uniform_(-1, 1)
    ts = []
    for _ in range(5):
        sess.reset(); torch.cuda.synchronize(); t = time.perf_counter()
        sess.forward(emb); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    e2e = []
    ue = np.random.uniform(-1, 1, (U, H * d)).astype(np.float32)
    for _ in range(3):
        t = time.perf_counter(); ek.collaborative_decode(sess, ue, 64); e2e.append(time.perf_counter() - t)
    prof = np.mean([sess.profile_step() for _ in range(3)], axis=0) if False else None
    print(f"S={S} U={U}: prefill {1e3*min(ts):.2f} ms ; collaborative_decode(U, 64 steps) {1e3*min(e2e):.2f} ms")
