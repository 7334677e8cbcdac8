"""Decode tok/s of the persistent kernel on the C2 edge model vs context length S, for the
current EKV_MEGA_PREFETCH setting (diagnostics: where the L2 prefetch warp stops paying)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_14085_b200 import edgekv as ek
ctx = ek.Context(0); st = ctx.stream
L, H, d, U = 22, 32, 64, 16
out = []
for S in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024,2048,4096,8192,16384").split(",")]:
    m = ek.EdgeModel(ctx, L, H, d, S + U + 400); m.synthesize(1234)
    kvc = ek.AssembledContext(m, S, [16] * 11 + [8] * 11, group=d); kvc.synthesize(99)
    s = ek.Session(m, kvc, U + 320)
    s.forward(torch.empty((U, H * d), device="cuda").uniform_(-1, 1)); s.decode(5)
    best = 0.0
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(st); s.decode(100, sync=False); e1.record(st); st.synchronize()
        best = max(best, 100 / e0.elapsed_time(e1) * 1e3)
    out.append(f"S={S}: {best:.0f}")
    del s, kvc, m
print(f"PF={os.environ.get('EKV_MEGA_PREFETCH', 'default')}:", ", ".join(out))
