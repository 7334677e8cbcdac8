"""Decode tok/s of the persistent kernel at BASELINE configs[0]'s edge (4L 8x32, S=512) for
a given EKV_MEGA_GRID (diagnostics: grid-size sweep for small models)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_14085_b200 import edgekv as ek
ctx = ek.Context(0); st = ctx.stream
for L, H, d, S, fm in [(4, 8, 32, 512, [16, 16, 8, 8]), (22, 32, 64, 2048, [16] * 11 + [8] * 11)]:
    m = ek.EdgeModel(ctx, L, H, d, S + 1024); m.synthesize(13)
    kvc = ek.AssembledContext(m, S, fm, group=d); kvc.synthesize(2)
    s = ek.Session(m, kvc, 16 + 700); s.forward(torch.zeros((16, H * d), device="cuda")); s.decode(5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(st); s.decode(300, sync=False); e1.record(st); st.synchronize()
    print(f"L={L} h={H*d} grid={os.environ.get('EKV_MEGA_GRID', 'default')}: {300 / e0.elapsed_time(e1) * 1e3:.0f} tok/s")
