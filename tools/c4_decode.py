"""Decode tok/s over the configs[3] 32k context (persistent kernel), after the user prefill
(diagnostics: run-to-run variance of the C4 decode block)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_14085_b200 import edgekv as ek
ctx = ek.Context(0); st = ctx.stream
L, H, d, S, U = 22, 32, 64, 32768, 16
m = ek.EdgeModel(ctx, L, H, d, S + U + 700); m.synthesize(1234)
kvc = ek.AssembledContext(m, S, [16] * 11 + [8] * 11, group=d); kvc.synthesize(99)
for trial in range(3):
    s = ek.Session(m, kvc, U + 420)
    s.forward(torch.empty((U, H * d), device="cuda").uniform_(-1, 1)); s.decode(5)
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(st); s.decode(100, sync=False); e1.record(st); st.synchronize()
        print(f"trial {trial} rep {rep}: {100 / e0.elapsed_time(e1) * 1e3:.0f} tok/s")
    del s
