"""The configs[1] user prefill (16 rows over the S=2048 [11 bf16 | 11 int8] context) timed with
CUDA events, repeated (diagnostics; run under ncu for the per-kernel split)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_14085_b200 import edgekv as ek
ctx = ek.Context(0); st = ctx.stream
L, H, d, S, U = 22, 32, 64, int(os.environ.get("S", 2048)), int(os.environ.get("U", 16))
m = ek.EdgeModel(ctx, L, H, d, S + 64); m.synthesize(1234)
kvc = ek.AssembledContext(m, S, [16] * 11 + [8] * 11, group=d); kvc.synthesize(99)
s = ek.Session(m, kvc, U + 8)
ue = torch.empty((U, H * d), device="cuda").uniform_(-1, 1)
for it in range(int(os.environ.get("REPS", 4))):
    s.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(st); s.forward(ue); e1.record(st); st.synchronize()
    print(f"prefill {U} rows over S={S}: {e0.elapsed_time(e1):.3f} ms")
