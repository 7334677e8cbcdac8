"""C-ABI NCCL link throughput (2 ranks under torchrun): the 11 int8 deep layers of the C2
context (98 MB) from rank 0 to rank 1, per EKV_LINK_GROUP setting (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2505_14085_b200 import edgekv as ek
from paper_2505_14085_b200.dist import capi_link
dist.init_process_group("nccl")
r = dist.get_rank(); torch.cuda.set_device(r)
ctx = ek.Context(r)
L, H, d, S = 22, 32, 64, 2048
m = ek.EdgeModel(ctx, L, H, d, S + 64); m.synthesize(1)
kv = ek.AssembledContext(m, S, [16] * 11 + [8] * 11, group=d); kv.synthesize(2)
sess = ek.Session(m, kv, 4)
link = capi_link(ctx)
layers = list(range(11, 22))
ts = []
for rep in range(6):
    if r == 0:
        ts.append(link.send_layers(kv, layers, 1))
    else:
        ts.append(link.recv_forward(sess, layers, 0)[1])
    dist.barrier()
if r == 0:
    best = min(ts[1:])
    print(f"EKV_LINK_GROUP={os.environ.get('EKV_LINK_GROUP', '1')}: best {best * 1e3:.3f} ms "
          f"= {98041856 / best / 1e9:.0f} GB/s (all: {[round(t * 1e3, 3) for t in ts]})", flush=True)
dist.destroy_process_group()
