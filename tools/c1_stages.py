"""Wall-clock of each C-ABI call of the configs[0] device path (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_14085_b200 import edgekv as ek
ctx = ek.Context(0)
S, U, T = 512, 16, 64
mp = S + U + 2048
edge = ek.EdgeModel(ctx, 4, 8, 32, mp); edge.synthesize(13)
cloud = ek.EdgeModel(ctx, 8, 8, 64, mp); cloud.synthesize(11)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
def t(name, fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"{name:28s} {1e3 * (time.perf_counter() - t0):8.2f} ms"); return r
for it in range(2):
    print("--- run", it)
    pe = dev(ek.generate_embeddings(1, 64, 256)); pc = dev(ek.generate_embeddings(1, 64, 512))
    t("prefill edge 64", lambda: ek.prefill(edge, pe))
    t("prefill cloud 64", lambda: ek.prefill(cloud, pc))
    dm = t("deep_match", lambda: ek.deep_match(edge, cloud, pe, pc, 2, 0.0, -1.0))[0]
    ee = dev(ek.generate_embeddings(2, S, 256)); ec = dev(ek.generate_embeddings(2, S, 512))
    t("prefill edge 512 (kv)", lambda: ek.prefill(edge, ee, want_kv=True))
    t("prefill cloud 512 (all)", lambda: ek.prefill(cloud, ec, want_x0=True, want_kv=True))
    kvc = ek.AssembledContext(edge, S, [16, 16, 8, 8], group=32)
    t("prompt_context", lambda: ek.prompt_context(edge, cloud, ee, ec, dm, 0.5, kvc))
    sess = t("session create", lambda: ek.Session(edge, kvc, U + T))
    ue = ek.generate_embeddings(3, U, 256).astype(np.float32)
    t("collaborative_decode", lambda: ek.collaborative_decode(sess, ue, T))
