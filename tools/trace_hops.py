"""Split the intra-head waits of the persistent decode step into skew (waiting for the
slowest CTA of the head) and hop latency (after the slowest CTA published): per layer
and head, hop = stamp[k_done] - max over the head's CTAs of stamp[k_pub] (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_14085_b200 import edgekv as ek
L, H, d, S, DEEP = 22, 32, 64, 2048, 11
ctx = ek.Context(0)
G0 = torch.cuda.get_device_properties(0).multi_processor_count
m = ek.EdgeModel(ctx, L, H, d, S + 256); m.synthesize(1)
kvc = ek.AssembledContext(m, S, [16] * (L - DEEP) + [8] * DEEP, group=d); kvc.synthesize(2)
sess = ek.Session(m, kvc, 128)
sess.forward(torch.zeros((16, H * d), device="cuda")); sess.decode(3)
res = {"qkv": [], "merge": [], "x": []}
for rep in range(5):
    t = sess.trace_step(G0).astype(np.int64)
    G = t.size // (16 * (L + 1))
    t = t.reshape(L + 1, G, 16)[:L, :, :8]
    per = G // H
    for l in range(1, L):
        for h in range(H):
            cs = slice(h * per, (h + 1) * per)
            pub_a = t[l, cs, 2].max()            # slowest A of the head's CTAs (q/k/v rows)
            res["qkv"].append(np.mean(t[l, cs, 3] - pub_a) / 1e3)
            pub_b = t[l, cs, 4].max()            # slowest attention partial of the head
            res["merge"].append(np.mean(t[l, cs, 5] - pub_b) / 1e3)
        pub_r = t[l - 1, :, 7].max()             # slowest R of the previous layer
        res["x"].append(np.mean(t[l, :, 1] - pub_r) / 1e3)
for k, v in res.items():
    print(f"{k:6s} hop after the slowest producer: mean {np.mean(v):.2f} us, median {np.median(v):.2f}, p90 {np.percentile(v, 90):.2f}")
