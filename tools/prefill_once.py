import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_14085_b200 import edgekv as ek
L, H, d, S, DEEP = 22, 32, 64, 2048, 11
ctx = ek.Context(0)
model = ek.EdgeModel(ctx, L, H, d, S + 200); model.synthesize(seed=1234)
kvc = ek.AssembledContext(model, S, [16] * (L - DEEP) + [8] * DEEP, group=d); kvc.synthesize(seed=99)
sess = ek.Session(model, kvc, 100)
emb = torch.empty((8, H * d), device="cuda").uniform_(-1, 1)
sess.forward(emb); sess.reset(); sess.forward(emb)
