import time, sys, os
sys.path.insert(0, '/root/repo')
import torch
from paper_2505_14085_b200 import edgekv as ek
t = time.time()
print("maps before:", [l.split()[-1] for l in open('/proc/self/maps') if 'nccl' in l][:2], flush=True)
uid = ek.Link.unique_id()
print("uid ok", len(uid), time.time() - t, flush=True)
print("maps after:", sorted(set(l.split()[-1] for l in open('/proc/self/maps') if 'nccl' in l)), flush=True)
