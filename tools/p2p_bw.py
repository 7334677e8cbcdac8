import os, torch, torch.distributed as dist, time
dist.init_process_group("nccl"); r = dist.get_rank(); torch.cuda.set_device(r)
for nb in [256 << 10, 4 << 20, 9 << 20, 98 << 20]:
    t = torch.empty(nb, dtype=torch.uint8, device="cuda")
    for rep in range(8):
        torch.cuda.synchronize(); dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if r == 0: dist.send(t, 1)
        else: dist.recv(t, 0)
        e1.record(); torch.cuda.synchronize()
        if rep == 7 and r == 1: print(f"{nb/1e6:.1f} MB: {e0.elapsed_time(e1):.3f} ms = {nb/e0.elapsed_time(e1)/1e6:.0f} GB/s", flush=True)
dist.destroy_process_group()
