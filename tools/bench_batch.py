"""Batched-session decode sweep at the C2 shapes (BASELINE configs[2] on one GPU):
B sessions over one shared S=2048 context ([11 local bf16 | 11 cloud int8] layers),
U user rows each, then timed decode steps.  Prints one JSON line per B.

  python tools/bench_batch.py [--sessions 64,128,256] [--steps 20] [--warmup 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_14085_b200 import edgekv as ek  # noqa: E402

L, H, d, S, U, DEEP = 22, 32, 64, 2048, 16, 11


def step_bytes(B, rows_attended):
    h = H * d
    w = L * 4 * h * h * 2
    ctx = (L - DEEP) * 2 * H * S * d * 2 + DEEP * 2 * H * S * (d + 4)
    user = B * L * 2 * H * rows_attended * d * 2
    return w + ctx + user


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sessions", default="1,8,64,128,256")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    ctx = ek.Context(0)
    st = ctx.stream
    h = H * d
    for B in [int(x) for x in a.sessions.split(",")]:
        cap = U + a.warmup + a.steps + 4
        model = ek.EdgeModel(ctx, L, H, d, S + cap + 8)
        model.synthesize(seed=1234)
        kvc = ek.AssembledContext(model, S, [16] * (L - DEEP) + [8] * DEEP, group=d)
        kvc.synthesize(seed=99)
        batch = ek.SessionBatch(model, kvc, B, cap)
        emb = torch.empty((B, U, h), device="cuda").uniform_(-1, 1)
        torch.cuda.synchronize()
        batch.forward(emb)
        batch.decode(a.warmup)
        out = torch.empty((a.steps, B, h), device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            torch.cuda._sleep(200_000)
        e0.record(st)
        batch.decode(a.steps, out, sync=False)
        e1.record(st)
        st.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        rows = U + a.warmup + a.steps / 2.0
        gb = step_bytes(B, rows) / 1e9
        prof = np.mean([batch.profile_row() for _ in range(2)], axis=0) * 1e3  # us
        Lr = (len(prof) - 2) // 5
        parts = {k: float(prof[1 + i:1 + 5 * Lr:5].sum()) for i, k in
                 enumerate(["qkv_us", "ctx_us", "user_us", "out_us", "sum_us"])}
        parts["xprep0_us"] = float(prof[0])
        print(json.dumps({"B": B, "ms_per_step": ms, "tok_s": B / ms * 1e3, "GB_per_step": gb,
                          "GB_s": gb / ms * 1e3, "finite": bool(torch.isfinite(out).all().item()),
                          "kernels_per_step_us": parts, **batch.info()}), flush=True)
        del batch, model, kvc


if __name__ == "__main__":
    main()
