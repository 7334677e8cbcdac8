"""K3 (batched gather + quantise + pack) launch-time probe: how the source layout
(one contiguous [m][H][S][d_c] tensor vs one allocation per layer), the kept mask and
the destination (separate tensors vs assembled-context storage) change the launch."""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2505_14085_b200 import edgekv as ek

ctx = ek.Context(0)
st = ctx.stream
H, S, dc, d, m = 32, int(os.environ.get("S", 2048)), 128, 64, 11
HBM = 6551.4


def timeit(fn, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = []
    for it in range(reps + 1):
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            torch.cuda._sleep(400_000)
        e0.record(st)
        fn()
        e1.record(st)
        st.synchronize()
        if it:
            out.append(e0.elapsed_time(e1))
    return statistics.median(out)


one = torch.empty((m, H, S, dc), dtype=torch.bfloat16, device="cuda")
ctx.fill_uniform_bf16(one, 7, 3, -1, 1)
sep = [torch.empty((H, S, dc), dtype=torch.bfloat16, device="cuda") for _ in range(2 * m)]
for i, t in enumerate(sep):
    ctx.fill_uniform_bf16(t, 7, 100 + i, -1, 1)
codes = torch.empty((2 * m, H, S, d), dtype=torch.uint8, device="cuda")
scales = torch.empty((2 * m, H, S, 1), dtype=torch.float32, device="cuda")
model = ek.EdgeModel(ctx, 22, H, d, S + 8)
kvc = ek.AssembledContext(model, S, [16] * 11 + [8] * 11, group=d)
ctx.synchronize()
arr = lambda xs: (C.c_void_p * len(xs))(*xs)
nbytes = 2 * m * (H * S * dc * 2 + H * S * d + H * S * 4)
for kept_name, kept in (("even", torch.arange(0, dc, 2, dtype=torch.int32, device="cuda")),
                        ("random", torch.sort(torch.randperm(dc, device="cuda")[:d]).values.int())):
    for src_name, srcs in (("contiguous", [one[i // 2].data_ptr() for i in range(2 * m)]),
                           ("separate", [t.data_ptr() for t in sep])):
        for dst_name in ("tensors", "kvctx"):
            if dst_name == "tensors":
                cd = [codes[i].data_ptr() for i in range(2 * m)]
                sc = [scales[i].data_ptr() for i in range(2 * m)]
            else:
                cd, sc = [], []
                for le in range(11, 22):
                    s = kvc.segment(le)
                    cd += [s.k, s.v]
                    sc += [s.k_scales, s.v_scales]
            js, jc, jsc = arr(srcs), arr(cd), arr(sc)
            ms = timeit(lambda: ek.compress_batched(ctx, 2 * m, js, H * S, dc, kept, d, 8, d, jc, jsc))
            print(f"kept={kept_name:6s} src={src_name:10s} dst={dst_name:7s}: {ms * 1e3:7.1f} us "
                  f"{nbytes / ms / 1e6:7.0f} GB/s = {nbytes / ms / 1e6 / HBM:.3f} of HBM")
