"""GPU parity at the exact shapes bench.py times (BASELINE.json configs[1], "C2").

The other GPU suites pin every kernel at small shapes; this file runs the
configurations the headline numbers are measured on, against the same oracle:

* K8 (the persistent decode-step kernel, the bench's `value`): 22 layers x
  32 heads x 64, S = 2048, layers 11-21 int8 from 128-wide cloud heads, the
  128-CTA grid (4 CTAs per head), teacher-forced per step vs the oracle's
  collaborative_decode (cache_merge.cpp:230-273), through the host-buffer C-ABI
  call bench.py's e2e uses.
* K1 (tcgen05 grouped GEMM) over the 11 matched 4096-wide cloud layers bench.py
  aligns: 2816 tiles = 19 per CTA, so both TMEM accumulators and every
  tfull/tempty phase flip run; column sums vs an fp64 GEMM, and the mask vs the
  oracle's select_channels (head_prune.cpp:83-108) on the identical bf16 inputs.
* the batched path (K9-K12) at 128 sessions x 22 layers x 32 heads, sessions
  {0, 63, 127} spot-checked against the oracle.

Bars: normwise max|gpu-ref|/max|ref| <= 1e-3 per output row (fp32 outputs);
masks bit-exact (the cut margin must exceed 1e-6 -- a near tie fails, it does
not skip).
"""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import bf16_to_f64
from test_gpu_decode import TOL, make_context, normwise

pytestmark = pytest.mark.gpu

L, H, D, S, DEEP = 22, 32, 64, 2048, 11
HC, DC, LC = 32, 128, 32


@pytest.fixture(scope="module")
def ek():
    from paper_2505_14085_b200 import build
    build.build()
    from paper_2505_14085_b200 import edgekv
    return edgekv


@pytest.fixture(scope="module")
def ctx(ek):
    return ek.Context(0)


def synth_model(ek, ctx, n_layers, heads, d, max_pos, seed):
    """The bench's random-init edge model (ekv_model_synthesize on the device), read
    back so the oracle consumes the identical bf16 weights (exact in fp64)."""
    from paper_2505_14085_b200.capi import call
    m = ek.EdgeModel(ctx, n_layers, heads, d, max_pos)
    m.synthesize(seed)
    h = heads * d
    w0, _ = m.weight_ptrs(0)
    allw = np.zeros(n_layers * 4 * h * h, np.uint16)
    call("ekv_copy", ctx.h, allw.ctypes.data_as(C.c_void_p), C.c_void_p(w0), allw.nbytes, 1)
    g = C.c_void_p(); b = C.c_void_p(); p = C.c_void_p()
    call("ekv_model_io", m.hnd, C.byref(g), C.byref(b), C.byref(p))
    gamma = np.zeros(h, np.float32); bias = np.zeros(h, np.float32)
    pos = np.zeros(max_pos * h, np.uint16)
    for dst, src in ((gamma, g), (bias, b), (pos, p)):
        call("ekv_copy", ctx.h, dst.ctypes.data_as(C.c_void_p), src, dst.nbytes, 1)
    allw = allw.reshape(n_layers, 4 * h, h)
    f64 = dict(L=n_layers, H=heads, d=d, max_pos=max_pos,
               wqkvT=bf16_to_f64(allw[:, :3 * h]), woT=bf16_to_f64(allw[:, 3 * h:]),
               gamma=gamma.astype(np.float64), bias=bias.astype(np.float64),
               pos=bf16_to_f64(pos).reshape(max_pos, h))
    return m, f64


@pytest.fixture(scope="module")
def c2(ek, ctx, oracle):
    U, T = 3, 3
    max_pos = S + U + T + 8
    model, f64 = synth_model(ek, ctx, L, H, D, max_pos, seed=1234)
    formats = [16] * (L - DEEP) + [8] * DEEP
    kvc, ck, cv = make_context(ek, ctx, oracle, model, S, formats, seed=99, d_c=DC)
    return dict(model=model, f64=f64, kvc=kvc, ck=ck, cv=cv, U=U, T=T)


def test_k8_decode_at_c2_matches_oracle(ek, ctx, oracle, c2):
    """The bench's headline kernel at its own configuration."""
    U, T = c2["U"], c2["T"]
    h = H * D
    sess = ek.Session(c2["model"], c2["kvc"], U + T)
    assert sess.set_decode_path("mega") == "mega"
    ue = oracle.generate_embeddings(4242, U, h).astype(np.float32)
    pre, steps = ek.collaborative_decode(sess, ue, T)
    teacher = np.vstack([pre[-1:], steps[:-1]]).astype(np.float64)
    wp, ws = oracle.collaborative_decode(c2["f64"], c2["ck"], c2["cv"], ue.astype(np.float64), T,
                                         teacher=teacher, user_kv_bf16=True)
    errs = [normwise(pre[r], wp[r]) for r in range(U)] + [normwise(steps[t], ws[t]) for t in range(T)]
    assert max(errs) <= TOL, errs
    # 4 CTAs per head = one thread-block cluster per head (DSMEM q/k/v + partial
    # exchange); the global tagged-word exchange computes the identical bits
    sess.reset()
    import os
    os.environ["EKV_MEGA_CLUSTER"] = "0"
    try:
        pre_n, steps_n = ek.collaborative_decode(sess, ue, T)
    finally:
        del os.environ["EKV_MEGA_CLUSTER"]
    assert np.array_equal(steps_n, steps) and np.array_equal(pre_n, pre)
    # the prefill rows' context attention on the tensor cores (K10 + K11, the default)
    # against the split-KV kernel K4
    sess.reset()
    os.environ["EKV_PREFILL_K4"] = "1"
    try:
        pre_k4, _ = ek.collaborative_decode(sess, ue, 1)
    finally:
        del os.environ["EKV_PREFILL_K4"]
    assert max(normwise(pre[r], pre_k4[r].astype(np.float64)) for r in range(U)) <= 1e-4
    # the per-layer-kernel graph path agrees with the persistent kernel at this shape
    sess.reset()
    assert sess.set_decode_path("graph") == "graph"
    pre_g, steps_g = ek.collaborative_decode(sess, ue, T)
    assert normwise(pre_g, pre.astype(np.float64)) <= 1e-4
    assert max(normwise(steps_g[t], steps[t].astype(np.float64)) for t in range(T)) <= 1e-4


def test_batched_path_at_c2_128_sessions(ek, ctx, oracle, c2):
    """configs[2]'s per-GPU batch (128 sessions) on the C2 model and context."""
    from test_gpu_batch import check_sessions
    U, T, B = 2, 2, 128
    h = H * D
    batch = ek.SessionBatch(c2["model"], c2["kvc"], B, U + T)
    ue = np.stack([oracle.generate_embeddings(5000 + b, U, h) for b in range(B)]).astype(np.float32)
    pre, steps = ek.collaborative_decode_batch(batch, ue, T)
    assert np.all(np.isfinite(steps))
    check_sessions(oracle, c2["f64"], c2["ck"], c2["cv"], ue, pre, steps, [0, 63, 127])


def test_k1_mask_at_bench_shape(ek, ctx, oracle):
    """K1 over the bench's 11 matched cloud layers (S=2048, h_c=4096): 2816 tiles on
    148 CTAs.  Column sums vs an fp64 GEMM; mask vs oracle select_channels."""
    m = 11
    hc = HC * DC
    X = torch.empty((m, S, hc), dtype=torch.bfloat16, device="cuda")
    Wq = torch.empty((m, hc, hc), dtype=torch.bfloat16, device="cuda")
    Kc = torch.empty((m, HC, S, DC), dtype=torch.bfloat16, device="cuda")
    ctx.fill_uniform_bf16(X, 7, 1, -1.0, 1.0)       # the bench's inputs (bench.py run_b200)
    ctx.fill_uniform_bf16(Wq, 7, 2, -0.02, 0.02)
    ctx.fill_uniform_bf16(Kc, 7, 3, -1.0, 1.0)
    ctx.synchronize()
    got = ek.align_qnorm(ctx, X, Wq)                 # [m][hc] fp64
    want = torch.empty_like(got)
    q_rows = []
    for i in range(m):
        q = X[i].double() @ Wq[i].double().T        # fp64 GEMM of the identical bf16 values
        want[i] = (q * q).sum(dim=0)
        q_rows.append(q.reshape(S, HC, DC).transpose(0, 1).reshape(-1, DC).cpu().numpy())
        del q
    rel = ((got - want).abs() / want).max().item()
    assert rel < 1e-5, rel
    kept, margin, q_c, k_c = ek.select_channels(ctx, X, Wq, Kc, 0.5, DC)
    assert margin > 1e-6, f"near tie at the cut ({margin:.2e}): mask parity undecidable"
    q_stack = np.concatenate(q_rows)
    del q_rows
    k_stack = Kc.double().reshape(-1, DC).cpu().numpy()
    want_kept, _ = oracle.select_channels(q_stack, k_stack, oracle.prune_retained(0.5, DC))
    assert kept.tolist() == want_kept.tolist()
