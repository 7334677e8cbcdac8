"""Python host layer over the C ABI, mirroring the reference's interface.

Names, argument meaning and error texts follow namespace edgekv of the
reference (/root/reference/proj/include/edgekv/*.hpp), so the parity tests read
like the reference's own tests.  Device memory, streams and process groups
come from PyTorch (plumbing); every computation is a call into libekv.so.

Data layouts:
  cloud / edge KV         [layer][head][token][head_dim]  (reference KVCache [l][h] matrices)
  weights                 out-feature-major bf16 (W^T), QKV fused: wqkvT [3h][h], woT [h][h]
  compressed KV           codes [head][token][d_e*bits/8], scales fp32 [head][token][d_e/group]
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import capi
from .capi import EKV_KV_BF16, EKV_KV_INT4, EKV_KV_INT8, EkvError, call, ekv_model_config, ekv_segment

__all__ = [
    "Context", "EkvError", "prune_retained", "align_qnorm", "kv_colnorm", "rank_channels",
    "select_channels", "prune_cache", "kv_compress", "kv_dequant", "decode_attention",
    "match_layers", "match_layers_dev", "prefill", "deep_match", "prompt_context", "cache_source", "pipeline_schedule", "EdgeModel", "AssembledContext",
    "Session", "collaborative_decode", "build_deep_kv", "EKV_KV_BF16", "EKV_KV_INT8",
    "EKV_KV_INT4",
]


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


class Context:
    """ekv_ctx: one device + one CUDA stream (a torch.cuda.Stream we own)."""

    def __init__(self, device: int = 0):
        torch.cuda.set_device(device)
        self.device = device
        self.stream = torch.cuda.Stream(device=device)
        h = C.c_void_p()
        call("ekv_ctx_create", device, C.c_void_p(self.stream.cuda_stream), C.byref(h))
        self.h = h

    def synchronize(self):
        call("ekv_ctx_synchronize", self.h)

    def launches(self) -> int:
        n = C.c_int64()
        call("ekv_ctx_kernel_launches", self.h, C.byref(n))
        return n.value

    def memset(self, t: torch.Tensor, value: int = 0):
        """Byte fill of a device tensor on the context stream (no torch kernel)."""
        call("ekv_memset", self.h, _ptr(t), value, t.numel() * t.element_size())
        return t

    def fill_uniform_bf16(self, out: torch.Tensor, seed: int, stream_id: int, lo: float, hi: float):
        assert out.dtype == torch.bfloat16 and out.is_contiguous()
        call("ekv_fill_uniform_bf16", self.h, _ptr(out), out.numel(), seed, stream_id, lo, hi)
        return out

    def __del__(self):
        try:
            if getattr(self, "h", None):
                capi.load().ekv_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass


def _sync_in():
    torch.cuda.current_stream().synchronize()


# ------------------------------------------------------------------ stage 1
def mix(a: int, b: int) -> int:
    """Rng::mix (rng.hpp:35-40), the splitmix64 finaliser seeding every substream."""
    m = (1 << 64) - 1
    z = (a + 0x9E3779B97F4A7C15 * (b + 1)) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def generate_embeddings(seed: int, n: int, h: int) -> np.ndarray:
    """generate_embeddings (transformer.cpp:308-317) through the C ABI: fp64 [n][h]."""
    out = np.zeros((n, h), np.float64)
    call("ekv_generate_embeddings", seed, n, h, _dp(out))
    return out


def prune_retained(lam: float, head_dim: int) -> int:
    """PruneSpec::from_lambda(lambda, head_dim).retained (head_prune.cpp:14-22)."""
    r = C.c_int()
    call("ekv_prune_retained", lam, head_dim, C.byref(r))
    return r.value


def align_qnorm(ctx: Context, X: torch.Tensor, WqT: torch.Tensor, colsq: torch.Tensor | None = None):
    """K1: per-column sum over tokens of (X W_Q)^2 for m layers at once.
    X bf16 [m][S][h_c] (or [S][h_c]), WqT bf16 [m][n_cols][h_c] -> fp64 [m][n_cols]."""
    if X.dim() == 2:
        X = X.unsqueeze(0)
        WqT = WqT.unsqueeze(0)
    m, S, hc = X.shape
    n = WqT.shape[1]
    assert WqT.shape == (m, n, hc) and X.dtype == WqT.dtype == torch.bfloat16
    _sync_in()
    if colsq is None:
        colsq = torch.empty((m, n), dtype=torch.float64, device=X.device)
        ctx.memset(colsq)
    call("ekv_align_qnorm", ctx.h, _ptr(X), _ptr(WqT), m, S, hc, n, _ptr(colsq))
    ctx.synchronize()
    return colsq


def kv_colnorm(ctx: Context, K: torch.Tensor, colsq: torch.Tensor | None = None):
    """K2: per-channel sum of squares over every row of K (bf16 [..., d_c]) -> fp64 [d_c]."""
    d = K.shape[-1]
    _sync_in()
    if colsq is None:
        colsq = torch.empty(d, dtype=torch.float64, device=K.device)
        ctx.memset(colsq)
    call("ekv_kv_colnorm", ctx.h, _ptr(K), K.numel() // d, d, _ptr(colsq))
    ctx.synchronize()
    return colsq


def rank_channels(q_colsq, k_colsq, retained: int):
    """Reference ranking rule on column sums of squares (head_prune.cpp:98-107).
    Returns (kept int32 ascending, cut margin)."""
    q = np.ascontiguousarray(np.asarray(q_colsq, dtype=np.float64))
    k = np.ascontiguousarray(np.asarray(k_colsq, dtype=np.float64))
    kept = np.zeros(max(retained, 1), dtype=np.int32)
    margin = C.c_double()
    call("ekv_rank_channels", _dp(q), _dp(k), len(q), retained, _ip(kept), C.byref(margin))
    return kept[:retained].copy(), margin.value


def select_channels(ctx: Context, X: torch.Tensor, WqT: torch.Tensor, K: torch.Tensor, lam: float,
                    d_c: int):
    """select_channels (head_prune.cpp:83-108) over the stacked rows of every matched
    layer and head, with Q recomputed on the tensor cores (K1) and K norms read
    from the cloud cache (K2).  Returns (kept, margin, q_colsq, k_colsq)."""
    qs = align_qnorm(ctx, X, WqT).cpu().numpy()               # [m][H*d_c]
    q_c = qs.reshape(-1, d_c).sum(axis=0)                     # fp64 over layers and heads
    k_c = kv_colnorm(ctx, K).cpu().numpy()
    retained = prune_retained(lam, d_c)
    kept, margin = rank_channels(q_c, k_c, retained)
    return kept, margin, q_c, k_c


def prune_cache(ctx: Context, kv: torch.Tensor, kept) -> torch.Tensor:
    """prune_cache column slice (head_prune.cpp:170-197): bf16 [..., d_c] -> [..., d_e]."""
    kept_t = kept.to(device=kv.device, dtype=torch.int32) if isinstance(kept, torch.Tensor) else \
        torch.as_tensor(np.asarray(kept, dtype=np.int32), device=kv.device)
    d_c, d_e = kv.shape[-1], kept_t.numel()
    out = torch.empty(kv.shape[:-1] + (d_e,), dtype=kv.dtype, device=kv.device)
    _sync_in()
    call("ekv_kv_gather", ctx.h, _ptr(kv), kv.numel() // d_c, d_c, _ptr(kept_t), d_e, _ptr(out))
    ctx.synchronize()
    return out


def kv_compress(ctx: Context, src: torch.Tensor, kept, bits: int = 8, group: int | None = None,
                codes: torch.Tensor | None = None, scales: torch.Tensor | None = None):
    """K3: gather kept channels + quantise + pack.  src bf16 [..., d_c]."""
    kept_t = kept if isinstance(kept, torch.Tensor) else torch.as_tensor(
        np.asarray(kept, dtype=np.int32), device=src.device)
    d_c, d_e = src.shape[-1], kept_t.numel()
    group = group or (d_e if bits == 8 else 32)
    rows = src.numel() // d_c
    if codes is None:
        codes = torch.empty(src.shape[:-1] + (d_e * bits // 8,), dtype=torch.uint8, device=src.device)
    if scales is None:
        scales = torch.empty(src.shape[:-1] + (d_e // group,), dtype=torch.float32, device=src.device)
    _sync_in()
    call("ekv_kv_compress", ctx.h, _ptr(src), rows, d_c, _ptr(kept_t), d_e, bits, group,
         _ptr(codes), _ptr(scales))
    ctx.synchronize()
    return codes, scales


def kv_dequant(ctx: Context, codes: torch.Tensor, scales: torch.Tensor, d_e: int, bits: int,
               group: int) -> torch.Tensor:
    """K6: bf16_rn(code * scale)."""
    rows = codes.numel() // (d_e * bits // 8)
    out = torch.empty(codes.shape[:-1] + (d_e,), dtype=torch.bfloat16, device=codes.device)
    _sync_in()
    call("ekv_kv_dequant", ctx.h, _ptr(codes), _ptr(scales), rows, d_e, bits, group, _ptr(out))
    ctx.synchronize()
    return out


# ------------------------------------------------------------------ stage 3
@dataclass
class Segment:
    """One layer's context segment (head-major)."""
    format: int
    S: int
    k: torch.Tensor | None = None
    v: torch.Tensor | None = None
    k_scales: torch.Tensor | None = None
    v_scales: torch.Tensor | None = None
    group: int = 0

    def c(self) -> ekv_segment:
        return ekv_segment(self.format, self.S, self.group, _ptr(self.k), _ptr(self.v),
                           _ptr(self.k_scales), _ptr(self.v_scales))


def decode_attention(ctx: Context, q: torch.Tensor, seg: Segment, user_k: torch.Tensor,
                     user_v: torch.Tensor, user_base: int, want_lse: bool = False):
    """K4: q fp32 [R][H][d]; user_k/v bf16 [H][cap][d]; row r sees user rows
    0..user_base+r (causal, cache_merge.cpp:206-207) and all S context rows."""
    R, H, d = q.shape
    out = torch.empty_like(q)
    lse = torch.empty((R, H), dtype=torch.float32, device=q.device) if want_lse else None
    cs = seg.c()
    _sync_in()
    call("ekv_decode_attention", ctx.h, R, H, d, _ptr(q), C.byref(cs), _ptr(user_k), _ptr(user_v),
         user_k.shape[1], user_base, _ptr(out), _ptr(lse))
    ctx.synchronize()
    return (out, lse) if want_lse else out


# ------------------------------------------------------------------ host logic
def match_layers(ctx: "Context", edge_outs: np.ndarray, cloud_outs: np.ndarray, theta_cka: float,
                 theta_rsa: float):
    """match_layers (layer_match.cpp:166-228) from host fp64 probe outputs, computed by K7
    on the device: returns (cka, rsa, best) with best[le] = -1 for an unmatched edge layer."""
    e = np.ascontiguousarray(edge_outs, dtype=np.float64)
    c = np.ascontiguousarray(cloud_outs, dtype=np.float64)
    me, n, ce = e.shape
    nc, _, cc = c.shape
    cka = np.zeros((me, nc)); rsa = np.zeros((me, nc)); best = np.zeros(me, dtype=np.int32)
    call("ekv_match_layers", ctx.h, _dp(e), me, ce, _dp(c), nc, cc, n, theta_cka, theta_rsa, _dp(cka),
         _dp(rsa), _ip(best))
    return cka, rsa, best


def match_layers_dev(ctx: "Context", edge_outs: torch.Tensor, cloud_outs: torch.Tensor,
                     theta_cka: float, theta_rsa: float):
    """K7: match_layers on the device over fp64 probe outputs already in HBM
    ([me][n][ce], [nc][n][cc]); bit-identical to the reference.  Returns numpy
    (cka, rsa, best)."""
    assert edge_outs.dtype == torch.float64 and cloud_outs.dtype == torch.float64
    e, c = edge_outs.contiguous(), cloud_outs.contiguous()
    me, n, ce = e.shape
    nc, _, cc = c.shape
    cka = np.zeros((me, nc)); rsa = np.zeros((me, nc)); best = np.zeros(me, dtype=np.int32)
    call("ekv_match_layers_dev", ctx.h, _ptr(e), me, ce, _ptr(c), nc, cc, n, theta_cka, theta_rsa,
         _dp(cka), _dp(rsa), _ip(best))
    return cka, rsa, best


def cache_source(layer: int, cost_local: float, cost_peer: float, boundary: int, m: int) -> str:
    out = C.c_int()
    call("ekv_cache_source", layer, cost_local, cost_peer, boundary, m, C.byref(out))
    return ("local", "peer", "cloud")[out.value]


def pipeline_schedule(t_comm, t_comp):
    a = np.ascontiguousarray(t_comm, dtype=np.float64)
    b = np.ascontiguousarray(t_comp, dtype=np.float64)
    pip = np.zeros(len(a)); s = C.c_double(); p = C.c_double()
    call("ekv_pipeline_schedule", _dp(a), _dp(b), len(a), _dp(pip), C.byref(s), C.byref(p))
    return pip, s.value, p.value


# ------------------------------------------------------------------ model / context / session
class EdgeModel:
    """ekv_model: the edge SLM (Model, transformer.hpp:76-83) resident in HBM."""

    def __init__(self, ctx: Context, num_layers: int, num_heads: int, head_dim: int,
                 max_positions: int):
        self.ctx = ctx
        self.L, self.H, self.d, self.max_pos = num_layers, num_heads, head_dim, max_positions
        self.h = num_heads * head_dim
        cfg = ekv_model_config(num_layers, num_heads, head_dim, max_positions)
        hnd = C.c_void_p()
        call("ekv_model_create", ctx.h, C.byref(cfg), C.byref(hnd))
        self.hnd = hnd

    def set_layer(self, layer: int, wqkvT_bf16: np.ndarray, woT_bf16: np.ndarray):
        a = np.ascontiguousarray(wqkvT_bf16, dtype=np.uint16)
        b = np.ascontiguousarray(woT_bf16, dtype=np.uint16)
        assert a.shape == (3 * self.h, self.h) and b.shape == (self.h, self.h)
        call("ekv_model_set_layer", self.hnd, layer, a.ctypes.data_as(C.c_void_p),
             b.ctypes.data_as(C.c_void_p))

    def set_io(self, gamma: np.ndarray, bias: np.ndarray, pos_bf16: np.ndarray):
        g = np.ascontiguousarray(gamma, dtype=np.float32)
        b = np.ascontiguousarray(bias, dtype=np.float32)
        p = np.ascontiguousarray(pos_bf16, dtype=np.uint16)
        assert p.shape == (self.max_pos, self.h)
        call("ekv_model_set_io", self.hnd, g.ctypes.data_as(C.c_void_p),
             b.ctypes.data_as(C.c_void_p), p.ctypes.data_as(C.c_void_p))

    def synthesize(self, seed: int, w_scale: float | None = None, pos_scale: float = 0.1):
        call("ekv_model_synthesize", self.hnd, seed,
             w_scale if w_scale is not None else float(np.sqrt(3.0 / self.h)), pos_scale)

    def weight_ptrs(self, layer: int):
        a = C.c_void_p(); b = C.c_void_p()
        call("ekv_model_weights", self.hnd, layer, C.byref(a), C.byref(b))
        return a.value, b.value

    def __del__(self):
        try:
            capi.load().ekv_model_destroy(self.hnd)
        except Exception:
            pass


class AssembledContext:
    """ekv_kvctx (AssembledContext, cache_merge.hpp:48-51): per-layer context KV,
    bf16 for local layers, int8/int4 for layers delivered from the cloud."""

    def __init__(self, model: EdgeModel, S: int, layer_formats, group: int = 0):
        self.model = model
        self.S = S
        fm = np.ascontiguousarray(np.asarray(layer_formats, dtype=np.int32))
        assert len(fm) == model.L
        self.formats = fm.tolist()
        self.group = group
        hnd = C.c_void_p()
        call("ekv_kvctx_create", model.hnd, S, _ip(fm), group, C.byref(hnd))
        self.hnd = hnd

    def segment(self, layer: int) -> ekv_segment:
        s = ekv_segment()
        call("ekv_kvctx_layer", self.hnd, layer, C.byref(s))
        return s

    def upload_bf16(self, layer: int, k_bf16: np.ndarray, v_bf16: np.ndarray):
        k = np.ascontiguousarray(k_bf16, dtype=np.uint16)
        v = np.ascontiguousarray(v_bf16, dtype=np.uint16)
        call("ekv_kvctx_upload_bf16", self.hnd, layer, k.ctypes.data_as(C.c_void_p),
             v.ctypes.data_as(C.c_void_p))

    def set_layer(self, layer: int, k: torch.Tensor, v: torch.Tensor,
                  k_scales: torch.Tensor | None = None, v_scales: torch.Tensor | None = None):
        """Deliver one layer from device tensors (bf16 K/V, or codes + scales)."""
        _sync_in()
        call("ekv_kvctx_set_layer", self.hnd, layer, _ptr(k), _ptr(v), _ptr(k_scales),
             _ptr(v_scales))
        self.model.ctx.synchronize()

    def synthesize(self, seed: int):
        call("ekv_kvctx_synthesize", self.hnd, seed)

    def copy_layers_from(self, peer: "AssembledContext", layers):
        """Peer sharing (sim.cpp:757-786): the listed layers of a peer's context (same
        geometry, any GPU of this process) copied device to device over NVLink."""
        ly = np.ascontiguousarray(layers, np.int32)
        call("ekv_kvctx_copy_layers", self.hnd, peer.hnd, _ip(ly), len(ly))

    def __del__(self):
        try:
            capi.load().ekv_kvctx_destroy(self.hnd)
        except Exception:
            pass


class _LayerUpload(C.Structure):
    _fields_ = [("k", C.c_void_p), ("v", C.c_void_p), ("ks", C.c_void_p), ("vs", C.c_void_p)]


class Session:
    """ekv_session: one request's user/generated KV cache + decode state."""

    def __init__(self, model: EdgeModel, context: AssembledContext, max_user_rows: int):
        self.model, self.context, self.cap = model, context, max_user_rows
        hnd = C.c_void_p()
        call("ekv_session_create", model.hnd, context.hnd, max_user_rows, C.byref(hnd))
        self.hnd = hnd

    def reset(self):
        call("ekv_session_reset", self.hnd)

    def forward(self, emb: torch.Tensor) -> torch.Tensor:
        """merged_forward over n new rows (device fp32 [n][h])."""
        emb = emb.contiguous().float()
        out = torch.empty_like(emb)
        _sync_in()
        call("ekv_session_forward", self.hnd, _ptr(emb), emb.shape[0], _ptr(out))
        self.model.ctx.synchronize()
        return out

    def forward_pipelined(self, emb: torch.Tensor, uploads: dict, overlap: bool = True,
                          measure_compute: bool = True):
        """Eq. 20 pipelined prefill: `uploads` = {layer: (k, v, k_scales, v_scales)} pinned host
        tensors (scales None for bf16 layers) copied into the context while the rows are
        forwarded.  Returns (out [n][h], t_comm_ms [L], t_comp_ms [L] | None, total_ms);
        measure_compute re-runs the rows kernel by kernel for t_comp_ms (diagnostic)."""
        emb = emb.contiguous().float()
        out = torch.empty_like(emb)
        L = self.model.L
        arr = (_LayerUpload * L)()
        keep = []
        for l, (k, v, ks, vs) in uploads.items():
            keep += [k, v, ks, vs]
            arr[l].k = k.data_ptr(); arr[l].v = v.data_ptr()
            arr[l].ks = ks.data_ptr() if ks is not None else None
            arr[l].vs = vs.data_ptr() if vs is not None else None
        tc = np.zeros(L, np.float32); tp = np.zeros(L, np.float32); tot = C.c_float()
        _sync_in()
        call("ekv_session_forward_pipelined", self.hnd, _ptr(emb), emb.shape[0], _ptr(out),
             C.cast(arr, C.c_void_p), 1 if overlap else 0, tc.ctypes.data_as(C.POINTER(C.c_float)),
             tp.ctypes.data_as(C.POINTER(C.c_float)) if measure_compute else None, C.byref(tot))
        return out, tc, (tp if measure_compute else None), tot.value

    def forward_pack(self, emb: torch.Tensor, pack: torch.Tensor) -> torch.Tensor:
        """Eq. 20 over an EKVPACK1 stream in (pinned) host memory: its layers are uploaded
        and hashed layer by layer while the rows are forwarded layer-major."""
        emb = emb.contiguous().float()
        out = torch.empty_like(emb)
        _sync_in()
        call("ekv_session_forward_pack", self.hnd, _ptr(emb), emb.shape[0], _ptr(out),
             C.c_void_p(pack.data_ptr()), pack.numel())
        return out

    def forward_streamed(self, emb: torch.Tensor, layer_events: dict, sync: bool = True) -> torch.Tensor:
        """Layer-major forward of n rows where layer l's attention waits on layer_events[l]
        (a torch.cuda.Event recorded by whoever delivers that context layer, e.g. the NCCL
        receive of dist.stream_layers); layers without an event are resident."""
        emb = emb.contiguous().float()
        out = torch.empty_like(emb)
        L = self.model.L
        evs = (C.c_void_p * L)()
        for l, ev in layer_events.items():
            if ev is not None:
                evs[l] = ev.cuda_event
        _sync_in()
        call("ekv_session_forward_streamed", self.hnd, _ptr(emb), emb.shape[0], _ptr(out),
             C.cast(evs, C.c_void_p))
        if sync:
            self.model.ctx.synchronize()
        return out

    def decode(self, steps: int, out: torch.Tensor | None = None, sync: bool = True) -> torch.Tensor:
        if out is None:
            out = torch.empty((steps, self.model.h), dtype=torch.float32,
                              device=f"cuda:{self.model.ctx.device}")
        call("ekv_session_decode", self.hnd, steps, _ptr(out))
        if sync:
            self.model.ctx.synchronize()
        return out

    def set_decode_path(self, path: str) -> str:
        """'mega' (one persistent kernel per step, default) or 'graph' (per-layer kernels in a
        CUDA graph).  Returns the path that will actually run."""
        act = C.c_int()
        call("ekv_session_set_decode_path", self.hnd, 0 if path == "mega" else 1, C.byref(act))
        return "mega" if act.value == 0 else "graph"

    def trace_step(self, num_sms: int) -> np.ndarray:
        """Persistent path: phase stamps and ring counters of one step, [16*(L+1)*G]
        (see ekv_capi.h)."""
        n = 16 * (self.model.L + 1) * num_sms
        out = np.zeros(n, dtype=np.uint64)
        got = C.c_int()
        call("ekv_session_trace_step", self.hnd, out.ctypes.data_as(C.POINTER(C.c_uint64)), n,
             C.byref(got))
        return out[:got.value]  # [L+1][G][16], G = the kernel's grid

    def profile_step(self) -> np.ndarray:
        """One real decode step with CUDA-event times (ms).  Graph path: [3l] QKV projection,
        [3l+1] attention, [3l+2] output projection, [3L] advance; persistent path: [0] = step."""
        n = 3 * self.model.L + 1
        out = np.zeros(n, dtype=np.float32)
        got = C.c_int()
        call("ekv_session_profile_step", self.hnd, out.ctypes.data_as(C.POINTER(C.c_float)), n,
             C.byref(got))
        return out[:got.value]

    def user_kv(self, layer: int):
        k = C.c_void_p(); v = C.c_void_p(); cap = C.c_int()
        call("ekv_session_user_kv", self.hnd, layer, C.byref(k), C.byref(v), C.byref(cap))
        return k.value, v.value, cap.value

    def __del__(self):
        try:
            capi.load().ekv_session_destroy(self.hnd)
        except Exception:
            pass


class Link:
    """ekv_link: the emulated cloud -> edge link over NCCL from the C ABI (one process per
    GPU): per-layer sends of the cloud context's deep layers, received into the edge's
    context while its user rows run layer-major (Eq. 20)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        call("ekv_link_unique_id", C.cast(buf, C.c_void_p))
        return buf.raw

    def __init__(self, ctx: Context, uid: bytes, nranks: int, rank: int):
        self.ctx = ctx
        hnd = C.c_void_p()
        call("ekv_link_create", ctx.h, C.c_char_p(uid), nranks, rank, C.byref(hnd))
        self.hnd = hnd

    def send_layers(self, context: "AssembledContext", layers, peer: int) -> float:
        ly = np.ascontiguousarray(layers, np.int32)
        sec = C.c_float()
        call("ekv_link_send_layers", self.hnd, context.hnd, _ip(ly), len(ly), peer, C.byref(sec))
        return sec.value

    def recv_forward(self, session: "Session", layers, peer: int, emb: torch.Tensor | None = None):
        """Receive `layers` into the session's context; with emb (fp32 [n][h], device) the rows
        are forwarded meanwhile.  Returns (out [n][h] | None, link seconds)."""
        ly = np.ascontiguousarray(layers, np.int32)
        sec = C.c_float()
        out = None
        n = 0
        if emb is not None:
            emb = emb.contiguous().float()
            out = torch.empty_like(emb)
            n = emb.shape[0]
            _sync_in()
        call("ekv_link_recv_forward", self.hnd, session.hnd, _ip(ly), len(ly), peer, _ptr(emb), n,
             _ptr(out), C.byref(sec))
        return out, sec.value

    def __del__(self):
        try:
            capi.load().ekv_link_destroy(self.hnd)
        except Exception:
            pass


class SessionBatch:
    """ekv_batch: B concurrent sessions over one shared AssembledContext, advanced in
    lock-step (BASELINE configs[2]).  Per session the result is collaborative_decode
    (cache_merge.cpp:230-273); weights and context are streamed once per step for all
    sessions (k_batch.cu)."""

    def __init__(self, model: EdgeModel, context: AssembledContext, sessions: int, max_rows: int):
        self.model, self.context, self.B, self.cap = model, context, sessions, max_rows
        hnd = C.c_void_p()
        call("ekv_batch_create", model.hnd, context.hnd, sessions, max_rows, C.byref(hnd))
        self.hnd = hnd

    def reset(self):
        call("ekv_batch_reset", self.hnd)

    def info(self):
        b = C.c_int(); r = C.c_int(); sp = (C.c_int * 3)()
        call("ekv_batch_info", self.hnd, C.byref(b), C.byref(r), sp)
        return {"sessions": b.value, "rows": r.value, "qkv_splitk": sp[0], "out_splitk": sp[1],
                "ctx_splits": sp[2]}

    def forward(self, emb: torch.Tensor) -> torch.Tensor:
        """n user rows of every session: device fp32 [B][n][h] -> outputs [n][B][h]."""
        emb = emb.contiguous().float()
        n = emb.shape[1]
        out = torch.empty((n, self.B, self.model.h), dtype=torch.float32, device=emb.device)
        _sync_in()
        call("ekv_batch_forward", self.hnd, _ptr(emb), n, _ptr(out))
        self.model.ctx.synchronize()
        return out

    def profile_row(self) -> np.ndarray:
        """One real forward row with CUDA-event times per kernel (ms), see ekv_capi.h."""
        n = 5 * self.model.L + 2
        out = np.zeros(n, dtype=np.float32)
        got = C.c_int()
        call("ekv_batch_profile_row", self.hnd, out.ctypes.data_as(C.POINTER(C.c_float)), n, C.byref(got))
        return out[:got.value]

    def decode(self, steps: int, out: torch.Tensor | None = None, sync: bool = True) -> torch.Tensor:
        if out is None:
            out = torch.empty((steps, self.B, self.model.h), dtype=torch.float32,
                              device=f"cuda:{self.model.ctx.device}")
        call("ekv_batch_decode", self.hnd, steps, _ptr(out))
        if sync:
            self.model.ctx.synchronize()
        return out

    def __del__(self):
        try:
            capi.load().ekv_batch_destroy(self.hnd)
        except Exception:
            pass


def collaborative_decode_batch(batch: SessionBatch, user_embeddings: np.ndarray, steps: int):
    """collaborative_decode of every session of the batch through the host-buffer C-ABI
    entry point: user_embeddings [B][U][h] -> (prefill [U][B][h], steps [steps][B][h])."""
    h, B = batch.model.h, batch.B
    ue = np.ascontiguousarray(np.asarray(user_embeddings, dtype=np.float32).reshape(B, -1, h))
    U = ue.shape[1]
    pre = np.zeros((max(U, 1), B, h), dtype=np.float32)
    st = np.zeros((max(steps, 1), B, h), dtype=np.float32)
    call("ekv_collaborative_decode_batch", batch.hnd, ue.ctypes.data_as(C.c_void_p), U, steps,
         pre.ctypes.data_as(C.c_void_p), st.ctypes.data_as(C.c_void_p))
    return pre[:U], st[:steps]


def collaborative_decode(session: Session, user_embeddings: np.ndarray, steps: int):
    """collaborative_decode (cache_merge.cpp:230-273) through the host-buffer C-ABI entry
    point.  Returns (prefill_outputs [U][h], step_outputs [steps][h]) as fp32 numpy."""
    h = session.model.h
    ue = np.ascontiguousarray(np.asarray(user_embeddings, dtype=np.float32).reshape(-1, h))
    U = ue.shape[0]
    pre = np.zeros((max(U, 1), h), dtype=np.float32)
    st = np.zeros((max(steps, 1), h), dtype=np.float32)
    call("ekv_collaborative_decode", session.hnd, ue.ctypes.data_as(C.c_void_p), U, steps,
         pre.ctypes.data_as(C.c_void_p), st.ctypes.data_as(C.c_void_p))
    return pre[:U], st[:steps]


def prefill(model: "EdgeModel", emb: torch.Tensor, want_x0: bool = False, want_kv: bool = False):
    """prefill (transformer.cpp:244-251) on the device: emb fp32 [n][h] (device) at positions
    0..n-1.  Returns (layer_outputs fp32 [L][n][h], x0 fp32 [n][h] | None,
    k bf16 [L][H][n][d] | None, v | None)."""
    emb = emb.contiguous().float()
    n = emb.shape[0]
    dev = emb.device
    lo = torch.empty((model.L, n, model.h), dtype=torch.float32, device=dev)
    x0 = torch.empty((n, model.h), dtype=torch.float32, device=dev) if want_x0 else None
    k = v = None
    if want_kv:
        k = torch.empty((model.L, model.H, n, model.d), dtype=torch.bfloat16, device=dev)
        v = torch.empty_like(k)
    _sync_in()
    call("ekv_prefill", model.hnd, _ptr(emb), n, _ptr(lo), _ptr(x0), _ptr(k), _ptr(v))
    return lo, x0, k, v


def deep_match(edge: "EdgeModel", cloud: "EdgeModel", edge_probe: torch.Tensor,
               cloud_probe: torch.Tensor, deep_layers: int, theta_cka: float, theta_rsa: float):
    """Artifacts::deep_match (sim.cpp:100-122) on the device: probe prefill of both models,
    K7 layer map, deep edge layer -> cloud layer.  Returns ({le: lc}, cka, rsa, best)."""
    ep = edge_probe.contiguous().float()
    cp = cloud_probe.contiguous().float()
    n = ep.shape[0]
    if cp.shape[0] != n:
        raise ValueError("deep_match: probe row-count mismatch")
    M, N = edge.L, cloud.L
    dm = np.zeros(max(deep_layers, 1), np.int32)
    cka = np.zeros((M, N)); rsa = np.zeros((M, N)); best = np.zeros(M, np.int32)
    _sync_in()
    call("ekv_deep_match", edge.hnd, cloud.hnd, _ptr(ep), _ptr(cp), n, deep_layers, theta_cka,
         theta_rsa, _ip(dm), _dp(cka), _dp(rsa), _ip(best))
    return {M - deep_layers + i: int(dm[i]) for i in range(deep_layers)}, cka, rsa, best


def prompt_context(edge: "EdgeModel", cloud: "EdgeModel", emb_edge: torch.Tensor,
                   emb_cloud: torch.Tensor | None, deep_map: dict, lam: float,
                   context: "AssembledContext"):
    """Artifacts::prompt + build_deep_kv + assembled_context (sim.cpp:124-138, 186-265) on
    the device: edge prefill of the S context rows -> local layers of `context`; cloud
    prefill -> hidden states + KV of the matched layers -> K1/K2 mask -> K3 codes into the
    deep layers [M - n, M).  deep_map {edge_layer: cloud_layer} covers exactly those layers.
    Returns (kept, cut_margin)."""
    M = edge.L
    les = sorted(deep_map)
    n = len(les)
    if les != list(range(M - n, M)):
        raise ValueError("prompt_context: the deep layers must be the last n edge layers")
    dm = np.asarray([deep_map[le] for le in les] or [0], np.int32)
    ee = emb_edge.contiguous().float()
    ec = emb_cloud.contiguous().float() if emb_cloud is not None else None
    kept = np.zeros(max(prune_retained(lam, cloud.d), 1), np.int32)
    margin = C.c_double(float("inf"))
    _sync_in()
    call("ekv_prompt_context", edge.hnd, cloud.hnd, _ptr(ee), _ptr(ec), n, _ip(dm), lam, context.hnd,
         _ip(kept), C.byref(margin))
    return kept[:prune_retained(lam, cloud.d)], margin.value


def build_deep_kv(ctx: Context, context: AssembledContext, deep_match: dict, X: torch.Tensor,
                  WqT: torch.Tensor, cloud_k, cloud_v, lam: float, cloud_layers: list,
                  x_index=None, wq_index=None, wq_stride: int = 0):
    """Artifacts::build_deep_kv (sim.cpp:217-265) through ekv_build_deep_kv: K1 channel
    scores (K column norms fused) over every distinct matched cloud layer, the reference
    ranking on the device and one batched K3 launch into the context's deep layers.

    deep_match: {edge_layer: cloud_layer}; cloud_layers: the distinct matched cloud layers
    (sorted) in the order of cloud_k / cloud_v (a [m][H][S][d_c] tensor or a list of m
    [H][S][d_c] tensors, bf16).  X: bf16 [m][S][h_c] (or, with x_index, any [*][S][h_c]
    stack), WqT: bf16 [m][H*d_c][h_c] (or with wq_index / wq_stride an ekv_model's weights).
    Returns (kept, cut_margin)."""
    m = len(cloud_layers)
    ks = [cloud_k[i] for i in range(m)]
    vs = [cloud_v[i] for i in range(m)]
    H, S, d_c = ks[0].shape
    for t in ks + vs:
        if t.dtype != torch.bfloat16 or tuple(t.shape) != (H, S, d_c) or not t.is_contiguous():
            raise ValueError("build_deep_kv: cloud K/V must be contiguous bf16 [H][S][d_c] per layer")
    if H != context.model.H:
        raise ValueError(f"assemble_context: head count mismatch (cloud {H}, edge {context.model.H})")
    if prune_retained(lam, d_c) != context.model.d:
        raise ValueError("assemble_context: dim mismatch; align with head pruning")
    if S != context.S:
        raise ValueError(f"assemble_context: dim mismatch (cloud context {S}, assembled {context.S})")
    le_list = sorted(deep_match)
    src = [cloud_layers.index(deep_match[le]) for le in le_list]
    kp = (C.c_void_p * m)(*[t.data_ptr() for t in ks])
    vp = (C.c_void_p * m)(*[t.data_ptr() for t in vs])
    xi = (C.c_int * m)(*(x_index if x_index is not None else range(m)))
    wi = (C.c_int * m)(*(wq_index if wq_index is not None else range(m)))
    cl = capi.ekv_cloud_kv(m, S, H, d_c, X.data_ptr(), 0, xi, WqT.data_ptr(), wq_stride, wi,
                           C.cast(kp, C.POINTER(C.c_void_p)), C.cast(vp, C.POINTER(C.c_void_p)))
    kept = np.zeros(prune_retained(lam, d_c), np.int32)
    margin = C.c_double()
    le_a = np.asarray(le_list, np.int32); src_a = np.asarray(src, np.int32)
    _sync_in()
    call("ekv_build_deep_kv", ctx.h, C.byref(cl), lam, context.hnd, len(le_list), _ip(le_a), _ip(src_a),
         _ip(kept), C.byref(margin))
    return kept, margin.value


def compress_batched(ctx: Context, n: int, src_ptrs, rows: int, d_c: int, kept_t: torch.Tensor,
                     d_e: int, bits: int, group: int, code_ptrs, scale_ptrs):
    """K3 over n (src, codes, scales) device-pointer triples in one launch."""
    _sync_in()
    call("ekv_kv_compress_batched", ctx.h, n, C.cast(src_ptrs, C.POINTER(C.c_void_p)), rows, d_c,
         _ptr(kept_t), d_e, bits, group, C.cast(code_ptrs, C.POINTER(C.c_void_p)),
         C.cast(scale_ptrs, C.POINTER(C.c_void_p)))

# ------------------------------------------------------------------ packed-KV wire format
def fnv1a64(data: bytes | np.ndarray, seed: int = 14695981039346656037) -> int:
    """The reference's fnv1a64 (rng.cpp:7-15) through the C ABI (host)."""
    buf = np.ascontiguousarray(np.frombuffer(bytes(data), np.uint8) if isinstance(data, (bytes, bytearray))
                               else data).view(np.uint8)
    out = C.c_uint64()
    call("ekv_fnv1a64", buf.ctypes.data_as(C.c_void_p), buf.nbytes, seed, C.byref(out))
    return out.value


def kvpack_size(n_layers: int, H: int, S: int, d_e: int, bits: int, group: int) -> int:
    out = C.c_size_t()
    call("ekv_kvpack_size", n_layers, H, S, d_e, bits, group, C.byref(out))
    return out.value


def kvpack_export(context: "AssembledContext", layers, cloud_layers, kept, d_c: int,
                  out: torch.Tensor | None = None) -> torch.Tensor:
    """The compressed `layers` of the context as one EKVPACK1 byte stream (pinned host uint8;
    `out` reuses a buffer of at least kvpack_size bytes)."""
    seg = context.segment(int(layers[0]))
    m = context.model
    n = len(layers)
    size = kvpack_size(n, m.H, seg.S, m.d, seg.format, seg.group)
    buf = out if out is not None else torch.empty(size, dtype=torch.uint8).pin_memory()
    if buf.numel() < size:
        raise ValueError("kvpack_export: buffer too small")
    ly = np.ascontiguousarray(layers, np.int32); cl = np.ascontiguousarray(cloud_layers, np.int32)
    kp = np.ascontiguousarray(kept, np.int32)
    call("ekv_kvpack_export", context.hnd, _ip(ly), _ip(cl), n, _ip(kp), d_c, C.c_void_p(buf.data_ptr()), size)
    return buf[:size]


def kvpack_layer_uploads(buf: torch.Tensor, L: int) -> dict:
    """Per-layer host sources of a validated pack for Session.forward_pipelined: {edge layer:
    (k codes, v codes, k scales, v scales)} as views into the pack's payload."""
    info = kvpack_parse(buf)
    H, S, de, bits, g = info["H"], info["S"], info["d_e"], info["bits"], info["group"]
    rows = H * S
    cb, sb = rows * de * bits // 8, rows * (de // g) * 4
    lb = 2 * cb + 2 * sb
    hb = info["bytes"] - info["n_layers"] * lb
    ups = {}
    for i, l in enumerate(info["layers"]):
        p = hb + i * lb
        ups[l] = (buf[p:p + cb], buf[p + cb:p + 2 * cb], buf[p + 2 * cb:p + 2 * cb + sb].view(torch.float32),
                  buf[p + 2 * cb + sb:p + lb].view(torch.float32))
    return ups


def kvpack_parse(buf) -> dict:
    """Validate a pack (host) and return its description."""
    a = np.ascontiguousarray(buf.numpy() if isinstance(buf, torch.Tensor) else buf).view(np.uint8)
    info = capi.ekv_kvpack_info()
    call("ekv_kvpack_parse", a.ctypes.data_as(C.c_void_p), a.nbytes, C.byref(info), None, None, None)
    n, de = info.n_layers, info.d_e
    ly = np.zeros(n, np.int32); cl = np.zeros(n, np.int32); kp = np.zeros(de, np.int32)
    call("ekv_kvpack_parse", a.ctypes.data_as(C.c_void_p), a.nbytes, C.byref(info), _ip(ly), _ip(cl), _ip(kp))
    return {"n_layers": n, "H": info.H, "S": info.S, "d_e": de, "d_c": info.d_c, "bits": info.bits,
            "group": info.group, "bytes": info.bytes, "layers": ly.tolist(), "cloud_layers": cl.tolist(),
            "kept": kp.tolist()}


def kvpack_import(context: "AssembledContext", buf) -> None:
    a = buf if isinstance(buf, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(buf))
    call("ekv_kvpack_import", context.hnd, C.c_void_p(a.data_ptr()), a.numel())
