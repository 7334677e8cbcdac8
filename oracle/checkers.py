"""TEST INFRASTRUCTURE ONLY -- ctypes front-ends of the two CPU checkers.

* ``Oracle`` wraps ``oracle/lib/libekv_oracle.so``: the plain-C restatement of
  the reference hot path (``oracle/ekv_oracle.c``, every function cites the
  reference file:line it restates) plus the quantiser contract that has no
  reference (parity unpinned vs reference).
* ``Reference`` wraps ``oracle/_ref/libedgekv_refc.so``: the UNMODIFIED
  reference sources compiled by ``oracle/Makefile`` (target ``ref``) plus the
  thin extern "C" shim ``oracle/ref_capi.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "lib", "libekv_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libedgekv_refc.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_fp = C.POINTER(C.c_float)
_u8p = C.POINTER(C.c_uint8)
_u16p = C.POINTER(C.c_uint16)
_u64p = C.POINTER(C.c_uint64)


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def build(ref: bool = False) -> None:
    """Compile the checkers (``make -C oracle [ref]``)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "-j8", "ref"], check=True)


def bf16_to_f64(u16: np.ndarray) -> np.ndarray:
    """Exact widening of raw bf16 bits (uint16) to float64."""
    return (np.asarray(u16, dtype=np.uint32) << 16).view(np.float32).astype(np.float64)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 raw bits (numpy, vectorised)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    r[nan] = 0x7FC0
    return r


class Oracle:
    """The C restatement (oracle/ekv_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.ekvo_mix.restype = C.c_uint64
        L.ekvo_mix.argtypes = [C.c_uint64, C.c_uint64]
        L.ekvo_fnv1a64.restype = C.c_uint64
        L.ekvo_fnv1a64.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
        L.ekvo_mt64_stream.argtypes = [C.c_uint64, C.c_int64, _u64p]
        L.ekvo_generate_embeddings.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp]
        L.ekvo_init_model.restype = C.c_uint64
        L.ekvo_init_model.argtypes = [C.c_int] * 4 + [C.c_uint64] + [_dp] * 5
        L.ekvo_fill_uniform_bf16.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_double,
                                             C.c_double, _u16p]
        L.ekvo_f32_to_bf16.restype = C.c_uint16
        L.ekvo_f32_to_bf16.argtypes = [C.c_float]
        L.ekvo_prune_retained.restype = C.c_int
        L.ekvo_prune_retained.argtypes = [C.c_double, C.c_int]
        L.ekvo_colsq.argtypes = [_dp, C.c_int64, C.c_int, _dp]
        L.ekvo_select_channels.argtypes = [_dp, C.c_int64, _dp, C.c_int64, C.c_int, C.c_int,
                                           _ip, _dp]
        L.ekvo_rank_channels.argtypes = [_dp, _dp, C.c_int, C.c_int, _ip]
        L.ekvo_prune_rows_f64.argtypes = [_dp, C.c_int64, C.c_int, _ip, C.c_int, _dp]
        L.ekvo_prune_rows_bf16.argtypes = [_u16p, C.c_int64, C.c_int, _ip, C.c_int, _u16p]
        L.ekvo_kv_compress.argtypes = [_u16p, C.c_int64, C.c_int, _ip, C.c_int, C.c_int, C.c_int,
                                       _u8p, _fp]
        L.ekvo_kv_dequant_bf16.argtypes = [_u8p, _fp, C.c_int64, C.c_int, C.c_int, C.c_int, _u16p]
        L.ekvo_kv_dequant_f64.argtypes = [_u8p, _fp, C.c_int64, C.c_int, C.c_int, C.c_int, _dp]
        L.ekvo_segment_attention.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_int, _dp, _dp,
                                             _dp]
        L.ekvo_merge_attention.restype = C.c_int
        L.ekvo_merge_attention.argtypes = [_dp, C.c_double, C.c_double, _dp, C.c_double,
                                           C.c_double, C.c_int, _dp, _dp, _dp]
        L.ekvo_collaborative_decode.restype = C.c_int
        L.ekvo_collaborative_decode.argtypes = ([C.c_int] * 4 + [_dp] * 5 + [C.c_int, _dp, _dp,
                                                _dp, C.c_int, C.c_int, _dp, C.c_int, _dp, _dp])
        L.ekvo_prefill.argtypes = [C.c_int] * 4 + [_dp] * 6 + [C.c_int, _dp, _dp, _dp]
        L.ekvo_prefill_ex.argtypes = [C.c_int] * 4 + [_dp] * 6 + [C.c_int, C.c_int, _dp, _dp, _dp]
        L.ekvo_align_qnorm.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, _dp]
        L.ekvo_cka.restype = C.c_int
        L.ekvo_cka.argtypes = [_dp, C.c_int, _dp, C.c_int, C.c_int, _dp]
        L.ekvo_rsa.restype = C.c_int
        L.ekvo_rsa.argtypes = [_dp, C.c_int, _dp, C.c_int, C.c_int, _dp]
        L.ekvo_match_layers.restype = C.c_int
        L.ekvo_match_layers.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_int,
                                        C.c_double, C.c_double, _dp, _dp, _ip]
        L.ekvo_cache_source.restype = C.c_int
        L.ekvo_cache_source.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_int]
        L.ekvo_pipeline_schedule.restype = C.c_int
        L.ekvo_pipeline_schedule.argtypes = [_dp, _dp, C.c_int, _dp, _dp, _dp]

    # --- rng ---------------------------------------------------------------
    def mix(self, a, b):
        return int(self.lib.ekvo_mix(a, b))

    def mt64_stream(self, seed, n):
        out = np.zeros(n, dtype=np.uint64)
        self.lib.ekvo_mt64_stream(seed, n, out.ctypes.data_as(_u64p))
        return out

    def generate_embeddings(self, seed, n, h):
        out = np.zeros((n, h))
        self.lib.ekvo_generate_embeddings(seed, n, h, _d(out))
        return out

    def init_model(self, L, H, d, max_pos, seed):
        h = H * d
        wq = np.zeros((L, H, h, d)); wk = np.zeros_like(wq); wv = np.zeros_like(wq)
        out = np.zeros((L, h, h)); pos = np.zeros((max_pos, h))
        ck = self.lib.ekvo_init_model(L, H, d, max_pos, seed, _d(wq), _d(wk), _d(wv), _d(out),
                                      _d(pos))
        return dict(wq=wq, wk=wk, wv=wv, out_proj=out, pos=pos, checksum=int(ck))

    def fill_uniform_bf16(self, seed, stream, n, lo, hi):
        out = np.zeros(n, dtype=np.uint16)
        self.lib.ekvo_fill_uniform_bf16(seed, stream, n, lo, hi, out.ctypes.data_as(_u16p))
        return out

    # --- alignment / projection -------------------------------------------
    def prune_retained(self, lam, d):
        return int(self.lib.ekvo_prune_retained(lam, d))

    def select_channels(self, q, k, retained):
        q = _f64(q); k = _f64(k)
        d = q.shape[1]
        kept = np.zeros(max(retained, 1), dtype=np.int32)
        score = np.zeros(d)
        self.lib.ekvo_select_channels(_d(q), q.shape[0], _d(k), k.shape[0], d, retained,
                                      _i(kept), _d(score))
        return kept[:retained].copy(), score

    def rank_channels(self, qsq, ksq, retained):
        qsq = _f64(qsq); ksq = _f64(ksq)
        kept = np.zeros(max(retained, 1), dtype=np.int32)
        self.lib.ekvo_rank_channels(_d(qsq), _d(ksq), len(qsq), retained, _i(kept))
        return kept[:retained].copy()

    def colsq(self, m):
        m = _f64(m)
        out = np.zeros(m.shape[1])
        self.lib.ekvo_colsq(_d(m), m.shape[0], m.shape[1], _d(out))
        return out

    def align_qnorm(self, X, wqT):
        X = _f64(X); wqT = _f64(wqT)
        out = np.zeros(wqT.shape[0])
        self.lib.ekvo_align_qnorm(_d(X), X.shape[0], X.shape[1], _d(wqT), wqT.shape[0], _d(out))
        return out

    def prune_rows_bf16(self, src_u16, kept):
        src = np.ascontiguousarray(src_u16, dtype=np.uint16)
        rows, d_c = src.shape
        kept = np.ascontiguousarray(kept, dtype=np.int32)
        dst = np.zeros((rows, len(kept)), dtype=np.uint16)
        self.lib.ekvo_prune_rows_bf16(src.ctypes.data_as(_u16p), rows, d_c, _i(kept), len(kept),
                                      dst.ctypes.data_as(_u16p))
        return dst

    # --- quantiser (own contract; parity unpinned vs reference) -------------
    def kv_compress(self, src_u16, kept, bits, group):
        src = np.ascontiguousarray(src_u16, dtype=np.uint16)
        rows, d_c = src.shape
        kept = np.ascontiguousarray(kept, dtype=np.int32)
        d_e = len(kept)
        codes = np.zeros((rows, d_e * bits // 8), dtype=np.uint8)
        scales = np.zeros((rows, d_e // group), dtype=np.float32)
        self.lib.ekvo_kv_compress(src.ctypes.data_as(_u16p), rows, d_c, _i(kept), d_e, bits, group,
                                  codes.ctypes.data_as(_u8p), scales.ctypes.data_as(_fp))
        return codes, scales

    def kv_dequant_bf16(self, codes, scales, d_e, bits, group):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        scales = np.ascontiguousarray(scales, dtype=np.float32)
        rows = codes.shape[0]
        dst = np.zeros((rows, d_e), dtype=np.uint16)
        self.lib.ekvo_kv_dequant_bf16(codes.ctypes.data_as(_u8p), scales.ctypes.data_as(_fp), rows,
                                      d_e, bits, group, dst.ctypes.data_as(_u16p))
        return dst

    def kv_dequant_f64(self, codes, scales, d_e, bits, group):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        scales = np.ascontiguousarray(scales, dtype=np.float32)
        rows = codes.shape[0]
        dst = np.zeros((rows, d_e))
        self.lib.ekvo_kv_dequant_f64(codes.ctypes.data_as(_u8p), scales.ctypes.data_as(_fp), rows,
                                     d_e, bits, group, _d(dst))
        return dst

    # --- decode attention ----------------------------------------------------
    def segment_attention(self, q, k, v, visible=None):
        q = _f64(q); k = _f64(k); v = _f64(v)
        vis = k.shape[0] if visible is None else visible
        o = np.zeros(v.shape[1]); s = C.c_double(); sh = C.c_double()
        self.lib.ekvo_segment_attention(_d(q), _d(k), _d(v), vis, k.shape[1], v.shape[1], _d(o),
                                        C.byref(s), C.byref(sh))
        return o, s.value, sh.value

    def merge_attention(self, ctx, user):
        (oc, sc, hc), (ou, su, hu) = ctx, user
        oc = _f64(oc); ou = _f64(ou)
        o = np.zeros(len(oc)); ac = C.c_double(); au = C.c_double()
        rc = self.lib.ekvo_merge_attention(_d(oc), sc, hc, _d(ou), su, hu, len(oc), _d(o),
                                           C.byref(ac), C.byref(au))
        if rc:
            raise ValueError("merge_attention: non-positive or non-finite sigma")
        return o, ac.value, au.value

    def collaborative_decode(self, model, ctx_k, ctx_v, user_emb, steps, teacher=None,
                             user_kv_bf16=False):
        """model: dict(L,H,d,max_pos,wqkvT,woT,gamma,bias,pos) in the B200 layout;
        ctx_k/ctx_v [L][H][S][d] (S may be 0)."""
        L, H, d, mp = model["L"], model["H"], model["d"], model["max_pos"]
        h = H * d
        W = _f64(model["wqkvT"]); Wo = _f64(model["woT"])
        g = _f64(model["gamma"]); b = _f64(model["bias"]); p = _f64(model["pos"])
        S = 0 if ctx_k is None else ctx_k.shape[2]
        ck = _f64(ctx_k) if S else np.zeros(1)
        cv = _f64(ctx_v) if S else np.zeros(1)
        ue = _f64(user_emb).reshape(-1, h) if user_emb is not None else np.zeros((0, h))
        U = ue.shape[0]
        pre = np.zeros((max(U, 1), h)); st = np.zeros((steps, h))
        tp = _d(_f64(teacher)) if teacher is not None else None
        keep = teacher
        rc = self.lib.ekvo_collaborative_decode(L, H, d, mp, _d(W), _d(Wo), _d(g), _d(b), _d(p), S,
                                                _d(ck), _d(cv), _d(ue), U, steps, tp,
                                                int(user_kv_bf16), _d(pre), _d(st))
        del keep
        if rc == -2:
            raise ValueError("position overflow")
        if rc:
            raise ValueError("collaborative_decode: steps must be >= 1")
        return pre[:U], st

    def prefill(self, model, emb, kv_bf16=False):
        """prefill (forward_rows over an empty cache); kv_bf16 rounds the cached K/V rows
        to bf16 as the B200 prefill stores them."""
        L, H, d, mp = model["L"], model["H"], model["d"], model["max_pos"]
        h = H * d
        emb = _f64(emb)
        n = emb.shape[0]
        lo = np.zeros((L, n, h)); ko = np.zeros((L, H, n, d)); vo = np.zeros((L, H, n, d))
        self.lib.ekvo_prefill_ex(L, H, d, mp, _d(_f64(model["wqkvT"])), _d(_f64(model["woT"])),
                                 _d(_f64(model["gamma"])), _d(_f64(model["bias"])),
                                 _d(_f64(model["pos"])), _d(emb), n, int(kv_bf16), _d(lo), _d(ko),
                                 _d(vo))
        return lo, ko, vo

    # --- layer matching ------------------------------------------------------
    def cka(self, oe, oc):
        oe = _f64(oe); oc = _f64(oc)
        out = C.c_double()
        if self.lib.ekvo_cka(_d(oe), oe.shape[1], _d(oc), oc.shape[1], oe.shape[0], C.byref(out)):
            raise ValueError("cka: degenerate representation")
        return out.value

    def rsa(self, oe, oc):
        oe = _f64(oe); oc = _f64(oc)
        out = C.c_double()
        rc = self.lib.ekvo_rsa(_d(oe), oe.shape[1], _d(oc), oc.shape[1], oe.shape[0], C.byref(out))
        if rc == -1:
            raise ValueError("pearson_corr: zero variance")
        if rc < -1:
            raise ValueError(f"rsa: zero-norm row {-rc - 2}")
        return out.value

    def match_layers(self, edge_outs, cloud_outs, theta_cka, theta_rsa):
        e = _f64(edge_outs); c = _f64(cloud_outs)
        me, n, ce = e.shape
        nc, _, cc = c.shape
        cka = np.zeros((me, nc)); rsa = np.zeros((me, nc)); best = np.zeros(me, dtype=np.int32)
        rc = self.lib.ekvo_match_layers(_d(e), me, ce, _d(c), nc, cc, n, theta_cka, theta_rsa,
                                        _d(cka), _d(rsa), _i(best))
        if rc:
            raise ValueError(f"match_layers failed ({rc})")
        return cka, rsa, best

    # --- scheduler interface -------------------------------------------------
    def cache_source(self, layer, cost_local, cost_peer, boundary, m):
        return int(self.lib.ekvo_cache_source(layer, cost_local, cost_peer, boundary, m))

    def pipeline_schedule(self, t_comm, t_comp):
        a = _f64(t_comm); b = _f64(t_comp)
        pip = np.zeros(len(a)); s = C.c_double(); p = C.c_double()
        if self.lib.ekvo_pipeline_schedule(_d(a), _d(b), len(a), _d(pip), C.byref(s), C.byref(p)):
            raise ValueError("pipeline_schedule: invalid input")
        return pip, s.value, p.value


class RefError(RuntimeError):
    pass


class Reference:
    """The unmodified reference library (oracle/_ref/libedgekv_refc.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference is mounted")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_mix.restype = C.c_uint64
        L.ref_mix.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_mt64_stream.argtypes = [C.c_uint64, C.c_int64, _u64p]
        L.ref_init_model.argtypes = [C.c_int] * 4 + [C.c_uint64] + [_dp] * 5 + [_u64p]
        L.ref_generate_embeddings.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp]
        L.ref_prune_retained.argtypes = [C.c_double, C.c_int]
        L.ref_select_channels.argtypes = [_dp, C.c_int64, _dp, C.c_int64, C.c_int, C.c_double, _ip]
        L.ref_prune_objective.restype = C.c_double
        L.ref_prune_objective.argtypes = [_dp, C.c_int64, _dp, C.c_int64, C.c_int, _ip, C.c_int]
        L.ref_prune_cache.argtypes = [C.c_int] * 4 + [_dp, _dp, _ip, C.c_int, _dp, _dp]
        L.ref_segment_attention.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        L.ref_merge_attention.argtypes = [_dp, C.c_double, C.c_double, _dp, C.c_double, C.c_double,
                                          C.c_int, _dp, _dp, _dp]
        L.ref_collaborative_decode.argtypes = ([C.c_int] * 4 + [_dp] * 5 + [C.c_int, _dp, _dp,
                                               C.c_int, _dp, C.c_int, C.c_int, _dp, _dp])
        L.ref_prefill.argtypes = [C.c_int] * 4 + [_dp] * 6 + [C.c_int, _dp, _dp, _dp]
        L.ref_cka.argtypes = [_dp, C.c_int, _dp, C.c_int, C.c_int, _dp]
        L.ref_rsa.argtypes = [_dp, C.c_int, _dp, C.c_int, C.c_int, _dp]
        L.ref_match_layers.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_int,
                                       C.c_double, C.c_double, _dp, _dp, _ip]
        L.ref_cache_source.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_int]
        L.ref_pipeline_schedule.argtypes = [_dp, _dp, C.c_int, _dp, _dp, _dp]
        L.ref_bench_setup.restype = C.c_void_p
        L.ref_bench_setup.argtypes = [C.c_int] * 6 + [C.c_uint64]
        L.ref_bench_run.argtypes = [C.c_void_p] + [C.c_int] * 4 + [_dp, C.POINTER(C.c_int64)]
        L.ref_bench_free.argtypes = [C.c_void_p]
        L.ref_full_path.argtypes = ([C.c_int] * 7 + [_dp] * 10 + [C.c_uint64, C.c_int, C.c_double,
                                    C.c_double, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                    _dp, C.POINTER(C.c_int), C.POINTER(C.c_int), _dp])

    def _chk(self, rc):
        if rc < 0:
            raise RefError(self.lib.ref_last_error().decode())
        return rc

    def mix(self, a, b):
        return int(self.lib.ref_mix(a, b))

    def mt64_stream(self, seed, n):
        out = np.zeros(n, dtype=np.uint64)
        self.lib.ref_mt64_stream(seed, n, out.ctypes.data_as(_u64p))
        return out

    def init_model(self, L, H, d, max_pos, seed):
        h = H * d
        wq = np.zeros((L, H, h, d)); wk = np.zeros_like(wq); wv = np.zeros_like(wq)
        out = np.zeros((L, h, h)); pos = np.zeros((max_pos, h)); ck = C.c_uint64()
        self._chk(self.lib.ref_init_model(L, H, d, max_pos, seed, _d(wq), _d(wk), _d(wv), _d(out),
                                          _d(pos), C.byref(ck)))
        return dict(wq=wq, wk=wk, wv=wv, out_proj=out, pos=pos, checksum=int(ck.value))

    def generate_embeddings(self, seed, n, h):
        out = np.zeros((n, h))
        self._chk(self.lib.ref_generate_embeddings(seed, n, h, _d(out)))
        return out

    def prune_retained(self, lam, d):
        return self._chk(self.lib.ref_prune_retained(lam, d))

    def select_channels(self, q, k, lam):
        q = _f64(q); k = _f64(k)
        kept = np.zeros(q.shape[1], dtype=np.int32)
        n = self._chk(self.lib.ref_select_channels(_d(q), q.shape[0], _d(k), k.shape[0],
                                                   q.shape[1], lam, _i(kept)))
        return kept[:n].copy()

    def prune_objective(self, q, k, kept):
        q = _f64(q); k = _f64(k); kept = np.ascontiguousarray(kept, dtype=np.int32)
        return self.lib.ref_prune_objective(_d(q), q.shape[0], _d(k), k.shape[0], q.shape[1],
                                            _i(kept), len(kept))

    def prune_cache(self, keys, values, kept):
        keys = _f64(keys); values = _f64(values); kept = np.ascontiguousarray(kept, dtype=np.int32)
        L, H, S, dc = keys.shape
        ok = np.zeros((L, H, S, len(kept))); ov = np.zeros_like(ok)
        self._chk(self.lib.ref_prune_cache(L, H, S, dc, _d(keys), _d(values), _i(kept), len(kept),
                                           _d(ok), _d(ov)))
        return ok, ov

    def segment_attention(self, q, k, v):
        q = _f64(q); k = _f64(k); v = _f64(v)
        o = np.zeros(v.shape[1]); s = C.c_double(); sh = C.c_double()
        self._chk(self.lib.ref_segment_attention(_d(q), _d(k), _d(v), k.shape[0], k.shape[1],
                                                 v.shape[1], _d(o), C.byref(s), C.byref(sh)))
        return o, s.value, sh.value

    def merge_attention(self, ctx, user):
        (oc, sc, hc), (ou, su, hu) = ctx, user
        oc = _f64(oc); ou = _f64(ou)
        o = np.zeros(len(oc)); ac = C.c_double(); au = C.c_double()
        self._chk(self.lib.ref_merge_attention(_d(oc), sc, hc, _d(ou), su, hu, len(oc), _d(o),
                                               C.byref(ac), C.byref(au)))
        return o, ac.value, au.value

    def collaborative_decode(self, model, ctx_k, ctx_v, user_emb, steps, boundary=None):
        L, H, d, mp = model["L"], model["H"], model["d"], model["max_pos"]
        h = H * d
        S = 0 if ctx_k is None else ctx_k.shape[2]
        ck = _f64(ctx_k) if S else np.zeros(1)
        cv = _f64(ctx_v) if S else np.zeros(1)
        ue = _f64(user_emb).reshape(-1, h)
        U = ue.shape[0]
        pre = np.zeros((max(U, 1), h)); st = np.zeros((steps, h))
        b = L // 2 if boundary is None else boundary
        self._chk(self.lib.ref_collaborative_decode(
            L, H, d, mp, _d(_f64(model["wqkvT"])), _d(_f64(model["woT"])),
            _d(_f64(model["gamma"])), _d(_f64(model["bias"])), _d(_f64(model["pos"])), S, _d(ck),
            _d(cv), b, _d(ue), U, steps, _d(pre), _d(st)))
        return pre[:U], st

    def prefill(self, model, emb):
        L, H, d, mp = model["L"], model["H"], model["d"], model["max_pos"]
        h = H * d
        emb = _f64(emb)
        n = emb.shape[0]
        lo = np.zeros((L, n, h)); ko = np.zeros((L, H, n, d)); vo = np.zeros((L, H, n, d))
        self._chk(self.lib.ref_prefill(L, H, d, mp, _d(_f64(model["wqkvT"])),
                                       _d(_f64(model["woT"])), _d(_f64(model["gamma"])),
                                       _d(_f64(model["bias"])), _d(_f64(model["pos"])), _d(emb), n,
                                       _d(lo), _d(ko), _d(vo)))
        return lo, ko, vo

    def cka(self, oe, oc):
        oe = _f64(oe); oc = _f64(oc); out = C.c_double()
        self._chk(self.lib.ref_cka(_d(oe), oe.shape[1], _d(oc), oc.shape[1], oe.shape[0],
                                   C.byref(out)))
        return out.value

    def rsa(self, oe, oc):
        oe = _f64(oe); oc = _f64(oc); out = C.c_double()
        self._chk(self.lib.ref_rsa(_d(oe), oe.shape[1], _d(oc), oc.shape[1], oe.shape[0],
                                   C.byref(out)))
        return out.value

    def match_layers(self, edge_outs, cloud_outs, theta_cka, theta_rsa):
        e = _f64(edge_outs); c = _f64(cloud_outs)
        me, n, ce = e.shape
        nc, _, cc = c.shape
        cka = np.zeros((me, nc)); rsa = np.zeros((me, nc)); best = np.zeros(me, dtype=np.int32)
        self._chk(self.lib.ref_match_layers(_d(e), me, ce, _d(c), nc, cc, n, theta_cka, theta_rsa,
                                            _d(cka), _d(rsa), _i(best)))
        return cka, rsa, best

    def cache_source(self, layer, cost_local, cost_peer, boundary, m):
        return self._chk(self.lib.ref_cache_source(layer, cost_local, cost_peer, boundary, m))

    def pipeline_schedule(self, t_comm, t_comp):
        a = _f64(t_comm); b = _f64(t_comp)
        pip = np.zeros(len(a)); s = C.c_double(); p = C.c_double()
        self._chk(self.lib.ref_pipeline_schedule(_d(a), _d(b), len(a), _d(pip), C.byref(s),
                                                 C.byref(p)))
        return pip, s.value, p.value

    def bench_setup(self, L, H, d, S, boundary, max_pos, seed=42):
        h = self.lib.ref_bench_setup(L, H, d, S, boundary, max_pos, seed)
        if not h:
            raise RefError(self.lib.ref_last_error().decode())
        return h

    def bench_run(self, handle, U, steps, threads, calls):
        s = C.c_double(); n = C.c_int64()
        self._chk(self.lib.ref_bench_run(handle, U, steps, threads, calls, C.byref(s), C.byref(n)))
        return s.value, n.value

    def bench_free(self, handle):
        self.lib.ref_bench_free(handle)

    def full_path(self, edge, cloud, seed, n_probe, theta_cka, theta_rsa, S, deep, lam, U, steps):
        """The reference's whole value path for one request (Artifacts order, sim.cpp:100-265):
        edge / cloud = dict(L,H,d,max_pos,wqkvT,woT,gamma,bias,pos) in the B200 layout (fp64).
        Returns (stage seconds [8], kept, deep_map, step_outputs [steps][h_e])."""
        assert edge["max_pos"] == cloud["max_pos"]
        times = np.zeros(8)
        kept = np.zeros(cloud["d"], np.int32)
        dm = np.zeros(max(deep, 1), np.int32)
        out = np.zeros((steps, edge["H"] * edge["d"]))
        f = lambda m, k: _d(_f64(m[k]))
        keep = [_f64(m[k]) for m in (edge, cloud) for k in ("wqkvT", "woT", "gamma", "bias", "pos")]
        args = [edge["L"], edge["H"], edge["d"], cloud["L"], cloud["H"], cloud["d"], edge["max_pos"]]
        args += [_d(a) for a in keep]
        self._chk(self.lib.ref_full_path(*args, seed, n_probe, theta_cka, theta_rsa, S, deep, lam, U,
                                         steps, _d(times), kept.ctypes.data_as(C.POINTER(C.c_int)),
                                         dm.ctypes.data_as(C.POINTER(C.c_int)), _d(out)))
        del f
        return times, kept, dm[:deep], out


def model_from_reference_layout(ref_model: dict, L: int, H: int, d: int, max_pos: int) -> dict:
    """Translate init_model's per-head layout into the B200 layout (DESIGN.md s.2)."""
    h = H * d
    wq, wk, wv = ref_model["wq"], ref_model["wk"], ref_model["wv"]  # [L][H][h][d]
    wqkvT = np.zeros((L, 3 * h, h))
    for part, w in enumerate((wq, wk, wv)):
        # row part*h + hd*d + c, column k  == w[l][hd][k][c]
        wqkvT[:, part * h:(part + 1) * h, :] = w.transpose(0, 1, 3, 2).reshape(L, h, h)
    woT = ref_model["out_proj"].transpose(0, 2, 1).copy()
    return dict(L=L, H=H, d=d, max_pos=max_pos, wqkvT=wqkvT, woT=woT, gamma=np.ones(h),
                bias=np.zeros(h), pos=ref_model["pos"])
