"""ctypes binding of the C ABI (include/ekv_capi.h) in libekv.so.

This is plumbing for the Python host layer, tests and bench: every call goes
straight to the sm_100a library.  There is no fallback -- if libekv.so is
missing or the device is not a B200, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIBEKV = os.path.join(PKG, "lib", "libekv.so")

EKV_OK = 0
EKV_KV_BF16, EKV_KV_INT8, EKV_KV_INT4 = 16, 8, 4
_STATUS = {-1: "EINVAL", -2: "ECUDA", -3: "ENOMEM", -4: "ENODEV", -5: "EUNSUPPORTED"}


class EkvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{_STATUS.get(status, status)}] {msg}")
        self.status = status
        self.msg = msg


class ekv_segment(C.Structure):
    _fields_ = [("format", C.c_int), ("S", C.c_int), ("group", C.c_int), ("k", C.c_void_p),
                ("v", C.c_void_p), ("k_scales", C.c_void_p), ("v_scales", C.c_void_p)]


class ekv_kvpack_info(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("H", C.c_int), ("S", C.c_int), ("d_e", C.c_int), ("d_c", C.c_int),
                ("bits", C.c_int), ("group", C.c_int), ("bytes", C.c_size_t)]


class ekv_cloud_kv(C.Structure):
    _fields_ = [("m", C.c_int), ("S", C.c_int), ("H", C.c_int), ("d_c", C.c_int),
                ("x", C.c_void_p), ("x_stride", C.c_int64), ("x_index", C.POINTER(C.c_int)),
                ("wq", C.c_void_p), ("wq_stride", C.c_int64), ("wq_index", C.POINTER(C.c_int)),
                ("k", C.POINTER(C.c_void_p)), ("v", C.POINTER(C.c_void_p))]


class ekv_model_config(C.Structure):
    _fields_ = [("num_layers", C.c_int), ("num_heads", C.c_int), ("head_dim", C.c_int),
                ("max_positions", C.c_int)]


_vp, _i, _i64, _u64, _d = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double
_dp, _ip, _fp = C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_float)
_pp = C.POINTER(C.c_void_p)

# name -> argtypes (all return int status unless listed in _RET)
PROTOS = {
    "ekv_abi_version": [],
    "ekv_last_error": [],
    "ekv_ctx_create": [_i, _vp, _pp],
    "ekv_ctx_destroy": [_vp],
    "ekv_ctx_stream": [_vp, _pp],
    "ekv_ctx_synchronize": [_vp],
    "ekv_ctx_kernel_launches": [_vp, C.POINTER(C.c_int64)],
    "ekv_device_alloc": [_vp, C.c_size_t, _pp],
    "ekv_device_free": [_vp, _vp],
    "ekv_memset": [_vp, _vp, _i, C.c_size_t],
    "ekv_copy": [_vp, _vp, _vp, C.c_size_t, _i],
    "ekv_fill_uniform_bf16": [_vp, _vp, _i64, _u64, _u64, _d, _d],
    "ekv_prune_retained": [_d, _i, _ip],
    "ekv_generate_embeddings": [_u64, _i, _i, _dp],
    "ekv_align_qnorm": [_vp, _vp, _vp, _i, _i, _i, _i, _vp],
    "ekv_kv_colnorm": [_vp, _vp, _i64, _i, _vp],
    "ekv_rank_channels": [_dp, _dp, _i, _i, _ip, _dp],
    "ekv_match_layers": [_vp, _dp, _i, _i, _dp, _i, _i, _i, _d, _d, _dp, _dp, _ip],
    "ekv_colsq_f64": [_vp, _vp, _i64, _i, _vp],
    "ekv_prefill": [_vp, _vp, _i, _vp, _vp, _vp, _vp],
    "ekv_deep_match": [_vp, _vp, _vp, _vp, _i, _i, _d, _d, _ip, _dp, _dp, _ip],
    "ekv_align_select": [_vp, C.POINTER(ekv_cloud_kv), _d, _ip, _dp],
    "ekv_build_deep_kv": [_vp, C.POINTER(ekv_cloud_kv), _d, _vp, _i, _ip, _ip, _ip, _dp],
    "ekv_kv_dequant_f64": [_vp, _vp, _vp, _i64, _i, _i, _i, _vp],
    "ekv_prompt_context": [_vp, _vp, _vp, _vp, _i, _ip, _d, _vp, _ip, _dp],
    "ekv_forward_rows": [_vp, _vp, _vp, _i, _vp, _vp, _vp, _vp],
    "ekv_matmul_f64": [_vp, _vp, _vp, _i, _i, _i, _vp],
    "ekv_segment_attention_f64": [_vp, _vp, _vp, _vp, _i, _i, _i, _vp, _dp, _dp],
    "ekv_convert_f32_bf16": [_vp, _vp, _vp, _i64],
    "ekv_match_layers_dev": [_vp, _vp, _i, _i, _vp, _i, _i, _i, _d, _d, _dp, _dp, _ip],
    "ekv_kv_gather": [_vp, _vp, _i64, _i, _vp, _i, _vp],
    "ekv_gather_columns": [_vp, _vp, _i64, _i, _vp, _i, _i, _vp],
    "ekv_kv_compress": [_vp, _vp, _i64, _i, _vp, _i, _i, _i, _vp, _vp],
    "ekv_kv_compress_batched": [_vp, _i, _pp, _i64, _i, _vp, _i, _i, _i, _pp, _pp],
    "ekv_kv_dequant": [_vp, _vp, _vp, _i64, _i, _i, _i, _vp],
    "ekv_decode_attention": [_vp, _i, _i, _i, _vp, C.POINTER(ekv_segment), _vp, _vp, _i, _i, _vp,
                             _vp],
    "ekv_model_create": [_vp, C.POINTER(ekv_model_config), _pp],
    "ekv_model_destroy": [_vp],
    "ekv_model_set_layer": [_vp, _i, _vp, _vp],
    "ekv_model_set_io": [_vp, _vp, _vp, _vp],
    "ekv_model_synthesize": [_vp, _u64, _d, _d],
    "ekv_model_weights": [_vp, _i, _pp, _pp],
    "ekv_model_io": [_vp, _pp, _pp, _pp],
    "ekv_kvctx_create": [_vp, _i, _ip, _i, _pp],
    "ekv_kvctx_destroy": [_vp],
    "ekv_kvctx_layer": [_vp, _i, C.POINTER(ekv_segment)],
    "ekv_kvctx_upload_bf16": [_vp, _i, _vp, _vp],
    "ekv_kvctx_set_layer": [_vp, _i, _vp, _vp, _vp, _vp],
    "ekv_kvctx_synthesize": [_vp, _u64],
    "ekv_kvctx_copy_layers": [_vp, _vp, _ip, _i],
    "ekv_session_create": [_vp, _vp, _i, _pp],
    "ekv_session_destroy": [_vp],
    "ekv_session_reset": [_vp],
    "ekv_session_length": [_vp, _ip],
    "ekv_session_forward": [_vp, _vp, _i, _vp],
    "ekv_session_decode": [_vp, _i, _vp],
    "ekv_session_set_decode_path": [_vp, _i, _ip],
    "ekv_session_trace_step": [_vp, C.POINTER(C.c_uint64), _i, _ip],
    "ekv_session_profile_step": [_vp, _fp, _i, _ip],
    "ekv_session_user_kv": [_vp, _i, _pp, _pp, _ip],
    "ekv_session_forward_pipelined": [_vp, _vp, _i, _vp, _vp, _i, _fp, _fp, _fp],
    "ekv_session_forward_streamed": [_vp, _vp, _i, _vp, _vp],
    "ekv_batch_create": [_vp, _vp, _i, _i, _pp],
    "ekv_fnv1a64": [_vp, C.c_size_t, _u64, C.POINTER(C.c_uint64)],
    "ekv_kvpack_size": [_i, _i, _i, _i, _i, _i, C.POINTER(C.c_size_t)],
    "ekv_kvpack_export": [_vp, _ip, _ip, _i, _ip, _i, _vp, C.c_size_t],
    "ekv_kvpack_parse": [_vp, C.c_size_t, C.POINTER(ekv_kvpack_info), _ip, _ip, _ip],
    "ekv_kvpack_import": [_vp, _vp, C.c_size_t],
    "ekv_session_forward_pack": [_vp, _vp, _i, _vp, _vp, C.c_size_t],
    "ekv_batch_destroy": [_vp],
    "ekv_batch_reset": [_vp],
    "ekv_batch_info": [_vp, _ip, _ip, _ip],
    "ekv_batch_forward": [_vp, _vp, _i, _vp],
    "ekv_batch_decode": [_vp, _i, _vp],
    "ekv_batch_profile_row": [_vp, _fp, _i, _ip],
    "ekv_collaborative_decode_batch": [_vp, _vp, _i, _i, _vp, _vp],
    "ekv_collaborative_decode": [_vp, _vp, _i, _i, _vp, _vp],
    "ekv_link_unique_id": [_vp],
    "ekv_link_create": [_vp, _vp, _i, _i, _pp],
    "ekv_link_destroy": [_vp],
    "ekv_link_send_layers": [_vp, _vp, _ip, _i, _i, _fp],
    "ekv_link_recv_forward": [_vp, _vp, _ip, _i, _i, _vp, _i, _vp, _fp],
    "ekv_cache_source": [_i, _d, _d, _i, _i, _ip],
    "ekv_pipeline_schedule": [_dp, _dp, _i, _dp, _dp, _dp],
}
_RET = {"ekv_last_error": C.c_char_p}

_lib = None


def load(path: str = LIBEKV):
    """Load libekv.so (raises if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is not built: run `python -m paper_2505_14085_b200.build` "
                               "(the B200 path has no CPU fallback)")
        lib = C.CDLL(path)
        for name, args in PROTOS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RET.get(name, C.c_int)
        _lib = lib
    return _lib


def call(name: str, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != EKV_OK:
        raise EkvError(rc, lib.ekv_last_error().decode())
    return rc


def last_error() -> str:
    return load().ekv_last_error().decode()
