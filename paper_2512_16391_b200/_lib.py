"""ctypes binding of libkascade_b200.so (include/kascade_b200.h).

The engine has exactly one implementation -- the sm_100a CUDA library.  If
the library is missing or no CUDA device is present every entry point
raises; there is no CPU fallback.
"""

import ctypes
import os
import threading

from .exceptions import InvalidArgumentError, KascadeError, UnsupportedOperationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KSCD_LIB_PATH") or os.path.join(_HERE, "libkascade_b200.so")  # dev override: variant builds

KSCD_OK, KSCD_INVALID_ARGUMENT, KSCD_UNSUPPORTED, KSCD_CUDA_ERROR = 0, 1, 2, 3

c_i32, c_i64, c_f32, c_f64, c_vp, c_sz = (ctypes.c_int32, ctypes.c_int64, ctypes.c_float,
                                          ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t)


class DecodeParams(ctypes.Structure):
    _fields_ = [
        ("batch", c_i32), ("num_q_heads", c_i32), ("num_kv_heads", c_i32), ("head_dim", c_i32),
        ("seq_len", c_i32),
        ("q", c_vp), ("k_cache", c_vp), ("v_cache", c_vp),
        ("kv_stride_batch", c_i64), ("kv_stride_head", c_i64),
        ("softmax_scale", c_f32),
        ("out", c_vp), ("lse", c_vp),
        ("indices", c_vp), ("counts", c_vp), ("k_cap", c_i32), ("num_src_heads", c_i32),
        ("head_map", c_vp),
        ("scores", c_vp), ("score_stride", c_i64),
        ("workspace", c_vp), ("workspace_bytes", c_sz),
        ("num_splits", c_i32),
        ("seq_lens", c_vp),
    ]


class SelectDecodeParams(ctypes.Structure):
    _fields_ = [
        ("batch", c_i32), ("num_q_heads", c_i32), ("num_kv_heads", c_i32), ("seq_len", c_i32),
        ("scores", c_vp), ("score_stride", c_i64), ("lse", c_vp),
        ("pooled", c_vp), ("pooled_stride", c_i64),
        ("topk_fraction", c_f64), ("k_min", c_i32),
        ("indices", c_vp), ("counts", c_vp), ("k_cap", c_i32),
        ("seq_lens", c_vp),
    ]


class TopkParams(ctypes.Structure):
    _fields_ = [
        ("rows", c_i32), ("values", c_vp), ("value_stride", c_i64),
        ("lengths", c_vp), ("length", c_i32), ("ks", c_vp), ("k", c_i32),
        ("indices", c_vp), ("counts", c_vp), ("k_cap", c_i32),
    ]


class PrefillParams(ctypes.Structure):
    _fields_ = [
        ("num_q_heads", c_i32), ("num_kv_heads", c_i32), ("head_dim", c_i32), ("seq_len", c_i32),
        ("causal", c_i32),
        ("q", c_vp), ("k", c_vp), ("v", c_vp),
        ("q_stride_head", c_i64), ("kv_stride_head", c_i64),
        ("softmax_scale", c_f32),
        ("out", c_vp), ("lse", c_vp),
        ("indices", c_vp), ("counts", c_vp), ("k_cap", c_i32), ("num_src_heads", c_i32),
        ("head_map", c_vp), ("tile_size", c_i32),
    ]


class SelectPrefillParams(ctypes.Structure):
    _fields_ = [
        ("num_q_heads", c_i32), ("num_kv_heads", c_i32), ("head_dim", c_i32), ("seq_len", c_i32),
        ("q", c_vp), ("k", c_vp), ("q_stride_head", c_i64), ("kv_stride_head", c_i64),
        ("softmax_scale", c_f32), ("lse", c_vp),
        ("pooled", c_vp), ("pooled_stride", c_i64), ("pooled_bytes", c_sz),
        ("topk_fraction", c_f64), ("k_min", c_i32), ("all_heads", c_i32),
        ("indices", c_vp), ("counts", c_vp), ("k_cap", c_i32), ("tile_size", c_i32),
    ]


class ProbsParams(ctypes.Structure):
    _fields_ = [
        ("num_q_heads", c_i32), ("num_kv_heads", c_i32), ("head_dim", c_i32), ("seq_len", c_i32),
        ("causal", c_i32), ("q", c_vp), ("k", c_vp), ("q_stride_head", c_i64), ("kv_stride_head", c_i64),
        ("softmax_scale", c_f32), ("lse", c_vp), ("probs", c_vp),
    ]


class PoolTilesParams(ctypes.Structure):
    _fields_ = [
        ("num_q_heads", c_i32), ("num_kv_heads", c_i32), ("head_dim", c_i32), ("seq_len", c_i32),
        ("num_tiles", c_i32), ("tile_starts", c_vp), ("tile_ends", c_vp), ("pooling", c_i32),
        ("all_heads", c_i32), ("probs", c_vp), ("q", c_vp), ("k", c_vp), ("q_stride_head", c_i64),
        ("kv_stride_head", c_i64), ("pooled", c_vp), ("pooled_stride", c_i64), ("scratch", c_vp),
    ]


class AppendKvParams(ctypes.Structure):
    _fields_ = [
        ("num_layers", c_i32), ("batch", c_i32), ("num_kv_heads", c_i32), ("head_dim", c_i32),
        ("position", c_i32), ("kv_new", c_vp), ("k_caches", c_vp), ("v_caches", c_vp),
        ("kv_stride_batch", c_i64), ("kv_stride_head", c_i64),
        ("seq_lens", c_vp), ("cache_capacity", c_i32),
    ]


class SelectPreParams(ctypes.Structure):
    _fields_ = [
        ("batch", c_i32), ("num_q_heads", c_i32), ("num_kv_heads", c_i32), ("head_dim", c_i32),
        ("seq_len", c_i32), ("tile_size", c_i32), ("q", c_vp), ("q_stride_head", c_i64), ("k", c_vp),
        ("kv_stride_batch", c_i64), ("kv_stride_head", c_i64), ("softmax_scale", c_f32),
        ("pooled", c_vp), ("pooled_stride", c_i64), ("workspace", c_vp), ("workspace_bytes", c_sz),
        ("topk_fraction", c_f64), ("k_min", c_i32), ("all_heads", c_i32),
        ("indices", c_vp), ("counts", c_vp), ("k_cap", c_i32), ("seq_lens", c_vp),
    ]


class DecodeLayers(ctypes.Structure):
    _fields_ = [
        ("num_layers", c_i32), ("k_caches", c_vp), ("v_caches", c_vp),
        ("q_stride_layer", c_i64), ("out_stride_layer", c_i64), ("head_maps", c_vp),
        ("index_stride_layer", c_i64), ("count_stride_layer", c_i64),
        ("scores_stride_layer", c_i64), ("lse_stride_layer", c_i64),
        ("k_caches_host", c_vp), ("v_caches_host", c_vp),
    ]


# entry point name -> params struct (None for non-struct signatures)
class MaskedMassParams(ctypes.Structure):
    _fields_ = [
        ("num_sets", c_i32), ("num_dists", c_i32), ("rows", c_i32),
        ("dist", c_vp), ("dist_stride_head", c_i64), ("dist_stride_row", c_i64), ("dist_len", c_i32),
        ("indices", c_vp), ("counts", c_vp), ("k_cap", c_i32),
        ("mass", c_vp),
    ]


ENTRY_POINTS = {
    "kscd_dense_decode": DecodeParams,
    "kscd_anchor_scores_decode": DecodeParams,
    "kscd_sparse_decode": DecodeParams,
    "kscd_select_decode": SelectDecodeParams,
    "kscd_topk": TopkParams,
    "kscd_dense_prefill": PrefillParams,
    "kscd_anchor_lse_prefill": PrefillParams,
    "kscd_sparse_prefill": PrefillParams,
    "kscd_select_prefill": SelectPrefillParams,
    "kscd_dense_probs": ProbsParams,
    "kscd_pool_tiles": PoolTilesParams,
    "kscd_append_kv": AppendKvParams,
    "kscd_masked_mass": MaskedMassParams,
    "kscd_select_pre": SelectPreParams,
}

_lock = threading.Lock()
_lib = None


ABI_VERSION = 2   # include/kascade_b200.h KSCD_ABI_VERSION


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) the CUDA library; raises KascadeError when it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise KascadeError(
                f"{path} is missing: build it with `python -m paper_2512_16391_b200.build` "
                "(the engine has no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, st in ENTRY_POINTS.items():
            if os.environ.get("KSCD_LIB_PATH") and not hasattr(lib, name):
                continue            # dev override: an older variant build may lack newer entry points
            fn = getattr(lib, name)
            fn.argtypes = [ctypes.POINTER(st), c_vp]
            fn.restype = ctypes.c_int
        lib.kscd_last_error.restype = ctypes.c_char_p
        lib.kscd_last_error.argtypes = []
        lib.kscd_abi_version.restype = ctypes.c_int
        if lib.kscd_abi_version() != ABI_VERSION:
            raise KascadeError(f"{path} has ABI version {lib.kscd_abi_version()}, the binding expects "
                               f"{ABI_VERSION}: rebuild with `python -m paper_2512_16391_b200.build`")
        lib.kscd_k_budget.restype = c_i32
        lib.kscd_k_budget.argtypes = [c_f64, c_i32, c_i32]
        lib.kscd_decode_workspace_size.restype = ctypes.c_int
        lib.kscd_decode_workspace_size.argtypes = [ctypes.POINTER(DecodeParams), ctypes.POINTER(c_sz)]
        for name in ("kscd_sparse_decode_layers", "kscd_dense_decode_layers", "kscd_anchor_scores_decode_layers"):
            fn = getattr(lib, name)
            fn.argtypes = [ctypes.POINTER(DecodeParams), ctypes.POINTER(DecodeLayers), c_vp]
            fn.restype = ctypes.c_int
        lib.kscd_decode_layers_workspace_size.restype = ctypes.c_int
        lib.kscd_decode_layers_workspace_size.argtypes = [ctypes.POINTER(DecodeParams), c_i32, ctypes.POINTER(c_sz)]
        lib.kscd_select_prefill_scratch_size.restype = ctypes.c_int
        lib.kscd_select_prefill_scratch_size.argtypes = [ctypes.POINTER(SelectPrefillParams), ctypes.POINTER(c_sz)]
        lib.kscd_select_pre_workspace_size.restype = ctypes.c_int
        lib.kscd_select_pre_workspace_size.argtypes = [ctypes.POINTER(SelectPreParams), ctypes.POINTER(c_sz)]
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception taxonomy."""
    if rc == KSCD_OK:
        return
    msg = load().kscd_last_error().decode("utf-8", "replace")
    if rc == KSCD_INVALID_ARGUMENT:
        raise InvalidArgumentError(msg)
    if rc == KSCD_UNSUPPORTED:
        raise UnsupportedOperationError(msg)
    raise KascadeError(msg)


def call(name: str, params, stream_ptr: int, extra=None) -> None:
    fn = getattr(load(), name)
    if extra is None:
        check(fn(ctypes.byref(params), c_vp(stream_ptr)))
    else:
        check(fn(ctypes.byref(params), ctypes.byref(extra), c_vp(stream_ptr)))
