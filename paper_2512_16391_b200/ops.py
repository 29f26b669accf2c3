"""Batched PyTorch API over the C ABI (device tensors in, device tensors out).

Decode (one query token per sequence; the reference's decode tile
[n-1, n) with causal bound n, tiles.py:145-150):

    dense_decode(q, k, v, n)                       -> out, lse    (+scores)
    anchor_decode(q, k, v, n, policy, layer0=...)  -> out, lse, indices, counts
    reuse_decode(q, k, v, n, indices, counts, head_map) -> out
    select_decode(scores, lse, n, policy, Hkv)     -> indices, counts
    topk(values, k)                                -> indices, counts

Prefill (one layer, batch 1; tiles of 128 query rows, tiles.py:137-144):

    dense_prefill(q, k, v)                         -> out, lse
    anchor_lse_prefill(q, k)                       -> lse
    select_prefill(q, k, lse, policy)              -> indices, counts
    sparse_prefill(q, k, v, indices, counts, head_map) -> out, lse
    anchor_prefill(q, k, v, policy, layer0=...)    -> out, lse, indices, counts
    reuse_prefill(q, k, v, indices, counts, head_map) -> out

Prefill layouts: q bf16 [Hq][N][128], k/v bf16 [Hkv][N][128] (rows
contiguous, any head stride); out bf16 [Hq][N][128]; lse fp32 [Hq][N];
indices int32 [Hkv][T][k_cap] (T = ceil(N/128)), counts int32 [Hkv][T].

Layouts: q bf16 [B][Hq][128]; K/V caches bf16 [B][Hkv][n_cap][128] (any
batch/head strides, rows contiguous); out fp32 [B][Hq][128]; lse fp32
[B][Hq] (natural log); indices int32 [B][Hkv][k_cap] sorted ascending and
INT32_MAX-padded; counts int32 [B][Hkv].  Everything is enqueued on the
current torch stream; nothing synchronises.
"""

from __future__ import annotations

import ctypes
import math
from typing import Optional, Tuple

import torch

from . import _lib
from .exceptions import InvalidArgumentError, UnsupportedOperationError
from .host_types import KBudgetPolicy, k_budget

HEAD_DIM = 128
INT32_MAX = 2**31 - 1


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _need_cuda(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise InvalidArgumentError(f"{name} must be a CUDA tensor (the engine has no CPU path)")


def _check_q(q: torch.Tensor) -> Tuple[int, int]:
    _need_cuda(q, "q")
    if q.dtype != torch.bfloat16:
        raise UnsupportedOperationError(f"q must be bf16, got {q.dtype}")
    if q.dim() != 3 or q.shape[-1] != HEAD_DIM or not q.is_contiguous():
        raise InvalidArgumentError(f"q must be contiguous [B][Hq][128], got {tuple(q.shape)}")
    return q.shape[0], q.shape[1]


def _check_kv(k: torch.Tensor, v: Optional[torch.Tensor], B: int) -> Tuple[int, int, int, int]:
    _need_cuda(k, "k_cache")
    for name, t in (("k_cache", k), ("v_cache", v)):
        if t is None:
            continue
        if t.dtype != torch.bfloat16:
            raise UnsupportedOperationError(f"{name} must be bf16, got {t.dtype}")
        if t.dim() != 4 or t.shape[-1] != HEAD_DIM or t.stride(3) != 1 or t.stride(2) != HEAD_DIM:
            raise InvalidArgumentError(f"{name} must be [B][Hkv][n_cap][128] with contiguous rows")
        if t.shape[0] != B:
            raise InvalidArgumentError(f"{name} batch {t.shape[0]} != q batch {B}")
    if v is not None and (v.shape != k.shape or v.stride() != k.stride()):
        raise InvalidArgumentError("k_cache and v_cache must share shape and strides")
    return k.shape[1], k.shape[2], k.stride(0), k.stride(1)


def decode_workspace_bytes(B: int, Hq: int, Hkv: int) -> int:
    p = _lib.DecodeParams(batch=B, num_q_heads=Hq, num_kv_heads=Hkv, head_dim=HEAD_DIM, seq_len=1)
    nbytes = _lib.c_sz(0)
    _lib.check(_lib.load().kscd_decode_workspace_size(ctypes.byref(p), ctypes.byref(nbytes)))
    return nbytes.value


def new_decode_workspace(device, B: int, Hq: int, Hkv: int) -> torch.Tensor:
    """A zero-filled split-K workspace (partials + arrival counters).  The
    kernels leave it re-armed, so one workspace serves any number of
    stream-ordered calls; it must NOT be shared by calls that can run
    concurrently (other streams, other graphs).  The executors own one each."""
    return torch.zeros(decode_workspace_bytes(B, Hq, Hkv), dtype=torch.uint8, device=device)


_WS = {}


def decode_workspace(device: torch.device, B: int, Hq: int, Hkv: int) -> torch.Tensor:
    """Workspace for standalone op calls that pass none: one per (device,
    current stream, shape), so calls on different streams never share
    arrival counters.  Graph captures and executors pass their own."""
    dev = device.index if device.index is not None else torch.cuda.current_device()
    key = (dev, torch.cuda.current_stream(dev).cuda_stream, B, Hq, Hkv)
    ws = _WS.get(key)
    if ws is None:
        if torch.cuda.is_current_stream_capturing():
            raise InvalidArgumentError("pass workspace= when capturing a CUDA graph (the executors own one)")
        ws = new_decode_workspace(device, B, Hq, Hkv)
        _WS[key] = ws
    return ws


def new_decode_layers_workspace(device, B: int, Hq: int, Hkv: int, num_layers: int) -> torch.Tensor:
    """Zero-filled workspace of a multi-layer decode launch (one split-K
    block per layer, each self re-arming like new_decode_workspace's)."""
    p = _lib.DecodeParams(batch=B, num_q_heads=Hq, num_kv_heads=Hkv, head_dim=HEAD_DIM, seq_len=1)
    nbytes = _lib.c_sz(0)
    _lib.check(_lib.load().kscd_decode_layers_workspace_size(ctypes.byref(p), int(num_layers), ctypes.byref(nbytes)))
    return torch.zeros(nbytes.value, dtype=torch.uint8, device=device)


def _check_seq_lens(seq_lens: Optional[torch.Tensor], B: int, n: int) -> None:
    """Ragged batch: device int32 [B], every entry in [1, seq_len] (checked
    on the device side by the kernels' min(); values are the caller's)."""
    if seq_lens is None:
        return
    _need_cuda(seq_lens, "seq_lens")
    if seq_lens.dtype != torch.int32 or seq_lens.shape != (B,) or not seq_lens.is_contiguous():
        raise InvalidArgumentError(f"seq_lens must be a contiguous CUDA int32 [B={B}] tensor")


def _decode_params(q, k, v, n, out, lse, scores, scale, num_splits, seq_lens=None, workspace=None
                   ) -> _lib.DecodeParams:
    B, Hq = _check_q(q)
    Hkv, n_cap, sb, sh = _check_kv(k, v, B)
    if not (1 <= n <= n_cap):
        raise InvalidArgumentError(f"seq_len {n} outside [1, {n_cap}]")
    if Hq % Hkv:
        raise InvalidArgumentError(f"num_query_heads ({Hq}) must be divisible by num_kv_heads ({Hkv})")
    if workspace is None:
        ws = decode_workspace(q.device, B, Hq, Hkv)
    else:
        if workspace.dtype != torch.uint8 or not workspace.is_cuda or not workspace.is_contiguous():
            raise InvalidArgumentError("workspace must be a contiguous CUDA uint8 tensor (new_decode_workspace)")
        ws = workspace
    p = _lib.DecodeParams(
        batch=B, num_q_heads=Hq, num_kv_heads=Hkv, head_dim=HEAD_DIM, seq_len=int(n),
        q=q.data_ptr(), k_cache=k.data_ptr(), v_cache=_ptr(v), kv_stride_batch=sb, kv_stride_head=sh,
        softmax_scale=float(scale or 0.0), out=_ptr(out), lse=_ptr(lse),
        scores=_ptr(scores), score_stride=scores.stride(1) if scores is not None else 0,
        workspace=ws.data_ptr(), workspace_bytes=ws.numel(), num_splits=int(num_splits))
    _check_seq_lens(seq_lens, B, n)
    p.seq_lens = _ptr(seq_lens)
    return p


def _check_scores(scores: Optional[torch.Tensor], B: int, Hq: int, n: int) -> None:
    if scores is None:
        return
    if scores.dtype != torch.float32 or scores.dim() != 3 or scores.shape[:2] != (B, Hq) \
            or scores.stride(2) != 1 or scores.shape[2] < n or scores.stride(1) % 4 or \
            scores.stride(0) != Hq * scores.stride(1):
        raise InvalidArgumentError("scores must be fp32 [B][Hq][>=n] with a row stride multiple of 4")


def score_buffer(B: int, Hq: int, n: int, device) -> torch.Tensor:
    """log2-domain score scratch for anchor decode layers, rows padded to 4."""
    return torch.empty(B, Hq, (n + 3) // 4 * 4, dtype=torch.float32, device=device)


def dense_decode(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, seq_len: int, *,
                 out: Optional[torch.Tensor] = None, lse: Optional[torch.Tensor] = None,
                 scores: Optional[torch.Tensor] = None, scale: Optional[float] = None,
                 num_splits: int = 0, seq_lens: Optional[torch.Tensor] = None,
                 workspace: Optional[torch.Tensor] = None):
    """Dense attention of the step's query over keys [0, seq_len)
    (dense_attention's last row, attention.py:106-144).  If ``scores`` is
    given, the log2-domain scores s*log2(e) are written for the anchor-0
    selection.  ``seq_lens`` (device int32 [B]) gives a ragged batch its
    own key counts (each <= seq_len)."""
    B, Hq = q.shape[0], q.shape[1]
    out = torch.empty(B, Hq, HEAD_DIM, dtype=torch.float32, device=q.device) if out is None else out
    lse = torch.empty(B, Hq, dtype=torch.float32, device=q.device) if lse is None else lse
    _check_scores(scores, B, Hq, seq_len)
    p = _decode_params(q, k_cache, v_cache, seq_len, out, lse, scores, scale, num_splits, seq_lens, workspace)
    _lib.call("kscd_dense_decode", p, _stream())
    return out, lse


def anchor_scores_decode(q, k_cache, seq_len, scores, lse, *, scale=None, num_splits=0, seq_lens=None,
                         workspace=None):
    """Anchor pass 1: log2-domain scores + LSE; V is not read."""
    B, Hq = q.shape[0], q.shape[1]
    _check_scores(scores, B, Hq, seq_len)
    p = _decode_params(q, k_cache, None, seq_len, None, lse, scores, scale, num_splits, seq_lens, workspace)
    _lib.call("kscd_anchor_scores_decode", p, _stream())
    return scores, lse


def sparse_decode(q, k_cache, v_cache, seq_len, indices, counts, head_map=None, *, out=None, lse=None,
                  scale=None, num_splits=0, workspace=None):
    """topk_attention over a decode tile (attention.py:185-253): kv head g of
    sequence b attends the keys indices[b][head_map[g]][:counts[b][head_map[g]]]
    (runner.py:210-225).  ``head_map`` is a device int32 [Hkv] tensor (None =
    identity)."""
    B, Hq = q.shape[0], q.shape[1]
    if indices.dtype != torch.int32 or counts.dtype != torch.int32 or indices.dim() != 3 \
            or not indices.is_contiguous() or not counts.is_contiguous() \
            or counts.shape != indices.shape[:2] or indices.shape[0] != B:
        raise InvalidArgumentError("indices must be int32 [B][Hsrc][k_cap], counts int32 [B][Hsrc]")
    out = torch.empty(B, Hq, HEAD_DIM, dtype=torch.float32, device=q.device) if out is None else out
    p = _decode_params(q, k_cache, v_cache, seq_len, out, lse, None, scale, num_splits, workspace=workspace)
    if head_map is not None:
        if head_map.dtype != torch.int32 or head_map.numel() != p.num_kv_heads or not head_map.is_cuda:
            raise InvalidArgumentError("head_map must be a CUDA int32 tensor with one entry per kv head")
    p.indices, p.counts = indices.data_ptr(), counts.data_ptr()
    p.k_cap, p.num_src_heads = indices.shape[2], indices.shape[1]
    p.head_map = _ptr(head_map)
    _lib.call("kscd_sparse_decode", p, _stream())
    return out


def select_decode(scores, lse, seq_len, policy: KBudgetPolicy, num_kv_heads: int, *, indices=None,
                  counts=None, pooled=None, all_heads: bool = False, seq_lens=None):
    """Pooled post-softmax weights + k_budget + exact Top-k of one decode
    step (runner.py:164-207).  With ``all_heads`` the pooled vectors of all
    kv heads are combined into one shared set (all-heads-pooled mode,
    runner.py:180-197): the result then has one source head."""
    B, Hq = scores.shape[0], scores.shape[1]
    Hsrc = 1 if all_heads else num_kv_heads
    k = k_budget(policy, seq_len)
    dev = scores.device
    if pooled is None:
        pooled = torch.empty(B * Hsrc, (seq_len + 3) // 4 * 4, dtype=torch.float32, device=dev)
    if indices is None:
        indices = torch.empty(B, Hsrc, k, dtype=torch.int32, device=dev)
    if counts is None:
        counts = torch.empty(B, Hsrc, dtype=torch.int32, device=dev)
    p = _lib.SelectDecodeParams(
        batch=B, num_q_heads=Hq, num_kv_heads=Hsrc, seq_len=int(seq_len), scores=scores.data_ptr(),
        score_stride=scores.stride(1), lse=lse.data_ptr(), pooled=pooled.data_ptr(),
        pooled_stride=pooled.stride(0), topk_fraction=float(policy.fraction), k_min=int(policy.k_min),
        indices=indices.data_ptr(), counts=counts.data_ptr(), k_cap=indices.shape[-1])
    _check_seq_lens(seq_lens, B, seq_len)
    p.seq_lens = _ptr(seq_lens)
    _lib.call("kscd_select_decode", p, _stream())
    return indices, counts


def topk(values: torch.Tensor, k, lengths: Optional[torch.Tensor] = None, k_cap: Optional[int] = None):
    """oracle_topk_indices (attention.py:147-174) for every row of a device
    fp32 matrix: ties to the smaller index, ascending output.  ``k`` is an
    int or a device int32 [rows] tensor."""
    _need_cuda(values, "values")
    if values.dtype != torch.float32 or values.dim() != 2 or values.stride(1) != 1:
        raise InvalidArgumentError("values must be fp32 [rows][len] with contiguous rows")
    rows, length = values.shape
    if isinstance(k, int):
        if k < 1:
            raise InvalidArgumentError(f"k must be >= 1, got {k}")
        kc = k_cap or min(k, length)
        ks = None
    else:
        ks = k
        kc = k_cap or length
    idx = torch.empty(rows, max(kc, 1), dtype=torch.int32, device=values.device)
    cnt = torch.empty(rows, dtype=torch.int32, device=values.device)
    p = _lib.TopkParams(rows=rows, values=values.data_ptr(), value_stride=values.stride(0),
                        lengths=_ptr(lengths), length=length, ks=_ptr(ks), k=k if ks is None else 0,
                        indices=idx.data_ptr(), counts=cnt.data_ptr(), k_cap=idx.shape[1])
    _lib.call("kscd_topk", p, _stream())
    return idx, cnt


def anchor_decode(q, k_cache, v_cache, seq_len, policy: KBudgetPolicy, *, layer0: bool = False,
                  scores=None, lse=None, out=None, indices=None, counts=None, pooled=None,
                  all_heads: bool = False, seq_lens=None):
    """One anchor layer of a decode step.  Layer 0 (anchor0) runs dense
    attention and selects from its scores (runner.py:250-262); other anchors
    run scores-only pass 1, select, then attend sparsely over their own fresh
    sets (runner.py:263-266).  Returns (out, lse, indices, counts)."""
    B, Hq = q.shape[0], q.shape[1]
    Hkv = k_cache.shape[1]
    if scores is None:
        scores = score_buffer(B, Hq, seq_len, q.device)
    lse = torch.empty(B, Hq, dtype=torch.float32, device=q.device) if lse is None else lse
    if layer0:
        out, lse = dense_decode(q, k_cache, v_cache, seq_len, out=out, lse=lse, scores=scores, seq_lens=seq_lens)
        indices, counts = select_decode(scores, lse, seq_len, policy, Hkv, indices=indices, counts=counts,
                                        pooled=pooled, all_heads=all_heads, seq_lens=seq_lens)
        return out, lse, indices, counts
    anchor_scores_decode(q, k_cache, seq_len, scores, lse, seq_lens=seq_lens)
    indices, counts = select_decode(scores, lse, seq_len, policy, Hkv, indices=indices, counts=counts,
                                    pooled=pooled, all_heads=all_heads, seq_lens=seq_lens)
    hm = None
    if all_heads:
        hm = torch.zeros(Hkv, dtype=torch.int32, device=q.device)
    out = sparse_decode(q, k_cache, v_cache, seq_len, indices, counts, hm, out=out)
    return out, lse, indices, counts


def decode_layers(q, k_caches, v_caches, seq_len, *, workspace, tables, out=None, indices=None, counts=None,
                  head_maps=None, index_layer_stride: int = 0, count_layer_stride: int = 0, scores=None,
                  lse=None, scores_layer_stride: int = 0, lse_layer_stride: int = 0, scale=None, num_splits=0):
    """Several independent decode layers in ONE launch:

    * sparse layers when ``indices`` is given -- layer l attends
      indices[b][head_maps[l][g]] (runner.py:210-225), the lists shared by
      every layer (a reuse run) or, with ``index_layer_stride`` /
      ``count_layer_stride`` (elements, may be negative), its own (a group of
      anchors over their fresh sets);
    * the anchor score pass (scores + lse, no V) when ``scores`` is given,
      each layer into scores + l * scores_layer_stride / lse + l * lse_layer_stride;
    * dense layers otherwise.

    q / out: [nl][B][Hq][128] layer-strided views; k_caches / v_caches: nl
    caches of one shape and stride layout with their device pointer arrays in
    ``tables`` (cache_pointer_tables-style); head_maps: device int32
    [nl][Hkv] or None (identity)."""
    nl = len(k_caches)
    if q.dim() != 4 or q.shape[0] != nl or not q[0].is_contiguous():
        raise InvalidArgumentError("q must be [nl][B][Hq][128] with contiguous layers")
    if out is not None and (out.dim() != 4 or out.shape != q.shape or not out[0].is_contiguous()):
        raise InvalidArgumentError("out must be [nl][B][Hq][128] with contiguous layers")
    sparse, score_pass = indices is not None, scores is not None
    if score_pass:
        B, Hq = q.shape[1], q.shape[2]
        _check_scores(scores, B, Hq, seq_len)
    p = _decode_params(q[0], k_caches[0], None if score_pass else v_caches[0], seq_len,
                       None if out is None else out[0], lse, scores, scale, num_splits, workspace=workspace)
    if sparse:
        if indices.dtype != torch.int32 or counts.dtype != torch.int32 or indices.dim() != 3 \
                or not indices.is_contiguous() or not counts.is_contiguous() or counts.shape != indices.shape[:2]:
            raise InvalidArgumentError("indices must be int32 [B][Hsrc][k_cap], counts int32 [B][Hsrc]")
        p.indices, p.counts = indices.data_ptr(), counts.data_ptr()
        p.k_cap, p.num_src_heads = indices.shape[2], indices.shape[1]
    if head_maps is not None and (head_maps.dtype != torch.int32 or tuple(head_maps.shape) != (nl, p.num_kv_heads)
                                  or not head_maps.is_contiguous()):
        raise InvalidArgumentError("head_maps must be a contiguous CUDA int32 [nl][Hkv] tensor")
    kp, vp = tables[0], tables[1]
    # host copies of the pointers: the dense / score passes encode one TMA
    # tensor map per layer on the host (read during the call only)
    kh = (ctypes.c_void_p * nl)(*[t_.data_ptr() for t_ in k_caches])
    vh = (ctypes.c_void_p * nl)(*[t_.data_ptr() for t_ in v_caches])
    t = _lib.DecodeLayers(num_layers=nl, k_caches=kp.data_ptr(), v_caches=vp.data_ptr(),
                          k_caches_host=ctypes.cast(kh, ctypes.c_void_p).value,
                          v_caches_host=ctypes.cast(vh, ctypes.c_void_p).value,
                          q_stride_layer=q.stride(0), out_stride_layer=out.stride(0) if out is not None else q.stride(0),
                          head_maps=_ptr(head_maps), index_stride_layer=int(index_layer_stride),
                          count_stride_layer=int(count_layer_stride), scores_stride_layer=int(scores_layer_stride),
                          lse_stride_layer=int(lse_layer_stride))
    name = ("kscd_anchor_scores_decode_layers" if score_pass else
            "kscd_sparse_decode_layers" if sparse else "kscd_dense_decode_layers")
    _lib.call(name, p, _stream(), t)
    return out


def reuse_decode(q, k_cache, v_cache, seq_len, indices, counts, head_map=None, *, out=None):
    """One reuse layer: the most recent anchor's sets routed through the
    head map (runner.py:267-275)."""
    return sparse_decode(q, k_cache, v_cache, seq_len, indices, counts, head_map, out=out)


def cache_pointer_tables(k_caches, v_caches, device) -> Tuple[torch.Tensor, torch.Tensor, int, int]:
    """Device pointer tables of per-layer caches for ``append_kv``; every
    layer's cache must share one shape and stride layout."""
    ref = k_caches[0]
    for t in list(k_caches) + list(v_caches):
        _need_cuda(t, "cache")
        if t.dtype != torch.bfloat16 or t.shape != ref.shape or t.stride() != ref.stride() or t.stride(3) != 1 \
                or t.stride(2) != HEAD_DIM:
            raise InvalidArgumentError("caches must be bf16 [B][Hkv][n_cap][128] with one shared stride layout")
    kp = torch.tensor([t.data_ptr() for t in k_caches], dtype=torch.int64, device=device)
    vp = torch.tensor([t.data_ptr() for t in v_caches], dtype=torch.int64, device=device)
    return kp, vp, ref.stride(0), ref.stride(1), ref.shape[2]


def append_kv(kv_new: torch.Tensor, position: int, tables, seq_lens: Optional[torch.Tensor] = None) -> None:
    """Write the step's new rows (bf16 [L][2][B][Hkv][128], device) into
    every layer's cache at row ``position`` with one launch -- or, for a
    ragged batch, sequence b's rows at seq_lens[b] - 1 (device int32 [B]);
    the kernel skips a ragged row outside the cache capacity."""
    kp, vp, sb, sh, n_cap = tables
    if not 0 <= position < n_cap:
        raise InvalidArgumentError(f"append position {position} outside the cache (capacity {n_cap})")
    _need_cuda(kv_new, "kv_new")
    if kv_new.dtype != torch.bfloat16 or kv_new.dim() != 5 or kv_new.shape[1] != 2 or kv_new.shape[4] != HEAD_DIM \
            or not kv_new.is_contiguous() or kv_new.shape[0] != kp.numel():
        raise InvalidArgumentError("kv_new must be contiguous bf16 [L][2][B][Hkv][128]")
    L, _, B, Hkv, _ = kv_new.shape
    p = _lib.AppendKvParams(num_layers=L, batch=B, num_kv_heads=Hkv, head_dim=HEAD_DIM, position=position,
                            kv_new=kv_new.data_ptr(), k_caches=kp.data_ptr(), v_caches=vp.data_ptr(),
                            kv_stride_batch=sb, kv_stride_head=sh, cache_capacity=n_cap)
    _check_seq_lens(seq_lens, B, position + 1)
    p.seq_lens = _ptr(seq_lens)
    _lib.call("kscd_append_kv", p, _stream())


def default_scale() -> float:
    return 1.0 / math.sqrt(HEAD_DIM)


# ------------------------------------------------------------------ prefill
TILE = 128


def _check_prefill_qkv(q, k, v):
    for name, t in (("q", q), ("k", k), ("v", v)):
        if t is None:
            continue
        _need_cuda(t, name)
        if t.dtype != torch.bfloat16:
            raise UnsupportedOperationError(f"{name} must be bf16, got {t.dtype}")
        if t.dim() != 3 or t.shape[-1] != HEAD_DIM or t.stride(2) != 1 or t.stride(1) != HEAD_DIM \
                or t.stride(0) % 8:
            raise InvalidArgumentError(f"{name} must be [H][N][128] with contiguous rows")
    Hq, N = q.shape[0], q.shape[1]
    Hkv = k.shape[0]
    if k.shape[1] != N or (v is not None and tuple(v.shape) != tuple(k.shape)):
        raise InvalidArgumentError("q/k/v sequence lengths differ")
    if v is not None and v.stride() != k.stride():
        raise InvalidArgumentError("k and v must share strides")
    if Hq % Hkv:
        raise InvalidArgumentError(f"num_query_heads ({Hq}) must be divisible by num_kv_heads ({Hkv})")
    return Hq, Hkv, N


def _prefill_params(q, k, v, out, lse, causal, scale) -> _lib.PrefillParams:
    Hq, Hkv, N = _check_prefill_qkv(q, k, v)
    return _lib.PrefillParams(
        num_q_heads=Hq, num_kv_heads=Hkv, head_dim=HEAD_DIM, seq_len=N, causal=1 if causal else 0,
        q=q.data_ptr(), k=k.data_ptr(), v=(v if v is not None else k).data_ptr(),
        q_stride_head=q.stride(0), kv_stride_head=k.stride(0), softmax_scale=float(scale or 0.0),
        out=_ptr(out), lse=_ptr(lse), tile_size=TILE)


def dense_prefill(q, k, v, *, causal: bool = True, out=None, lse=None, scale=None):
    """Dense prefill attention of one layer (attention.py:106-144): bf16 O
    and fp32 LSE per row; the Top-k = 100% baseline and anchor 0."""
    Hq, N = q.shape[0], q.shape[1]
    out = torch.empty(Hq, N, HEAD_DIM, dtype=torch.bfloat16, device=q.device) if out is None else out
    lse = torch.empty(Hq, N, dtype=torch.float32, device=q.device) if lse is None else lse
    _lib.call("kscd_dense_prefill", _prefill_params(q, k, v, out, lse, causal, scale), _stream())
    return out, lse


def anchor_lse_prefill(q, k, *, causal: bool = True, lse=None, scale=None):
    """Anchor pass A: per-row LSE only (QK^T and the online softmax sums)."""
    Hq, N = q.shape[0], q.shape[1]
    lse = torch.empty(Hq, N, dtype=torch.float32, device=q.device) if lse is None else lse
    _lib.call("kscd_anchor_lse_prefill", _prefill_params(q, k, None, None, lse, causal, scale), _stream())
    return lse


def prefill_k_cap(policy: KBudgetPolicy, N: int) -> int:
    return k_budget(policy, N)


def select_prefill_scratch(num_q_heads: int, num_kv_heads: int, N: int, device, all_heads: bool = False
                           ) -> torch.Tensor:
    """The pooled scratch select_prefill needs (flat fp32; rows of stride
    (N + 3) // 4 * 4): one row pair per SM when the pass B launch covers the
    kv group and selects in its own tail (G <= 4, post mode -- ~150 MB at
    128K), else the two [Hkv][T][N] partial planes of a separate Top-k."""
    p = _lib.SelectPrefillParams(num_q_heads=num_q_heads, num_kv_heads=num_kv_heads, head_dim=HEAD_DIM,
                                 seq_len=N, pooled_stride=(N + 3) // 4 * 4, all_heads=1 if all_heads else 0,
                                 tile_size=TILE)
    nbytes = _lib.c_sz(0)
    _lib.check(_lib.load().kscd_select_prefill_scratch_size(ctypes.byref(p), ctypes.byref(nbytes)))
    return torch.empty(nbytes.value // 4, dtype=torch.float32, device=device)


def select_prefill(q, k, lse, policy: KBudgetPolicy, *, indices=None, counts=None, pooled=None,
                   all_heads: bool = False, scale=None):
    """Anchor selection of every (kv head, tile): pooled post-softmax weights
    (pass B, runner.py:148-152) and the exact Top-k with k = k_budget(causal
    bound) (runner.py:199-206), fused into one launch when pass B covers the
    kv group.  all_heads -> one shared set per tile.  ``pooled``: a flat fp32
    scratch from select_prefill_scratch."""
    Hq, Hkv, N = _check_prefill_qkv(q, k, None)
    T = (N + TILE - 1) // TILE
    rows = 1 if all_heads else Hkv
    kc = prefill_k_cap(policy, N)
    dev = q.device
    if pooled is None:
        pooled = select_prefill_scratch(Hq, Hkv, N, dev, all_heads)
    if pooled.dtype != torch.float32 or not pooled.is_contiguous() or not pooled.is_cuda:
        raise InvalidArgumentError("pooled scratch must be a contiguous CUDA fp32 tensor (select_prefill_scratch)")
    if indices is None:
        indices = torch.empty(rows, T, kc, dtype=torch.int32, device=dev)
    if counts is None:
        counts = torch.empty(rows, T, dtype=torch.int32, device=dev)
    p = _lib.SelectPrefillParams(
        num_q_heads=Hq, num_kv_heads=Hkv, head_dim=HEAD_DIM, seq_len=N, q=q.data_ptr(), k=k.data_ptr(),
        q_stride_head=q.stride(0), kv_stride_head=k.stride(0), softmax_scale=float(scale or 0.0),
        lse=lse.data_ptr(), pooled=pooled.data_ptr(), pooled_stride=(N + 3) // 4 * 4,
        pooled_bytes=pooled.numel() * 4,
        topk_fraction=float(policy.fraction), k_min=int(policy.k_min), all_heads=1 if all_heads else 0,
        indices=indices.data_ptr(), counts=counts.data_ptr(), k_cap=indices.shape[-1], tile_size=TILE)
    _lib.call("kscd_select_prefill", p, _stream())
    return indices, counts


def sparse_prefill(q, k, v, indices, counts, head_map=None, *, out=None, lse=None, scale=None):
    """topk_attention over every prefill tile (attention.py:185-253) with the
    selections routed through head_map (runner.py:210-225)."""
    Hq, Hkv, N = _check_prefill_qkv(q, k, v)
    T = (N + TILE - 1) // TILE
    if indices.dtype != torch.int32 or indices.dim() != 3 or indices.shape[1] != T or not indices.is_contiguous() \
            or counts.shape != indices.shape[:2] or not counts.is_contiguous():
        raise InvalidArgumentError("indices must be int32 [Hsrc][T][k_cap], counts int32 [Hsrc][T]")
    if head_map is not None and (head_map.dtype != torch.int32 or head_map.numel() != Hkv):
        raise InvalidArgumentError("head_map must be int32 with one entry per kv head")
    out = torch.empty(Hq, N, HEAD_DIM, dtype=torch.bfloat16, device=q.device) if out is None else out
    p = _prefill_params(q, k, v, out, lse, True, scale)
    p.indices, p.counts = indices.data_ptr(), counts.data_ptr()
    p.k_cap, p.num_src_heads = indices.shape[2], indices.shape[0]
    p.head_map = _ptr(head_map)
    _lib.call("kscd_sparse_prefill", p, _stream())
    return out, lse


def anchor_prefill(q, k, v, policy: KBudgetPolicy, *, layer0: bool = False, out=None, lse=None,
                   indices=None, counts=None, pooled=None, all_heads: bool = False):
    """One anchor layer of a prefill: layer 0 runs dense attention and selects
    from it (runner.py:250-262); other anchors run pass A (LSE), pass B +
    Top-k, then attend sparsely over their own sets (runner.py:263-266)."""
    Hq, N = q.shape[0], q.shape[1]
    lse = torch.empty(Hq, N, dtype=torch.float32, device=q.device) if lse is None else lse
    if layer0:
        out, lse = dense_prefill(q, k, v, out=out, lse=lse)
    else:
        anchor_lse_prefill(q, k, lse=lse)
    indices, counts = select_prefill(q, k, lse, policy, indices=indices, counts=counts, pooled=pooled,
                                     all_heads=all_heads)
    if not layer0:
        hm = torch.zeros(k.shape[0], dtype=torch.int32, device=q.device) if all_heads else None
        out, _ = sparse_prefill(q, k, v, indices, counts, hm, out=out)
    return out, lse, indices, counts


def reuse_prefill(q, k, v, indices, counts, head_map=None, *, out=None):
    """One reuse layer of a prefill (runner.py:267-275)."""
    return sparse_prefill(q, k, v, indices, counts, head_map, out=out)[0]


# ------------------------------------------------- pre-softmax selection
def _pre_params(q, k, seq_len, policy, *, prefill, pooled, workspace, indices, counts, all_heads, seq_lens, scale):
    if prefill:
        Hq, Hkv, N = _check_prefill_qkv(q, k, None)
        B, q_sh, kv_sb, kv_sh = 1, q.stride(0), 0, k.stride(0)
    else:
        B, Hq = _check_q(q)
        Hkv, n_cap, kv_sb, kv_sh = _check_kv(k, None, B)
        if not (1 <= seq_len <= n_cap):
            raise InvalidArgumentError(f"seq_len {seq_len} outside [1, {n_cap}]")
        if Hq % Hkv:
            raise InvalidArgumentError(f"num_query_heads ({Hq}) must be divisible by num_kv_heads ({Hkv})")
        q_sh = 0
        _check_seq_lens(seq_lens, B, seq_len)
    return _lib.SelectPreParams(
        batch=B, num_q_heads=Hq, num_kv_heads=Hkv, head_dim=HEAD_DIM, seq_len=int(seq_len),
        tile_size=TILE if prefill else 0, q=q.data_ptr(), q_stride_head=q_sh, k=k.data_ptr(),
        kv_stride_batch=kv_sb, kv_stride_head=kv_sh, softmax_scale=float(scale or 0.0),
        topk_fraction=float(policy.fraction), k_min=int(policy.k_min), all_heads=1 if all_heads else 0,
        seq_lens=_ptr(seq_lens) if not prefill else None)


def select_pre_buffers(B: int, Hkv: int, n: int, policy: KBudgetPolicy, device, *, prefill: bool,
                       all_heads: bool = False, num_q_heads: Optional[int] = None):
    """(pooled, workspace, indices, counts) for select_*_pre: pooled rows are
    the per-(kv head, tile) probabilities plus, in all-heads mode, one mean
    row per tile / sequence."""
    T = (n + TILE - 1) // TILE if prefill else 1
    rows = Hkv * T if prefill else B * Hkv
    out_rows = (T if prefill else B) if all_heads else rows
    pooled = torch.empty(rows + (out_rows if all_heads else 0), (n + 3) // 4 * 4, dtype=torch.float32, device=device)
    p = _lib.SelectPreParams(batch=1 if prefill else B, num_q_heads=num_q_heads or Hkv, num_kv_heads=Hkv,
                             head_dim=HEAD_DIM, seq_len=n, tile_size=TILE if prefill else 0)
    nbytes = _lib.c_sz(0)
    _lib.check(_lib.load().kscd_select_pre_workspace_size(ctypes.byref(p), ctypes.byref(nbytes)))
    ws = torch.empty(nbytes.value, dtype=torch.uint8, device=device)
    kc = k_budget(policy, n)
    idx = torch.empty(out_rows, kc, dtype=torch.int32, device=device)
    cnt = torch.empty(out_rows, dtype=torch.int32, device=device)
    return pooled, ws, idx, cnt


def _run_pre(p, pooled, workspace, indices, counts):
    p.pooled, p.pooled_stride = pooled.data_ptr(), pooled.stride(0)
    p.workspace, p.workspace_bytes = workspace.data_ptr(), workspace.numel()
    p.indices, p.counts, p.k_cap = indices.data_ptr(), counts.data_ptr(), indices.shape[-1]
    _lib.call("kscd_select_pre", p, _stream())


def select_decode_pre(q, k_cache, seq_len, policy: KBudgetPolicy, *, pooled=None, workspace=None, indices=None,
                      counts=None, all_heads: bool = False, seq_lens=None, scale=None):
    """Pre-softmax pooled selection of one decode step (runner.py:155-161
    for the decode tile): q_bar = mean of the group's query heads, softmax
    of K q_bar / sqrt(d), exact Top-k.  No attention pass is needed.
    Returns (indices [B][Hsrc][k_cap], counts [B][Hsrc])."""
    B, Hkv = q.shape[0], k_cache.shape[1]
    if pooled is None or workspace is None or indices is None or counts is None:
        pb, wb, ib, cb = select_pre_buffers(B, Hkv, seq_len, policy, q.device, prefill=False, all_heads=all_heads,
                                            num_q_heads=q.shape[1])
        pooled = pb if pooled is None else pooled
        workspace = wb if workspace is None else workspace
        Hs = 1 if all_heads else Hkv
        indices = ib.view(B, Hs, -1) if indices is None else indices
        counts = cb.view(B, Hs) if counts is None else counts
    p = _pre_params(q, k_cache, seq_len, policy, prefill=False, pooled=pooled, workspace=workspace,
                    indices=indices, counts=counts, all_heads=all_heads, seq_lens=seq_lens, scale=scale)
    _run_pre(p, pooled, workspace, indices, counts)
    return indices, counts


def select_prefill_pre(q, k, policy: KBudgetPolicy, *, pooled=None, workspace=None, indices=None, counts=None,
                       all_heads: bool = False, scale=None):
    """Pre-softmax pooled selection of every (kv head, 128-row tile) of a
    prefill layer (runner.py:155-161,199-206).  Returns (indices
    [Hsrc][T][k_cap], counts [Hsrc][T])."""
    Hq, Hkv, N = _check_prefill_qkv(q, k, None)
    T = (N + TILE - 1) // TILE
    if pooled is None or workspace is None or indices is None or counts is None:
        pb, wb, ib, cb = select_pre_buffers(1, Hkv, N, policy, q.device, prefill=True, all_heads=all_heads,
                                            num_q_heads=Hq)
        pooled = pb if pooled is None else pooled
        workspace = wb if workspace is None else workspace
        Hs = 1 if all_heads else Hkv
        indices = ib.view(Hs, T, -1) if indices is None else indices
        counts = cb.view(Hs, T) if counts is None else counts
    p = _pre_params(q, k, N, policy, prefill=True, pooled=pooled, workspace=workspace, indices=indices,
                    counts=counts, all_heads=all_heads, seq_lens=None, scale=scale)
    _run_pre(p, pooled, workspace, indices, counts)
    return indices, counts
