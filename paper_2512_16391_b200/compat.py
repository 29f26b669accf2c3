"""The reference's trace-level API, executed by the B200 kernels.

Same names, arguments, results and errors as ``kascade`` 0.1.0 so a caller
can switch imports:

    dense_attention(trace, layer, causal=True) -> (P, Y)      attention.py:106-144
    oracle_topk_indices(p, k, kv_head=0, tile_id=0)          attention.py:147-174
    topk_attention(trace, layer, selections, tiles, causal=True, dense_P=None)
                                                              attention.py:185-253
    run_dense(trace)                                          runner.py:132-137
    run_kascade(trace, plan, phase="prefill") -> (outputs, RunReport)
                                                              runner.py:228-297
    compare(a, b) -> RunReport                                runner.py:321-344
    softmax_row(scores)                                       attention.py:77-90

Inputs are the reference's fp32 numpy traces; the engine computes in bf16
(Q/K/V are rounded to bf16 on upload -- parity inputs are bf16-representable,
SURVEY.md 8(c)) and returns fp32 numpy.  Prefill with 128-row tiles and
post-softmax pooling runs the performance kernels (tcgen05 prefill, pass-B
pooling, per-tile Top-k); any other TileSpec (decode phase, other tile
sizes, pre-softmax pooling) runs reference-scale kernels: materialised P,
pooled tile rows, and the decode sparse kernel with one query row per
"sequence".  ``mass_recovered`` is exp(LSE_sparse - LSE_dense), which equals
the reference's sum of dense P over the visible selected keys.
"""

from __future__ import annotations

import math
from typing import Dict, List, Mapping, Sequence, Tuple, Union

import numpy as np
import torch

from . import _lib, ops
from .exceptions import InvalidArgumentError, InvalidPlanError, NumericError, UnsupportedOperationError
from .host_types import (DECODE, KIND_ANCHOR, KIND_ANCHOR0, KIND_REUSE, MODE_ALL_HEADS_POOLED, MODE_REMAPPED,
                         POOL_POST, POOL_PRE, PREFILL, LayerReport, RunReport, TileSpec, TopkAttentionResult,
                         TopKIndexSet, k_budget, make_tiles, validate_plan)

MAX_P_SEQ = 8192        # materialised P is [Hq][N][N] fp32, like the reference


def _dev():
    if not torch.cuda.is_available():
        raise UnsupportedOperationError("the B200 engine needs a CUDA device (there is no CPU path)")
    return torch.device("cuda")


def _check_head_dim(d: int) -> None:
    if not 1 <= d <= ops.HEAD_DIM:
        raise UnsupportedOperationError(f"head_dim {d} unsupported (the engine's rows are {ops.HEAD_DIM} wide)")


def _scale(trace) -> float:
    """attention.py:120: 1/sqrt(d) of the trace's logical head dim."""
    return 1.0 / math.sqrt(trace.head_dim)


def _layer(trace, layer: int):
    """One layer as bf16 device tensors [H][N][128].  A trace with d < 128
    (the reference's own small-d tests) is zero-padded to the engine's row
    width: Q.K^T is unchanged, every call passes the trace's 1/sqrt(d) and
    the outputs are cut back to d (the C ABI's head_dim convention)."""
    if not 0 <= layer < trace.num_layers:
        raise InvalidArgumentError(f"layer {layer} out of range [0, {trace.num_layers})")
    _check_head_dim(trace.head_dim)
    dev = _dev()
    if hasattr(trace, "layer_device"):          # kscd_io.TraceFile: stream from the mmap
        q, k, v = trace.layer_device(layer, dev)
    else:
        to = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev).to(torch.bfloat16)  # noqa
        q, k, v = to(trace.Q[layer]), to(trace.K[layer]), to(trace.V[layer])
    pad = ops.HEAD_DIM - trace.head_dim
    if pad:
        q, k, v = (torch.nn.functional.pad(x, (0, pad)) for x in (q, k, v))
    return q, k, v


def _check_finite(Y: torch.Tensor, layer: int):
    bad = ~torch.isfinite(Y).all(dim=-1)          # [Hq][N]
    if bool(bad.any()):
        h, r = (int(x) for x in torch.nonzero(bad)[0])
        raise NumericError("non-finite attention intermediate", layer=layer, head=h, row=r)


def _probs(q, k, lse, causal: bool, d: int = 128) -> torch.Tensor:
    Hq, N = q.shape[0], q.shape[1]
    if N > MAX_P_SEQ:
        raise UnsupportedOperationError(f"materialised P needs N <= {MAX_P_SEQ} (got {N})")
    P = torch.empty(Hq, N, N, dtype=torch.float32, device=q.device)
    p = _lib.ProbsParams(num_q_heads=Hq, num_kv_heads=k.shape[0], head_dim=d, seq_len=N,
                         causal=1 if causal else 0, q=q.data_ptr(), k=k.data_ptr(), q_stride_head=q.stride(0),
                         kv_stride_head=k.stride(0), lse=lse.data_ptr(), probs=P.data_ptr())
    _lib.call("kscd_dense_probs", p, ops._stream())
    return P


def dense_attention(trace, layer: int, causal: bool = True) -> Tuple[np.ndarray, np.ndarray]:
    """(P [Hq][N][N], Y [Hq][N][d]) of one layer; P is materialised only
    because the reference returns it (N <= MAX_P_SEQ)."""
    q, k, v = _layer(trace, layer)
    d = trace.head_dim
    out, lse = ops.dense_prefill(q, k, v, causal=causal, scale=_scale(trace))
    Y = out[..., :d].float()
    _check_finite(Y, layer)
    P = _probs(q, k, lse, causal, d)
    return P.cpu().numpy(), Y.cpu().numpy()


def softmax_row(scores) -> np.ndarray:
    """attention.py:77-90: fp64 softmax of one score vector, fp32 result."""
    s = np.asarray(scores)
    if s.ndim != 1 or s.size == 0:
        raise InvalidArgumentError("scores must be a non-empty vector")
    if not np.isfinite(s).all():
        raise InvalidArgumentError("scores must be finite")
    t = torch.from_numpy(s.astype(np.float64)).to(_dev())
    return torch.softmax(t, dim=0).to(torch.float32).cpu().numpy()


def oracle_topk_indices(p, k: int, kv_head: int = 0, tile_id: int = 0) -> TopKIndexSet:
    """The k largest weights, ties to the smaller position, ascending (the
    exact radix-select kernel)."""
    if k < 1:
        raise InvalidArgumentError(f"k must be >= 1, got {k}")
    positions = None
    if hasattr(p, "weights") and hasattr(p, "key_positions"):
        weights = np.asarray(p.weights)
        positions = np.asarray(p.key_positions, dtype=np.int64)
    else:
        weights = np.asarray(p)
    if weights.ndim != 1 or weights.size == 0:
        raise InvalidArgumentError("p must be a non-empty vector")
    vals = torch.from_numpy(weights.astype(np.float32)).to(_dev())[None]
    idx, cnt = ops.topk(vals, int(k))
    sel = idx[0, :int(cnt.item())].cpu().numpy().astype(np.int64)
    if positions is not None:
        sel = positions[sel]
    return TopKIndexSet(kv_head=kv_head, tile_id=tile_id, indices=sel, k=k)


def _sel_map(selections) -> Dict[Tuple[int, int], np.ndarray]:
    if isinstance(selections, Mapping):
        items = selections.items()
    else:
        items = (((s.kv_head, s.tile_id), s) for s in selections)
    return {key: np.asarray(getattr(s, "indices", s), dtype=np.int64) for key, s in items}


def _standard_prefill(tiles, N: int, Hkv: int) -> bool:
    if tiles.phase != PREFILL or tiles.tile_size != ops.TILE:
        return False
    want = make_tiles(N, PREFILL, Hkv, Hkv, ops.TILE).tiles
    return sorted((t.kv_head, t.tile_id, t.start, t.end) for t in tiles.tiles) == \
        sorted((t.kv_head, t.tile_id, t.start, t.end) for t in want)


def _sparse_any_tiles(q, k, v, tiles, sels, causal: bool, scale: float):
    """Sparse attention for an arbitrary TileSpec: every query row is one
    'sequence' of the decode sparse kernel whose list is its tile's selection
    truncated to the keys <= row (the staircase), K/V shared (batch stride 0).
    Returns (Y [Hq][N][d] fp32, lse [Hq][N], vis [Hkv][N])."""
    Hq, N = q.shape[0], q.shape[1]
    Hkv = k.shape[0]
    dev = q.device
    kc = max(1, max((s.size for s in sels.values()), default=1))
    idx = np.full((N, Hkv, kc), 2**31 - 1, np.int32)
    vis = np.zeros((N, Hkv), np.int32)
    for t in tiles.tiles:
        sel = sels[(t.kv_head, t.tile_id)]
        rows = np.arange(t.start, t.end)
        idx[t.start:t.end, t.kv_head, :sel.size] = sel
        vis[t.start:t.end, t.kv_head] = np.searchsorted(sel, rows, side="right") if causal else sel.size
    q_rows = q.permute(1, 0, 2).contiguous()
    kx = k.unsqueeze(0).expand(N, Hkv, N, 128)
    vx = v.unsqueeze(0).expand(N, Hkv, N, 128)
    lse = torch.empty(N, Hq, dtype=torch.float32, device=dev)
    out = ops.sparse_decode(q_rows, kx, vx, N, torch.from_numpy(idx).to(dev), torch.from_numpy(vis).to(dev),
                            None, lse=lse, scale=scale)
    return out.permute(1, 0, 2).contiguous(), lse.t().contiguous(), vis.T


def topk_attention(trace, layer: int, selections, tiles, causal: bool = True, dense_P=None) -> TopkAttentionResult:
    """Sparse attention over per-(kv head, tile) selections; softmax
    renormalised over the selected keys, row r sees the selected keys <= r,
    rows with none fall back to V[g][r] and are flagged."""
    sels = _sel_map(selections)
    N, Hq, Hkv = trace.seq_len, trace.num_query_heads, trace.num_kv_heads
    G = Hq // Hkv
    for t in tiles.tiles:
        key = (t.kv_head, t.tile_id)
        if key not in sels:
            raise InvalidArgumentError(f"no Top-k set for kv head {t.kv_head}, tile {t.tile_id}")
        sel = sels[key]
        if causal and sel.size and sel[-1] >= t.causal_bound:
            raise InvalidArgumentError(f"selection for kv head {t.kv_head}, tile {t.tile_id} breaks the tile's "
                                       f"causal bound {t.causal_bound}")
    q, k, v = _layer(trace, layer)
    dev = q.device
    sc = _scale(trace)
    _, lse_d = ops.dense_prefill(q, k, v, causal=causal, scale=sc)
    if causal and _standard_prefill(tiles, N, Hkv):
        T = (N + ops.TILE - 1) // ops.TILE
        kc = max(1, max(s.size for s in sels.values()))
        idx = np.full((Hkv, T, kc), 2**31 - 1, np.int32)
        cnt = np.zeros((Hkv, T), np.int32)
        for (g, tid), sel in sels.items():
            if g < Hkv and tid < T:
                idx[g, tid, :sel.size] = sel
                cnt[g, tid] = sel.size
        lse_s = torch.empty(Hq, N, dtype=torch.float32, device=dev)
        out, _ = ops.sparse_prefill(q, k, v, torch.from_numpy(idx).to(dev), torch.from_numpy(cnt).to(dev),
                                    lse=lse_s, scale=sc)
        Y = out.float()
        rows = torch.arange(N, device=dev)
        vis_np = np.zeros((Hkv, N), np.int64)
        for t in tiles.tiles:
            sel = sels[(t.kv_head, t.tile_id)]
            vis_np[t.kv_head, t.start:t.end] = np.searchsorted(sel, np.arange(t.start, t.end), side="right")
        del rows
    else:
        Y, lse_s, vis_np = _sparse_any_tiles(q, k, v, tiles, sels, causal, sc)
        # rows with no visible selected key: the diagonal fallback V[g][r]
        dead = torch.from_numpy(vis_np == 0).to(dev)                     # [Hkv][N]
        if bool(dead.any()):
            dead_h = dead.repeat_interleave(G, dim=0)                    # [Hq][N]
            vrows = v.float().repeat_interleave(G, dim=0)                # [Hq][N][d]
            Y = torch.where(dead_h[..., None], vrows, Y)
    mass = torch.exp(lse_s - lse_d)
    mass = torch.where(torch.isfinite(lse_s), mass, torch.zeros_like(mass))
    fallback: List[Tuple[int, int]] = []
    for t in tiles.tiles:
        rows = np.arange(t.start, t.end)
        dead_rows = rows[vis_np[t.kv_head, t.start:t.end] == 0]
        for h in range(t.kv_head * G, (t.kv_head + 1) * G):
            fallback.extend((h, int(r)) for r in dead_rows)
    Y = Y[..., :trace.head_dim]
    return TopkAttentionResult(Y=Y.cpu().numpy(), mass_recovered=mass.float().cpu().numpy(), fallback_rows=fallback)


def run_dense(trace) -> np.ndarray:
    """Dense outputs of every layer: [L][Hq][N][d] fp32."""
    outs = []
    for layer in range(trace.num_layers):
        q, k, v = _layer(trace, layer)
        out, _ = ops.dense_prefill(q, k, v, scale=_scale(trace))
        outs.append(out[..., :trace.head_dim].float())
    return torch.stack(outs).cpu().numpy()


def _rel_l2(a: torch.Tensor, b: torch.Tensor) -> float:
    num = torch.linalg.vector_norm((a.double() - b.double()).flatten()).item()
    den = torch.linalg.vector_norm(b.double().flatten()).item()
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(num / den)


def _select_any_tiles(q, k, lse, tiles, plan, Hkv: int, d: int = 128) -> Dict[Tuple[int, int], np.ndarray]:
    """_anchor_selections (runner.py:164-207) for an arbitrary TileSpec via
    materialised P (post) or the pre-softmax pooled rows."""
    dev = q.device
    Hq, N = q.shape[0], q.shape[1]
    by_head: Dict[int, List] = {}
    for t in tiles.tiles:
        by_head.setdefault(t.kv_head, []).append(t)
    tiles0 = sorted(by_head[0], key=lambda t: t.tile_id)
    T = len(tiles0)
    starts = torch.tensor([t.start for t in tiles0], dtype=torch.int32, device=dev)
    ends = torch.tensor([t.end for t in tiles0], dtype=torch.int32, device=dev)
    all_heads = plan.mode == MODE_ALL_HEADS_POOLED
    stride = (N + 3) // 4 * 4
    pre = plan.pooling == POOL_PRE
    rows = Hkv
    pooled = torch.zeros(rows, T, stride, dtype=torch.float32, device=dev)
    pp = _lib.PoolTilesParams(num_q_heads=Hq, num_kv_heads=Hkv, head_dim=d, seq_len=N, num_tiles=T,
                              tile_starts=starts.data_ptr(), tile_ends=ends.data_ptr(), pooling=1 if pre else 0,
                              all_heads=0, q=q.data_ptr(), k=k.data_ptr(), q_stride_head=q.stride(0),
                              kv_stride_head=k.stride(0), pooled=pooled.data_ptr(), pooled_stride=stride)
    if pre:
        scratch = torch.empty(Hkv, T, stride, dtype=torch.float64, device=dev)
        pp.scratch = scratch.data_ptr()
    else:
        P = _probs(q, k, lse, True, d)
        pp.probs = P.data_ptr()
    _lib.call("kscd_pool_tiles", pp, ops._stream())
    if all_heads:
        # runner.py:188-196: np.mean over kv heads of the pooled vectors
        pooled = pooled.double().mean(dim=0, keepdim=True).float()
    lens = ends.long()
    ks = torch.tensor([k_budget(plan.k_policy, t.end) for t in tiles0], dtype=torch.int32, device=dev)
    nrow = pooled.shape[0]
    idx, cnt = ops.topk(pooled.reshape(nrow * T, stride), ks.repeat(nrow),
                        lengths=lens.to(torch.int32).repeat(nrow), k_cap=int(ks.max().item()))
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    out = {}
    for g in range(Hkv):
        r = 0 if all_heads else g
        for i, t in enumerate(tiles0):
            out[(g, t.tile_id)] = idx[r * T + i, :cnt[r * T + i]].astype(np.int64)
    return out


def run_kascade(trace, plan, phase: str = PREFILL) -> Tuple[np.ndarray, RunReport]:
    """The anchor/reuse pipeline with the reference's report (runner.py:228-318):
    layer 0 dense (+ selections), anchors select fresh sets and attend
    sparsely, reuse layers route the latest anchor's sets through their head
    map.  Fidelity (rel-L2 vs dense, recovered mass, fallback rows) per layer."""
    # runner.py:236 -- plan errors raise InvalidPlanError, head-map errors the
    # reference HeadMap's own InvalidArgumentError (heads.py:37-47), unchanged
    validate_plan(plan, trace)
    L, Hq, Hkv, N = trace.num_layers, trace.num_query_heads, trace.num_kv_heads, trace.seq_len
    G = Hq // Hkv
    tiles = make_tiles(N, phase, Hq, Hkv, plan.tile_size)
    fast = phase == PREFILL and plan.tile_size == ops.TILE   # the engine's prefill kernels (both poolings)
    anchors = set(plan.core.anchors)
    outputs = np.empty((L, Hq, N, trace.head_dim), np.float32)
    reports: List[LayerReport] = []
    cur = None               # fast path: (idx, cnt) device tensors; else dict of sets
    d, sc = trace.head_dim, _scale(trace)
    for layer in range(L):
        q, k, v = _layer(trace, layer)
        out_d, lse_d = ops.dense_prefill(q, k, v, scale=sc)
        Yd = out_d[..., :d].float()
        _check_finite(Yd, layer)
        is_anchor = layer == 0 or layer in anchors
        if is_anchor:
            if fast and plan.pooling == POOL_PRE:
                cur = ops.select_prefill_pre(q, k, plan.k_policy, all_heads=plan.mode == MODE_ALL_HEADS_POOLED,
                                             scale=sc)
            elif fast:
                cur = ops.select_prefill(q, k, lse_d, plan.k_policy, all_heads=plan.mode == MODE_ALL_HEADS_POOLED,
                                         scale=sc)
            else:
                cur = _select_any_tiles(q, k, lse_d, tiles, plan, Hkv, d)
        if layer == 0:
            outputs[0] = Yd.cpu().numpy()
            reports.append(LayerReport(0, KIND_ANCHOR0, 0.0, 1.0))
            continue
        kind = KIND_ANCHOR if layer in anchors else KIND_REUSE
        if fast:
            idx, cnt = cur
            if plan.mode == MODE_ALL_HEADS_POOLED:
                hmap = torch.zeros(Hkv, dtype=torch.int32, device=q.device)
            elif kind == KIND_REUSE:
                hmap = torch.tensor(plan.head_maps[layer].map, dtype=torch.int32, device=q.device)
            else:
                hmap = None
            lse_s = torch.empty(Hq, N, dtype=torch.float32, device=q.device)
            out, _ = ops.sparse_prefill(q, k, v, idx, cnt, hmap, lse=lse_s, scale=sc)
            Y = out[..., :d].float()
            fb = int((~torch.isfinite(lse_s)).sum().item())
        else:
            if kind == KIND_REUSE and plan.mode == MODE_REMAPPED:
                hm = plan.head_maps[layer].map
                sels = {(g, tid): cur[(hm[g], tid)] for (g, tid) in cur}
            else:
                sels = cur
            Y, lse_s, vis = _sparse_any_tiles(q, k, v, tiles, sels, True, sc)
            dead = torch.from_numpy(vis == 0).to(q.device)
            if bool(dead.any()):
                Y = torch.where(dead.repeat_interleave(G, dim=0)[..., None], v.float().repeat_interleave(G, dim=0), Y)
            Y = Y[..., :d]
            fb = int(dead.sum().item()) * G
        mass = torch.where(torch.isfinite(lse_s), torch.exp(lse_s - lse_d), torch.zeros_like(lse_s))
        outputs[layer] = Y.cpu().numpy()
        reports.append(LayerReport(layer, kind, _rel_l2(Y, Yd), float(mass.double().mean().item()), fb))
    errs = np.array([r.output_rel_err_l2 for r in reports])
    masses = np.array([r.mass_recovered_mean for r in reports])
    overall = {"mean_output_rel_err_l2": float(errs.mean()), "max_output_rel_err_l2": float(errs.max()),
               "mean_mass_recovered": float(masses.mean()),
               "fallback_rows": int(sum(r.fallback_rows for r in reports))}
    for kind in (KIND_ANCHOR0, KIND_ANCHOR, KIND_REUSE):
        sub = [r for r in reports if r.kind == kind]
        if sub:
            overall[f"{kind}_mean_rel_err"] = float(np.mean([r.output_rel_err_l2 for r in sub]))
            overall[f"{kind}_mean_mass_recovered"] = float(np.mean([r.mass_recovered_mean for r in sub]))
    config = {"plan": plan.digest() if hasattr(plan, "digest") else "", "prompt_id": trace.prompt_id,
              "phase": phase, "mode": plan.mode, "pooling": plan.pooling, "engine": "b200"}
    return outputs, RunReport(per_layer=reports, overall=overall, config=config)


def compare(outputs_a, outputs_b) -> RunReport:
    """Per-layer rel-L2 of a against reference b (runner.py:321-344)."""
    a, b = np.asarray(outputs_a), np.asarray(outputs_b)
    if a.shape != b.shape:
        raise InvalidArgumentError(f"shape mismatch: {a.shape} vs {b.shape}")
    rel = []
    for i in range(a.shape[0]):
        num = np.linalg.norm((a[i].astype(np.float64) - b[i].astype(np.float64)).ravel())
        den = np.linalg.norm(b[i].astype(np.float64).ravel())
        rel.append(0.0 if den == 0.0 and num == 0.0 else (float("inf") if den == 0.0 else float(num / den)))
    reports = [LayerReport(i, "compare", r, float("nan")) for i, r in enumerate(rel)]
    errs = np.array(rel)
    return RunReport(per_layer=reports,
                     overall={"mean_output_rel_err_l2": float(errs.mean()), "max_output_rel_err_l2": float(errs.max())})


# ------------------------------------------------ small reference utilities
# The reference's pooling / coverage helpers (tiles.py:92-114, metrics.py:
# 80-131, heads.py:155-171, attention.py:21-37) with the same signatures,
# evaluated on the device (fp64 accumulation, fp32 results as in numpy).

class AttentionDistribution:
    """attention.py:21-37: post-softmax weights over the attendable keys of one row."""

    def __init__(self, weights, key_positions):
        self.weights = np.asarray(weights)
        self.key_positions = np.asarray(key_positions)

    def validate(self):
        w = np.asarray(self.weights, dtype=np.float64)
        pos = np.asarray(self.key_positions)
        if w.shape != pos.shape or w.ndim != 1:
            raise InvalidArgumentError("weights/key_positions must be matching vectors")
        if abs(float(w.sum()) - 1.0) > 1e-6:
            raise InvalidArgumentError("weights must sum to 1 within 1e-6")
        if (w < 0).any():
            raise InvalidArgumentError("weights must be non-negative")
        if pos.size > 1 and not (np.diff(pos) > 0).all():
            raise InvalidArgumentError("key_positions must be strictly increasing")


def _dev64(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(_dev())


def pool_presoftmax(q_tile) -> np.ndarray:
    """tiles.py:92-97: mean of the tile's query vectors, fp64 -> fp32."""
    q = np.asarray(q_tile)
    if q.ndim != 2 or q.shape[0] < 1:
        raise InvalidArgumentError("q_tile must be a non-empty [T][d] array")
    return _dev64(q).mean(dim=0).to(torch.float32).cpu().numpy()


def pool_postsoftmax(rows) -> np.ndarray:
    """tiles.py:100-114: mean of per-query distributions, shorter rows
    zero-extended to the longest support."""
    rows = [np.asarray(r) for r in rows]
    if not rows:
        raise InvalidArgumentError("cannot pool an empty tile")
    width = max(r.shape[0] for r in rows)
    acc = torch.zeros(width, dtype=torch.float64, device=_dev())
    for r in rows:
        acc[: r.shape[0]] += _dev64(r)
    return (acc / len(rows)).to(torch.float32).cpu().numpy()


def layer_distribution(P) -> np.ndarray:
    """metrics.py:97-102: mean of the per-head distributions [Hq][N][N] -> [N][N]."""
    P = np.asarray(P)
    if P.ndim != 3:
        raise InvalidArgumentError("P must be [Hq][N][N]")
    return _dev64(P).mean(dim=0).to(torch.float32).cpu().numpy()


def mass_coverage(P, k: int, per_row: bool = False) -> np.ndarray:
    """metrics.py:80-94: attention mass captured by each row's top-k keys."""
    if k < 1:
        raise InvalidArgumentError(f"k must be >= 1, got {k}")
    P = np.asarray(P)
    if P.ndim == 2:
        P = P[None]
    take = min(k, P.shape[-1])
    t = torch.from_numpy(np.ascontiguousarray(P)).to(_dev())
    top = torch.topk(t, take, dim=-1, sorted=False).values.to(torch.float64)
    cov = top.sum(dim=-1)
    out = cov.to(torch.float32) if per_row else cov.mean(dim=-1).to(torch.float32)
    return out.cpu().numpy()


def sim_score(p_b, I_a, I_b) -> float:
    """metrics.py:111-131: mass of p_b on I_a relative to its own Top-k set I_b."""
    from .exceptions import UndefinedScoreError
    idx_a = np.asarray(I_a.indices if hasattr(I_a, "indices") else I_a, dtype=np.int64)
    idx_b = np.asarray(I_b.indices if hasattr(I_b, "indices") else I_b, dtype=np.int64)
    if idx_a.size != idx_b.size or idx_a.size == 0:
        raise InvalidArgumentError(
            f"index sets must be non-empty and equal-sized, got {idx_a.size} and {idx_b.size}")
    p = np.asarray(p_b, dtype=np.float64)
    if idx_a.max() >= p.size or idx_b.max() >= p.size:
        raise InvalidArgumentError("index set outside the distribution's support")
    pd = _dev64(p)
    num = float(pd[torch.from_numpy(idx_a).to(pd.device)].sum())
    den = float(pd[torch.from_numpy(idx_b).to(pd.device)].sum())
    if den == 0.0:
        raise UndefinedScoreError("distribution carries no mass on its own Top-k set")
    return float(np.float32(num / den))


def pooled_all_heads_topk(group_dists, k: int, tile_id: int = 0) -> TopKIndexSet:
    """heads.py:155-171: shared Top-k set of the mean of per-kv-head pooled
    distributions (kv_head recorded as -1), via the exact Top-k kernel."""
    g = np.asarray(group_dists)
    if g.ndim == 1:
        g = g[None]
    pooled = _dev64(g).mean(dim=0).cpu().numpy()
    return oracle_topk_indices(pooled, k, kv_head=-1, tile_id=tile_id)


def topk_table(arr, take: int) -> np.ndarray:
    """ranking.py:14-25: indices of the ``take`` largest entries along the
    last axis, ordered by (value descending, index ascending) -- a stable
    device sort of the negated values."""
    a = np.asarray(arr)
    take = min(int(take), a.shape[-1])
    t = torch.from_numpy(np.ascontiguousarray(a)).to(_dev())
    order = torch.sort(-t, dim=-1, stable=True).indices[..., :take]
    return order.cpu().numpy()


def topk_tables(P, k: int) -> np.ndarray:
    """heads.py:62-64: per-kv-head, per-token Top-k index tables [Hkv][N][min(k, N)]."""
    P = np.asarray(P)
    return topk_table(P, min(k, P.shape[-1]))


def group_distributions(trace, layer: int, P=None) -> np.ndarray:
    """heads.py:50-59: per-kv-head, per-token distributions (the mean of the
    group's query-head rows of P, fp64 -> fp32) [Hkv][N][N]; P from the
    device dense pass when not given."""
    from .calibration import layer_probs
    Pd = layer_probs(trace, layer) if P is None else torch.from_numpy(np.ascontiguousarray(P)).to(_dev())
    Hq, N = Pd.shape[0], Pd.shape[1]
    Hkv = trace.num_kv_heads
    return Pd.double().view(Hkv, Hq // Hkv, N, Pd.shape[2]).mean(dim=1).float().cpu().numpy()


def _token_topk(pooled, k: int):
    """metrics.py:133-149: per-token Top-k over the causal rows of a pooled
    [N][N] distribution: (idx [N][take] padded with -1, valid [N][take],
    den [N] = each row's fp64 mass on its own set)."""
    pooled = np.asarray(pooled)
    N = pooled.shape[0]
    take = min(k, N)
    order = torch.from_numpy(topk_table(pooled, take)).to(_dev())
    ar = torch.arange(take, device=order.device)
    valid = ar[None, :] < torch.clamp(torch.arange(N, device=order.device) + 1, max=take)[:, None]
    pd = torch.from_numpy(np.ascontiguousarray(pooled)).to(_dev()).double()
    gathered = torch.gather(pd, 1, torch.where(valid, order, torch.zeros_like(order)))
    den = torch.where(valid, gathered, torch.zeros_like(gathered)).sum(dim=1)
    idx = torch.where(valid, order, torch.full_like(order, -1))
    return idx.cpu().numpy(), valid.cpu().numpy(), den.cpu().numpy()


def head_similarity_from_dists(Pa, Pb, k: int = 64, token_agg: str = "mean", idx_a=None) -> np.ndarray:
    """heads.py:67-108 with the reference's signature: [Hkv][Hkv] reuse
    scores from two layers' per-kv-head distributions (numpy, as from
    group_distributions) or the anchor's Top-k tables ``idx_a``.  The
    masked sums run in the kscd_masked_mass kernel (fp64)."""
    from . import calibration as cal
    cal._check_agg(token_agg)
    Db = torch.from_numpy(np.ascontiguousarray(Pb, dtype=np.float32)).to(_dev())
    Hkv, N = Db.shape[0], Db.shape[1]
    take = min(k, N)
    if idx_a is None:
        idx, cnt = cal._token_sets(torch.from_numpy(np.ascontiguousarray(Pa, dtype=np.float32)).to(_dev()), k)
    else:
        # only the first min(r + 1, take) entries of each table row count
        # (heads.py:86); the masked sum does not depend on their order
        idx = torch.from_numpy(np.ascontiguousarray(idx_a, dtype=np.int32)[..., :take]).to(_dev())
        cnt = torch.clamp(torch.arange(N, device=idx.device, dtype=torch.int32) + 1, max=take).repeat(Hkv, 1)
        idx = torch.where(torch.arange(take, device=idx.device)[None, None, :] < cnt[..., None], idx,
                          torch.zeros_like(idx))
    idx_b, cnt_b = cal._token_sets(Db, k)
    num = cal.masked_mass(Db, idx, cnt, N).cpu().numpy()
    own = cal.masked_mass(Db, idx_b, cnt_b, N).cpu().numpy()
    den = np.stack([own[j, j] for j in range(Hkv)])
    return cal._aggregate_scores(num, den, token_agg)
