"""GPU acceleration of the reference's offline calibration (SURVEY.md 8(f)
rank 3): the planning similarity matrix, head similarity and head maps, and
the plan builder on top of them.

The reference computes these with Python loops over (layer pair, head pair,
tile) on numpy copies of dense P (metrics.py:226-295, heads.py:67-143,
pipeline.py:31-118) -- 2.7 s and 3.8 s on the 4-layer config-1 trace.  Here
every heavy step stays on the device and reuses the engine's kernels:

    P [Hq][N][N]          kscd_dense_prefill (LSE) + kscd_dense_probs
    pooled distributions  kscd_pool_tiles (fp64 sums over heads x tile rows;
                          per-token group distributions are 1-row tiles)
    Top-k sets            kscd_topk (exact radix select, ties -> smaller
                          index, so the SETS equal argsort(kind="stable"))
    num / den masses      kscd_masked_mass (fp64 gather-sums, calib.cu)

and only [I][J][rows] masses come back for the small aggregations (token /
tile means, argmax head maps), which follow the reference's fp32 rounding of
each score.  The anchor DP (planner.py:84-128) and the layer importance
weights (metrics.py:338-396) are O(L^2) host arithmetic and are restated
here so build_plan runs without the reference package.

Pooled distributions are sums, not means: every score is a ratio of two
masses of the same (head, tile) distribution, so the constant 1/(G*rows)
cancels.  No CPU fallback: every entry point needs the CUDA library.
"""

import hashlib
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple, Union

import numpy as np
import torch

from . import _lib, ops
from .compat import _check_head_dim, _dev, _layer, _probs, _scale
from .exceptions import InvalidArgumentError, UnsupportedOperationError
from .host_types import (DECODE, MODE_ALL_HEADS_POOLED, MODE_IDENTITY, MODE_REMAPPED, POOL_POST, PREFILL,
                         AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy)

PLANNING_K = 64                      # metrics.py:36
TOKEN_AGG_MEAN, TOKEN_AGG_MIN = "mean", "min"
MODE_DIAGNOSTIC, MODE_PLANNING = "diagnostic", "planning"
DEFAULT_ANCHOR_BUDGET = 5            # planner.py:21
DEFAULT_TILE_SIZE = 128


@dataclass
class SimilarityMatrix:
    """metrics.py:43-68 (same fields and digest)."""

    S: np.ndarray
    k_used: int
    token_aggregation: str
    prompt_aggregation: str = "mean"
    importance_weighted: bool = False
    mode: str = MODE_DIAGNOSTIC
    prompt_count: int = 1
    undefined_scores: int = 0

    @property
    def num_layers(self) -> int:
        return self.S.shape[0]

    def digest(self) -> str:
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(self.S, dtype=np.float32).tobytes())
        h.update(f"{self.k_used}|{self.token_aggregation}|{self.mode}|{self.importance_weighted}".encode())
        return h.hexdigest()[:16]


@dataclass
class LayerImportance:
    """metrics.py:71-77."""

    w: np.ndarray
    source_prompt_count: int
    skipped_tokens: int = 0


def _as_traces(traces) -> list:
    """metrics.py:171-189."""
    if hasattr(traces, "num_layers"):
        return [traces]
    traces = list(traces)
    if not traces:
        raise InvalidArgumentError("at least one trace is required")
    L = traces[0].num_layers
    for t in traces[1:]:
        if t.num_layers != L:
            raise InvalidArgumentError(f"traces disagree on layer count: {t.num_layers} != {L}")
        if (t.num_query_heads, t.num_kv_heads) != (traces[0].num_query_heads, traces[0].num_kv_heads):
            raise InvalidArgumentError("traces disagree on head counts")
    return traces


def _check_agg(token_agg: str) -> None:
    if token_agg not in (TOKEN_AGG_MEAN, TOKEN_AGG_MIN):
        raise InvalidArgumentError(f"unknown token aggregation {token_agg!r}")


# ------------------------------------------------------------ device steps
def layer_probs(trace, layer: int) -> torch.Tensor:
    """dense_attention's P (attention.py:106-144) on the device: [Hq][N][N]."""
    q, k, v = _layer(trace, layer)
    _, lse = ops.dense_prefill(q, k, v, scale=_scale(trace))
    return _probs(q, k, lse, True, trace.head_dim)


def pooled_tiles(P: torch.Tensor, num_kv_heads: int, starts: Sequence[int], ends: Sequence[int],
                 all_heads: bool = False) -> torch.Tensor:
    """fp64-accumulated sums of P over the heads of each kv group (or all
    heads) and the rows [start, end) of each tile, columns < end (zeros
    beyond): [Hkv or 1][T][stride] fp32 (kscd_pool_tiles)."""
    Hq, N = P.shape[0], P.shape[1]
    T = len(starts)
    dev = P.device
    stride = (N + 3) // 4 * 4
    st = torch.tensor(list(starts), dtype=torch.int32, device=dev)
    en = torch.tensor(list(ends), dtype=torch.int32, device=dev)
    rows = 1 if all_heads else num_kv_heads
    out = torch.zeros(rows, T, stride, dtype=torch.float32, device=dev)
    pp = _lib.PoolTilesParams(num_q_heads=Hq, num_kv_heads=num_kv_heads, head_dim=128, seq_len=N, num_tiles=T,
                              tile_starts=st.data_ptr(), tile_ends=en.data_ptr(), pooling=0,
                              all_heads=1 if all_heads else 0, probs=P.data_ptr(), pooled=out.data_ptr(),
                              pooled_stride=stride)
    _lib.call("kscd_pool_tiles", pp, ops._stream())
    return out


def group_distributions(trace, layer: int, P: Optional[torch.Tensor] = None) -> torch.Tensor:
    """heads.py:50-59 up to the factor G: per-kv-head, per-token pooled
    rows [Hkv][N][stride] (one 1-row tile per token)."""
    if P is None:
        P = layer_probs(trace, layer)
    N = P.shape[1]
    return pooled_tiles(P, trace.num_kv_heads, range(N), range(1, N + 1))


def row_topk(D: torch.Tensor, k: int, lengths: Sequence[int]) -> Tuple[torch.Tensor, torch.Tensor]:
    """Top-min(k, len) set of every row of D [H][R][stride] (row r of each
    head has support lengths[r]): (idx [H][R][k_cap] ascending, counts [H][R])."""
    H, R, stride = D.shape
    lens = torch.tensor(list(lengths), dtype=torch.int32, device=D.device)
    k_cap = max(1, min(k, int(max(lengths))))
    idx, cnt = ops.topk(D.reshape(H * R, stride), int(k), lengths=lens.repeat(H), k_cap=k_cap)
    return idx.reshape(H, R, k_cap), cnt.reshape(H, R)


def masked_mass(dist: torch.Tensor, idx: torch.Tensor, counts: torch.Tensor, dist_len: int) -> torch.Tensor:
    """mass[i][j][r] = fp64 sum of dist[j][r][idx[i][r][t]], t < counts[i][r]
    (kscd_masked_mass).  dist [J][R][stride] fp32, idx [I][R][k_cap]."""
    J, R, stride = dist.shape
    I, R2, k_cap = idx.shape
    if R2 != R:
        raise InvalidArgumentError("index sets and distributions disagree on the row count")
    idx = idx.contiguous()
    counts = counts.to(torch.int32).contiguous()
    out = torch.empty(I, J, R, dtype=torch.float64, device=dist.device)
    p = _lib.MaskedMassParams(num_sets=I, num_dists=J, rows=R, dist=dist.data_ptr(),
                              dist_stride_head=dist.stride(0), dist_stride_row=dist.stride(1), dist_len=stride,
                              indices=idx.data_ptr(), counts=counts.data_ptr(), k_cap=k_cap, mass=out.data_ptr())
    _lib.call("kscd_masked_mass", p, ops._stream())
    return out


def _token_sets(D: torch.Tensor, k: int):
    N = D.shape[1]
    return row_topk(D, k, range(1, N + 1))


# ----------------------------------------------------------- head similarity
def _aggregate_scores(num: np.ndarray, den: np.ndarray, token_agg: str) -> np.ndarray:
    """heads.py:100-108 for every (i, j): scores fp32(num / den) over rows
    with den != 0, then the fp64 mean or the min (0 with no defined row)."""
    I, J, _ = num.shape
    hs = np.zeros((I, J), np.float64)
    for j in range(J):
        ok = den[j] != 0.0
        for i in range(I):
            s = (num[i, j][ok] / den[j][ok]).astype(np.float32)
            if s.size == 0:
                hs[i, j] = 0.0
            elif token_agg == TOKEN_AGG_MEAN:
                hs[i, j] = s.mean(dtype=np.float64)
            else:
                hs[i, j] = s.min()
    return hs


def head_similarity_from_dists(idx_a, cnt_a, Db: torch.Tensor, k: int = PLANNING_K,
                               token_agg: str = TOKEN_AGG_MEAN) -> np.ndarray:
    """heads.py:67-108 on device tensors: entry [i][j] scores anchor head
    i's per-token Top-k sets (idx_a/cnt_a from _token_sets) against reuse
    head j's own, on reuse head j's distribution Db."""
    _check_agg(token_agg)
    N = Db.shape[1]
    idx_b, cnt_b = _token_sets(Db, k)
    num = masked_mass(Db, idx_a, cnt_a, N).cpu().numpy()
    own = masked_mass(Db, idx_b, cnt_b, N).cpu().numpy()
    den = np.stack([own[j, j] for j in range(Db.shape[0])])
    return _aggregate_scores(num, den, token_agg)


def head_similarity(traces, anchor_layer: int, reuse_layer: int, k: int = PLANNING_K,
                    token_agg: str = TOKEN_AGG_MEAN) -> np.ndarray:
    """heads.py:111-126: [Hkv][Hkv], averaged over prompts."""
    traces = _as_traces(traces)
    per = []
    for t in traces:
        Da = group_distributions(t, anchor_layer)
        Db = Da if reuse_layer == anchor_layer else group_distributions(t, reuse_layer)
        idx_a, cnt_a = _token_sets(Da, k)
        per.append(head_similarity_from_dists(idx_a, cnt_a, Db, k, token_agg))
    return np.mean(per, axis=0)


def compute_head_map(simmat, reuse_layer: int = -1, anchor_layer: int = -1) -> HeadMap:
    """heads.py:129-143: argmax of each column (ties -> smaller anchor head)."""
    simmat = np.asarray(simmat)
    if simmat.ndim != 2 or simmat.shape[0] != simmat.shape[1]:
        raise InvalidArgumentError("head similarity matrix must be square")
    return HeadMap(reuse_layer, anchor_layer, [int(m) for m in simmat.argmax(axis=0)], MODE_REMAPPED)


def compute_head_maps(traces, anchors: Sequence[int], k: int = PLANNING_K,
                      head_map_mode: str = MODE_REMAPPED) -> Dict[int, HeadMap]:
    """pipeline.py:31-73: a head map for every reuse layer against its most
    recent anchor; each layer's group distributions are computed once."""
    traces = _as_traces(traces)
    L, Hkv = traces[0].num_layers, traces[0].num_kv_heads
    anchor_set = set(int(a) for a in anchors)
    maps: Dict[int, HeadMap] = {}
    if head_map_mode == MODE_IDENTITY:
        for layer in range(L):
            if layer not in anchor_set:
                a = max(x for x in anchors if x <= layer)
                maps[layer] = HeadMap(layer, a, list(range(Hkv)), MODE_IDENTITY)
        return maps
    if head_map_mode != MODE_REMAPPED:
        raise InvalidArgumentError(f"unknown head-map mode {head_map_mode!r}")
    srt = sorted(anchor_set)
    for n, anchor in enumerate(srt):
        end = srt[n + 1] if n + 1 < len(srt) else L
        reuse = list(range(anchor + 1, end))
        if not reuse:
            continue
        sets_a = [_token_sets(group_distributions(t, anchor), k) for t in traces]
        for layer in reuse:
            per = [head_similarity_from_dists(ia, ca, group_distributions(t, layer), k)
                   for t, (ia, ca) in zip(traces, sets_a)]
            maps[layer] = compute_head_map(np.mean(per, axis=0), reuse_layer=layer, anchor_layer=anchor)
    return maps


# ------------------------------------------------------ similarity matrices
def _tiles(N: int, phase: str, tile_size: int) -> Tuple[List[int], List[int]]:
    if phase == PREFILL:
        s = list(range(0, N, tile_size))
        return s, [min(x + tile_size, N) for x in s]
    if phase == DECODE:
        return list(range(N)), list(range(1, N + 1))
    raise InvalidArgumentError(f"unknown phase {phase!r}")


def _planning_matrix(trace, k: int, token_agg: str, tile_size: int, phase: str) -> Tuple[np.ndarray, int]:
    """metrics.py:226-295 for one trace."""
    L, Hkv, N = trace.num_layers, trace.num_kv_heads, trace.seq_len
    starts, ends = _tiles(N, phase, tile_size)
    dists, sets, dens = [], [], []
    for layer in range(L):
        D = pooled_tiles(layer_probs(trace, layer), Hkv, starts, ends)      # [Hkv][T][stride]
        idx, cnt = row_topk(D, k, ends)
        own = masked_mass(D, idx, cnt, D.shape[2])
        dists.append(D), sets.append((idx, cnt))
        dens.append(torch.stack([own[j, j] for j in range(Hkv)]).cpu().numpy())   # [Hkv][T]
    S = np.zeros((L, L), np.float32)
    undefined = 0
    for b in range(L):
        den = dens[b]
        ok = den != 0.0
        for a in range(b + 1):
            num = masked_mass(dists[b], sets[a][0], sets[a][1], dists[b].shape[2]).cpu().numpy()  # [i][j][t]
            with np.errstate(divide="ignore", invalid="ignore"):
                sc = (num / den[None]).astype(np.float32).astype(np.float64)          # pair_score
            hs = np.zeros((Hkv, Hkv))
            for i in range(Hkv):
                for j in range(Hkv):
                    v = sc[i, j][ok[j]]
                    hs[i, j] = float(np.mean(v)) if v.size else 0.0
            hm = hs.argmax(axis=0)
            per_tile = []
            for t in range(len(starts)):
                kept = [sc[hm[j], j, t] for j in range(Hkv) if ok[j, t]]
                undefined += Hkv - len(kept)
                if kept:
                    per_tile.append(float(np.mean(kept)))
            if per_tile:
                S[a, b] = np.float32(np.mean(per_tile) if token_agg == TOKEN_AGG_MEAN else np.min(per_tile))
    return S, undefined


def _diagnostic_matrix(trace, k: int, token_agg: str) -> Tuple[np.ndarray, int]:
    """metrics.py:205-223 for one trace: per-token distributions averaged
    over all query heads, per-token Top-k sets, scores of layer b's
    distribution on layer a's sets."""
    L, N = trace.num_layers, trace.seq_len
    S = np.zeros((L, L), np.float32)
    undefined = 0
    sets = []
    for b in range(L):
        D = pooled_tiles(layer_probs(trace, b), trace.num_kv_heads, range(N), range(1, N + 1), all_heads=True)
        idx_b, cnt_b = _token_sets(D, k)
        sets.append((idx_b, cnt_b))
        den = masked_mass(D, idx_b, cnt_b, D.shape[2]).cpu().numpy()[0, 0]
        ok = den != 0.0
        for a in range(b + 1):
            num = masked_mass(D, sets[a][0], sets[a][1], D.shape[2]).cpu().numpy()[0, 0]
            undefined += int((~ok).sum())
            s = (num[ok] / den[ok]).astype(np.float32)
            if s.size == 0:
                S[a, b] = 0.0
            elif token_agg == TOKEN_AGG_MEAN:
                S[a, b] = np.float32(s.mean(dtype=np.float64))
            else:
                S[a, b] = s.min()
    return S, undefined


def similarity_matrix(traces, k: int = PLANNING_K, token_agg: str = TOKEN_AGG_MEAN, mode: str = MODE_DIAGNOSTIC,
                      tile_size: int = DEFAULT_TILE_SIZE, phase: str = PREFILL) -> SimilarityMatrix:
    """metrics.py:298-335: cross-layer reuse scores averaged over prompts."""
    traces = _as_traces(traces)
    if k < 1:
        raise InvalidArgumentError(f"k must be >= 1, got {k}")
    _check_agg(token_agg)
    mats, undefined = [], 0
    for t in traces:
        _check_head_dim(t.head_dim)
        if mode == MODE_DIAGNOSTIC:
            S, und = _diagnostic_matrix(t, k, token_agg)
        elif mode == MODE_PLANNING:
            S, und = _planning_matrix(t, k, token_agg, tile_size, phase)
        else:
            raise InvalidArgumentError(f"unknown similarity mode {mode!r}")
        mats.append(S.astype(np.float64))
        undefined += und
    return SimilarityMatrix(S=np.mean(mats, axis=0).astype(np.float32), k_used=k, token_aggregation=token_agg,
                            mode=mode, prompt_count=len(traces), undefined_scores=undefined)


# -------------------------------------------------- host planning arithmetic
def layer_importance(traces, norm_floor: float = 1e-12) -> LayerImportance:
    """metrics.py:338-377: mean over tokens and prompts of 1 - cos(X, Y)."""
    traces = _as_traces(traces)
    missing = [t.prompt_id for t in traces if getattr(t, "X", None) is None or getattr(t, "Y", None) is None]
    if missing:
        raise UnsupportedOperationError("trace(s) carry no attention input/output hidden states: "
                                        + ", ".join(repr(m) for m in missing))
    L = traces[0].num_layers
    total = np.zeros(L, np.float64)
    count = np.zeros(L, np.int64)
    skipped = 0
    for t in traces:
        for layer in range(L):
            x = np.asarray(t.X[layer], np.float64)
            y = np.asarray(t.Y[layer], np.float64)
            nx, ny = np.linalg.norm(x, axis=1), np.linalg.norm(y, axis=1)
            ok = (nx > norm_floor) & (ny > norm_floor)
            skipped += int((~ok).sum())
            cos = np.clip((x[ok] * y[ok]).sum(axis=1) / (nx[ok] * ny[ok]), -1.0, 1.0)
            total[layer] += (1.0 - cos).sum()
            count[layer] += int(ok.sum())
    w = np.where(count > 0, total / np.maximum(count, 1), 0.0)
    return LayerImportance(w=w.astype(np.float64), source_prompt_count=len(traces), skipped_tokens=skipped)


def apply_importance(S: SimilarityMatrix, importance: LayerImportance) -> SimilarityMatrix:
    """metrics.py:380-396: S'[i][j] = w[j] S[i][j]."""
    if importance.w.shape[0] != S.num_layers:
        raise InvalidArgumentError(f"importance has {importance.w.shape[0]} layers, matrix has {S.num_layers}")
    return SimilarityMatrix(S=(S.S.astype(np.float64) * importance.w[None, :]).astype(np.float32), k_used=S.k_used,
                            token_aggregation=S.token_aggregation, prompt_aggregation=S.prompt_aggregation,
                            importance_weighted=True, mode=S.mode, prompt_count=S.prompt_count,
                            undefined_scores=S.undefined_scores)


def _matrix_of(S) -> np.ndarray:
    arr = S.S if isinstance(S, SimilarityMatrix) else np.asarray(S)
    if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
        raise InvalidArgumentError("similarity matrix must be square")
    return arr.astype(np.float64)


def objective(S, anchors: Sequence[int]) -> float:
    """planner.py:56-73."""
    mat = _matrix_of(S)
    L = mat.shape[0]
    anchors = [int(a) for a in anchors]
    if not anchors or anchors[0] != 0:
        raise InvalidArgumentError("anchors must start at layer 0")
    if any(b <= a for a, b in zip(anchors, anchors[1:])) or anchors[-1] >= L:
        raise InvalidArgumentError("anchors must be strictly increasing and < L")
    return float(sum(mat[a, a:end].sum() for a, end in zip(anchors, anchors[1:] + [L])))


def select_anchors(S, M: int) -> AnchorPlanCore:
    """planner.py:84-128: the optimal M-anchor set by DP over suffixes,
    ties to the lexicographically smallest set (exact float comparison
    against the stored optimum)."""
    mat = _matrix_of(S)
    L = mat.shape[0]
    if not (1 <= M <= L):
        raise InvalidArgumentError(f"anchor budget {M} outside [1, {L}]")
    cum = np.zeros((L, L + 1), np.float64)
    cum[:, 1:] = np.cumsum(mat, axis=1)
    seg = cum - cum[np.arange(L), np.arange(L)][:, None]
    suffix = np.full((M + 1, L), -np.inf, np.float64)
    suffix[1] = seg[np.arange(L), L]
    for m in range(2, M + 1):
        for i in range(L - m + 1):
            lo, hi = i + 1, L - m + 2
            suffix[m, i] = (seg[i, lo:hi] + suffix[m - 1, lo:hi]).max()
    anchors, i, m = [0], 0, M
    while m > 1:
        lo, hi = i + 1, L - m + 2
        cand = seg[i, lo:hi] + suffix[m - 1, lo:hi]
        j = lo + int(np.flatnonzero(cand == suffix[m, i])[0])
        anchors.append(j)
        i, m = j, m - 1
    digest = S.digest() if isinstance(S, SimilarityMatrix) else ""
    return AnchorPlanCore(anchors, M, objective(mat, anchors), digest)


EXHAUSTIVE_LIMIT = 10**6     # planner.py:128


def exhaustive_select(S, M: int) -> AnchorPlanCore:
    """planner.py:131-160: brute force over every anchor set in lexicographic
    order, keeping the first maximum (select_anchors' tie-break)."""
    import math
    from itertools import combinations
    mat = _matrix_of(S)
    L = mat.shape[0]
    if not (1 <= M <= L):
        raise InvalidArgumentError(f"anchor budget {M} outside [1, {L}]")
    n_sets = math.comb(L - 1, M - 1)
    if n_sets > EXHAUSTIVE_LIMIT:
        raise UnsupportedOperationError(f"{n_sets} candidate sets exceed the exhaustive bound {EXHAUSTIVE_LIMIT}")
    best, best_value = None, -np.inf
    for rest in combinations(range(1, L), M - 1):
        anchors = [0, *rest]
        value = objective(mat, anchors)
        if value > best_value:
            best, best_value = anchors, value
    return AnchorPlanCore(best, M, best_value, S.digest() if isinstance(S, SimilarityMatrix) else "")


def build_plan(traces, budget: int = DEFAULT_ANCHOR_BUDGET, k: int = PLANNING_K, token_agg: str = TOKEN_AGG_MIN,
               tile_size: int = DEFAULT_TILE_SIZE, pooling: str = POOL_POST, mode: str = MODE_REMAPPED,
               k_policy: Optional[KBudgetPolicy] = None, use_importance: bool = True,
               similarity: Optional[SimilarityMatrix] = None) -> AnchorPlan:
    """pipeline.py:76-118 with the similarity matrix and head maps on the GPU."""
    traces = _as_traces(traces)
    if similarity is None:
        similarity = similarity_matrix(traces, k=k, token_agg=token_agg, mode=MODE_PLANNING, tile_size=tile_size)
    if use_importance and all(getattr(t, "X", None) is not None and getattr(t, "Y", None) is not None
                              for t in traces):
        similarity = apply_importance(similarity, layer_importance(traces))
    core = select_anchors(similarity, budget)
    head_maps: Dict[int, HeadMap] = {}
    if mode == MODE_REMAPPED:
        head_maps = compute_head_maps(traces, core.anchors, k=k)
    elif mode != MODE_ALL_HEADS_POOLED:
        raise InvalidArgumentError(f"unknown plan mode {mode!r}")
    plan = AnchorPlan(core=core, head_maps=head_maps, pooling=pooling, k_policy=k_policy or KBudgetPolicy(),
                      tile_size=tile_size, mode=mode)
    plan.validate(traces[0].num_layers, traces[0].num_kv_heads)
    return plan
