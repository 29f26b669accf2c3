"""CPU oracle for the Kascade anchor/reuse attention path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's hot path
(`/root/reference/pkg/src/kascade`, the public `kascade` 0.1.0 API).  It exists
so that parity tests, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` have an independent checker that
travels to the GPU box (the reference tree does not).  Nothing in the product
package (`paper_2512_16391_b200`) imports it; the product path has no CPU
fallback and fails loudly when its CUDA library is missing.

Parity is PINNED: ``tests/golden/make_golden.py`` runs the reference itself
(imported from /root/reference in the dev container) on seeded inputs and
freezes its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks every function below against those vectors (bit-exact for index sets
and, where the arithmetic order is the same, for floats).

Every function cites the reference file:line it restates.  Arrays are float32
at the interface like the reference; the normaliser accumulates in float64
exactly where the reference does.
"""

from __future__ import annotations

import math
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

Key = Tuple[int, int]  # (kv_head, tile_id)

POST, PRE = "post", "pre"
REMAPPED, ALL_HEADS_POOLED = "remapped", "all_heads_pooled"


# --------------------------------------------------------------------------
# inputs
# --------------------------------------------------------------------------

def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even), returned as
    float32.  The engine computes in bf16; parity inputs are fed to both sides
    already bf16-representable."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(a.shape)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """Upper 16 bits of bf16-representable float32 values (uint16)."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    return (a.view(np.uint32) >> 16).astype(np.uint16)


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint32) << 16).view(np.float32)


def _unit(a: np.ndarray) -> np.ndarray:
    return a / np.linalg.norm(a, axis=-1, keepdims=True)


def synth_qkv(L: int, Hq: int, Hkv: int, d: int, N: int, seed: int = 0,
              rho: float = 1.0, perms: Optional[Sequence[Sequence[int]]] = None,
              tau: float = 4.0, qcorr: float = 0.85, tau0_scale: float = 1.0):
    """Heavy-tailed synthetic Q/K/V, restating ``generate_synthetic``
    (traceio.py:218-273) draw for draw so that identical arguments give
    identical bytes (pinned by SHA-256 in tests/golden/golden.json).
    X/Y hidden states are not generated (they are drawn after Q/K/V,
    traceio.py:275-285, so omitting them does not perturb Q/K/V)."""
    G = Hq // Hkv
    rng = np.random.default_rng(seed)
    kb = rng.standard_normal((Hkv, N, d))
    vb = rng.standard_normal((Hkv, N, d))
    gdir = _unit(rng.standard_normal((Hkv, d)))
    jit = _unit(rng.standard_normal((Hq, N, d)))
    heads = np.arange(Hq) // G
    dirs = _unit(np.sqrt(qcorr) * gdir[heads][:, None, :] + np.sqrt(1.0 - qcorr) * jit)
    perms = [list(range(Hkv))] * L if perms is None else [list(p) for p in perms]
    mix = np.sqrt(1.0 - rho * rho)
    Q = np.empty((L, Hq, N, d), np.float32)
    K = np.empty((L, Hkv, N, d), np.float32)
    V = np.empty((L, Hkv, N, d), np.float32)
    for l in range(L):
        kn = rng.standard_normal((Hkv, N, d))
        vn = rng.standard_normal((Hkv, N, d))
        t = tau * (tau0_scale if l == 0 else 1.0)
        p = perms[l]
        for g in range(Hkv):
            K[l, g] = (rho * kb[p[g]] + mix * kn[g]).astype(np.float32)
            V[l, g] = (rho * vb[p[g]] + mix * vn[g]).astype(np.float32)
            src = p[g] * G + np.arange(G)
            Q[l, g * G:(g + 1) * G] = (t * np.sqrt(d) * dirs[src]).astype(np.float32)
    return Q, K, V


def random_qkv(seed: int, L: int, Hq: int, Hkv: int, d: int, N: int):
    """iid-normal fp32 Q/K/V in the draw order of the reference tests'
    ``random_trace`` (pkg/tests/conftest.py:15-31)."""
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((L, Hq, N, d)).astype(np.float32)
    K = rng.standard_normal((L, Hkv, N, d)).astype(np.float32)
    V = rng.standard_normal((L, Hkv, N, d)).astype(np.float32)
    return Q, K, V


# --------------------------------------------------------------------------
# budgets and tiles
# --------------------------------------------------------------------------

def k_budget(fraction: float, k_min: int, n: int) -> int:
    """tiles.py:81-89: floor the fp64 product, clamp below by k_min and
    above by the number of visible keys."""
    if n < 1:
        raise ValueError("n must be >= 1")
    return min(max(math.floor(fraction * n), k_min), n)


def prefill_tiles(N: int, tile: int) -> List[Tuple[int, int, int]]:
    """(start, end, tile_id) of tiles.py:137-144 for one kv head."""
    return [(s, min(s + tile, N), i) for i, s in enumerate(range(0, N, tile))]


def decode_tiles(N: int) -> List[Tuple[int, int, int]]:
    """tiles.py:145-150: one single-row tile per token, tile_id = token."""
    return [(t, t + 1, t) for t in range(N)]


# --------------------------------------------------------------------------
# dense attention and the Top-k contract
# --------------------------------------------------------------------------

def masked_softmax(s: np.ndarray, vis: np.ndarray) -> np.ndarray:
    """attention.py:93-103.  exp in the score precision, float64 row sum,
    division back in the score precision; masked entries are exact zeros."""
    z = np.where(vis, s, -np.inf)
    e = np.exp(z - z.max(axis=1, keepdims=True))
    e[~vis] = 0.0
    tot = e.sum(axis=1, keepdims=True, dtype=np.float64)
    return np.divide(e, tot, dtype=e.dtype)


def softmax_vec(scores: np.ndarray) -> np.ndarray:
    """attention.py:77-90 (float64 internally, float32 result)."""
    s = np.asarray(scores, dtype=np.float64)
    e = np.exp(s - s.max())
    return (e / e.sum()).astype(np.float32)


def _scale(d: int) -> np.float32:
    return np.float32(1.0 / math.sqrt(d))


def dense_layer(Ql: np.ndarray, Kl: np.ndarray, Vl: np.ndarray, causal: bool = True):
    """attention.py:106-144 for one layer: Ql [Hq][N][d], Kl/Vl [Hkv][N][d]
    -> (P [Hq][N][N], Y [Hq][N][d]); query head h reads kv head h // G
    (trace.py:38-43)."""
    Hq, N, d = Ql.shape
    G = Hq // Kl.shape[0]
    vis = np.tril(np.ones((N, N), bool)) if causal else np.ones((N, N), bool)
    P = np.empty((Hq, N, N), np.float32)
    Y = np.empty((Hq, N, d), np.float32)
    for h in range(Hq):
        kk = Kl[h // G].astype(np.float32)
        P[h] = masked_softmax((Ql[h].astype(np.float32) @ kk.T) * _scale(d), vis)
        Y[h] = P[h] @ Vl[h // G].astype(np.float32)
    return P, Y


def topk_sorted(w: np.ndarray, k: int) -> np.ndarray:
    """attention.py:147-174: the k largest weights, ties to the smaller
    position (stable descending order), returned ascending as int64."""
    if k < 1:
        raise ValueError("k must be >= 1")
    w = np.asarray(w)
    sel = np.argsort(-w, kind="stable")[: min(k, w.size)]
    return np.sort(sel).astype(np.int64)


# --------------------------------------------------------------------------
# pooling, selection and routing (runner.py)
# --------------------------------------------------------------------------

def pooled_post(P: np.ndarray, g: int, G: int, start: int, end: int) -> np.ndarray:
    """runner.py:148-152: float64 mean over the group's heads and the tile's
    rows of the post-softmax rows, truncated at the causal bound ``end``."""
    return P[g * G:(g + 1) * G, start:end, :end].mean(axis=(0, 1), dtype=np.float64)


def pooled_pre(Ql: np.ndarray, Kl: np.ndarray, g: int, G: int, start: int, end: int) -> np.ndarray:
    """runner.py:155-161: softmax of the float64 mean query of the tile
    against the keys below the causal bound."""
    d = Ql.shape[-1]
    qbar = Ql[g * G:(g + 1) * G, start:end].reshape(-1, d).mean(axis=0, dtype=np.float64)
    s = (Kl[g, :end].astype(np.float64) @ qbar) / math.sqrt(d)
    return softmax_vec(s).astype(np.float64)


def select(pooled: Dict[Key, np.ndarray], bounds: Dict[int, int], fraction: float,
           k_min: int, mode: str = REMAPPED, Hkv: Optional[int] = None) -> Dict[Key, np.ndarray]:
    """runner.py:179-207.  ``pooled`` maps (kv head, tile) to the pooled
    vector, ``bounds`` maps tile id to its causal bound.  In all-heads-pooled
    mode the kv-head vectors of a tile are averaged (np.mean) and one set is
    shared by every kv head."""
    out: Dict[Key, np.ndarray] = {}
    if mode == ALL_HEADS_POOLED:
        tids = sorted({t for (_, t) in pooled})
        for t in tids:
            heads = sorted(g for (g, tt) in pooled if tt == t)
            shared = topk_sorted(np.mean([pooled[(g, t)] for g in heads], axis=0),
                                 k_budget(fraction, k_min, bounds[t]))
            for g in range(Hkv if Hkv is not None else len(heads)):
                out[(g, t)] = shared
        return out
    for (g, t), w in pooled.items():
        out[(g, t)] = topk_sorted(w, k_budget(fraction, k_min, bounds[t]))
    return out


def route(anchor_sels: Dict[Key, np.ndarray], head_map: Optional[Sequence[int]],
          Hkv: int) -> Dict[Key, np.ndarray]:
    """runner.py:210-225: reuse kv head g borrows the anchor set of
    head_map[g] (identity when None) for the same tile id."""
    tids = {t for (_, t) in anchor_sels}
    return {(g, t): anchor_sels[(head_map[g] if head_map is not None else g, t)]
            for t in tids for g in range(Hkv)}


def sparse_tile(Ql, Kl, Vl, g: int, G: int, start: int, end: int, sel: np.ndarray,
                causal: bool = True, dense_P: Optional[np.ndarray] = None):
    """attention.py:228-252 for one (kv head, tile): each row r sees the
    prefix of ``sel`` that is <= r; the softmax renormalises over it; a row
    with an empty prefix outputs V[g][r] (diagonal fallback).  Returns
    (Y [G][T][d], mass [G][T], fallback rows as (head, row))."""
    d = Ql.shape[-1]
    T = end - start
    rows = np.arange(start, end)
    nvis = np.searchsorted(sel, rows, side="right") if causal else np.full(T, sel.size)
    vis = np.arange(sel.size)[None, :] < nvis[:, None]
    ks = np.asarray(Kl[g, sel], dtype=np.float32)
    vs = np.asarray(Vl[g, sel], dtype=np.float32)
    live = nvis > 0
    Y = np.zeros((G, T, d), np.float32)
    mass = np.zeros((G, T), np.float32)
    fb = []
    for j in range(G):
        h = g * G + j
        if sel.size and live.any():
            s = (Ql[h, rows[live]].astype(np.float32) @ ks.T) * _scale(d)
            Y[j, live] = masked_softmax(s, vis[live]) @ vs
            if dense_P is not None:
                dm = dense_P[h][rows[live]][:, sel].astype(np.float64)
                dm[~vis[live]] = 0.0
                mass[j, live] = dm.sum(axis=1).astype(np.float32)
        for i in np.nonzero(~live)[0]:
            Y[j, i] = Vl[g, rows[i]]
            fb.append((h, int(rows[i])))
    return Y, mass, fb


def sparse_layer(Ql, Kl, Vl, sels: Dict[Key, np.ndarray], tiles, causal=True, dense_P=None):
    """attention.py:185-253 over every (kv head, tile)."""
    Hq, N, d = Ql.shape
    Hkv = Kl.shape[0]
    G = Hq // Hkv
    Y = np.zeros((Hq, N, d), np.float32)
    mass = np.zeros((Hq, N), np.float32)
    fb: List[Tuple[int, int]] = []
    for g in range(Hkv):
        for (s, e, t) in tiles:
            if (g, t) not in sels:
                raise KeyError(f"no Top-k set for kv head {g}, tile {t}")
            sel = np.asarray(sels[(g, t)], dtype=np.int64)
            if causal and sel.size and sel[-1] >= e:
                raise ValueError("selection breaks the tile's causal bound")
            y, m, f = sparse_tile(Ql, Kl, Vl, g, G, s, e, sel, causal, dense_P)
            Y[g * G:(g + 1) * G, s:e] = y
            mass[g * G:(g + 1) * G, s:e] = m
            fb.extend(f)
    return Y, mass, fb


def rel_l2(a: np.ndarray, b: np.ndarray) -> float:
    """runner.py:140-145."""
    num = np.linalg.norm((a.astype(np.float64) - b.astype(np.float64)).ravel())
    den = np.linalg.norm(b.astype(np.float64).ravel())
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(num / den)


def layer_pooled(Ql, Kl, P, tiles, Hkv: int, pooling: str) -> Dict[Key, np.ndarray]:
    G = Ql.shape[0] // Hkv
    out = {}
    for g in range(Hkv):
        for (s, e, t) in tiles:
            out[(g, t)] = (pooled_post(P, g, G, s, e) if pooling == POST
                           else pooled_pre(Ql, Kl, g, G, s, e))
    return out


def run_kascade(Q, K, V, anchors: Sequence[int], head_maps: Dict[int, Sequence[int]],
                fraction: float, k_min: int, tile_size: int = 128, phase: str = "prefill",
                pooling: str = POST, mode: str = REMAPPED):
    """runner.py:228-297: layer 0 dense (and selects), other anchors select
    fresh sets and attend sparsely over them, reuse layers route the most
    recent anchor's sets through their head map.  Returns (outputs
    [L][Hq][N][d], per-layer dicts with kind / rel_l2 / mass / fallback)."""
    L, Hq, N, d = Q.shape
    Hkv = K.shape[1]
    tiles = prefill_tiles(N, tile_size) if phase == "prefill" else decode_tiles(N)
    bounds = {t: e for (_, e, t) in tiles}
    outs = np.empty((L, Hq, N, d), np.float32)
    rep = []
    cur = None
    aset = set(anchors)
    for l in range(L):
        P, Yd = dense_layer(Q[l], K[l], V[l])
        if l == 0 or l in aset:
            cur = select(layer_pooled(Q[l], K[l], P, tiles, Hkv, pooling), bounds,
                         fraction, k_min, mode, Hkv)
        if l == 0:
            outs[0] = Yd
            rep.append(dict(layer=0, kind="anchor0", rel=0.0, mass=1.0, fallback=0))
            continue
        if l in aset:
            kind, sels = "anchor", cur
        else:
            kind = "reuse"
            hm = head_maps.get(l) if mode == REMAPPED else None
            sels = route(cur, hm, Hkv)
        Y, mass, fb = sparse_layer(Q[l], K[l], V[l], sels, tiles, dense_P=P)
        outs[l] = Y
        rep.append(dict(layer=l, kind=kind, rel=rel_l2(Y, Yd),
                        mass=float(mass.mean(dtype=np.float64)), fallback=len(fb)))
    return outs, rep


# --------------------------------------------------------------------------
# O(n) drivers for sizes the full reference cannot hold
# --------------------------------------------------------------------------

def dense_row(q: np.ndarray, Kg: np.ndarray, Vg: np.ndarray, want_y: bool = True):
    """Post-softmax row and output of one query over all keys of its kv head
    (the last causal row).  Uses 4-row GEMMs: on OpenBLAS a 1-row sgemm
    (and, for P@V, a 2-row one) rounds differently from the rows of the
    reference's full GEMMs; 4-row blocks are bit-equal (tests pin this)."""
    d = q.shape[-1]
    q4 = np.stack([q] * 4).astype(np.float32)
    # no-copy views of fp32 K/V, as the reference's np.asarray(..., float32)
    s = ((q4 @ np.asarray(Kg, dtype=np.float32).T) * _scale(d))[:1]
    p = masked_softmax(s, np.ones_like(s, dtype=bool))
    if not want_y:
        return p[0], None
    y = (np.concatenate([p] * 4) @ np.asarray(Vg, dtype=np.float32))[0]
    return p[0], y


def decode_step(q: np.ndarray, K: np.ndarray, V: np.ndarray, anchors: Sequence[int],
                head_maps: Dict[int, Sequence[int]], fraction: float, k_min: int,
                pooling: str = POST, mode: str = REMAPPED, want_mass: bool = True,
                layers: Optional[Iterable[int]] = None, timings: Optional[Dict[int, float]] = None,
                pooled_out: Optional[Dict[int, List[np.ndarray]]] = None):
    """One decode step (the last token t = n-1) of ``run_kascade(phase=
    'decode')`` for one sequence, in O(n) per layer.

    q [L][Hq][d] is the step's query, K/V [L][Hkv][n][d] the cache including
    the token itself.  Returns (Y [L][Hq][d], sels {layer: [Hkv] arrays of the
    selection used by that layer}, mass [L][Hq]).  Tile = [n-1, n), causal
    bound n, k = k_budget(n) (runner.py:199-206, tiles.py:145-150).
    ``timings`` (optional) receives the wall time of every layer;
    ``pooled_out`` (optional) the pooled vector of every kv head of every
    anchor layer (the ranking the selection was taken from).

    K and V are only indexed as K[l, g] (one head's rows) and K[l, g, sel]
    (a gather), so any object with that indexing and a ``shape`` works --
    the scale tests pass lazy views of device caches."""
    L, Hq, d = q.shape
    Hkv, n = K.shape[1], K.shape[2]
    G = Hq // Hkv
    kk = k_budget(fraction, k_min, n)
    Y = np.zeros((L, Hq, d), np.float32)
    mass = np.zeros((L, Hq), np.float32)
    sels_used: Dict[int, List[np.ndarray]] = {}
    aset = set(anchors)
    cur = None
    todo = set(range(L)) if layers is None else set(layers)
    clock = __import__("time").perf_counter
    for l in range(L):
        is_anchor = l == 0 or l in aset
        if l not in todo and not is_anchor:
            continue
        t_start = clock()
        P = np.zeros((Hq, 1, n), np.float32)
        Yd = np.zeros((Hq, d), np.float32)
        if l == 0 or want_mass or (is_anchor and pooling == POST):
            for h in range(Hq):
                P[h, 0], y = dense_row(q[l, h], K[l, h // G], V[l, h // G] if l == 0 else None, want_y=l == 0)
                if y is not None:
                    Yd[h] = y
        if is_anchor:
            pooled = {}
            for g in range(Hkv):
                if pooling == POST:
                    pooled[(g, n - 1)] = P[g * G:(g + 1) * G, 0:1, :n].mean(axis=(0, 1), dtype=np.float64)
                else:
                    qbar = q[l, g * G:(g + 1) * G].astype(np.float32).mean(axis=0, dtype=np.float64)
                    s = (np.asarray(K[l, g], dtype=np.float64) @ qbar) / math.sqrt(d)
                    pooled[(g, n - 1)] = softmax_vec(s).astype(np.float64)
            cur = select(pooled, {n - 1: n}, fraction, k_min, mode, Hkv)
            if pooled_out is not None:
                pooled_out[l] = [pooled[(g, n - 1)] for g in range(Hkv)]
        if l == 0:
            Y[0] = Yd
            mass[0] = 1.0
            sels_used[0] = [cur[(g, n - 1)] for g in range(Hkv)]
            if timings is not None:
                timings[0] = clock() - t_start
            continue
        if l in aset:
            sels = cur
        else:
            hm = head_maps.get(l) if mode == REMAPPED else None
            sels = route(cur, hm, Hkv)
        sels_used[l] = [sels[(g, n - 1)] for g in range(Hkv)]
        if l not in todo:
            continue
        for g in range(Hkv):
            sel = sels[(g, n - 1)]
            ks = np.asarray(K[l, g, sel], dtype=np.float32)     # the gather is the only copy
            vs = np.asarray(V[l, g, sel], dtype=np.float32)
            for j in range(G):
                h = g * G + j
                s = (q[l, h][None].astype(np.float32) @ ks.T) * _scale(d)
                p = masked_softmax(s, np.ones_like(s, dtype=bool))
                Y[l, h] = (p @ vs)[0]
                if want_mass:
                    mass[l, h] = np.float32(P[h, 0, sel].astype(np.float64).sum())
        if timings is not None:
            timings[l] = clock() - t_start
    del kk
    return Y, sels_used, mass


def prefill_tile_rows(Ql, Kl, g: int, G: int, start: int, end: int) -> np.ndarray:
    """Dense post-softmax rows [G][T][N] of one prefill tile (attention.py:
    128-134 restricted to the tile's rows; 128-row GEMMs are bit-equal to the
    reference's full-GEMM rows)."""
    d = Ql.shape[-1]
    N = Kl.shape[1]
    rows = np.arange(start, end)
    vis = np.arange(N)[None, :] <= rows[:, None]
    kk = np.asarray(Kl[g], dtype=np.float32)
    return np.stack([masked_softmax((Ql[g * G + j, start:end].astype(np.float32) @ kk.T) * _scale(d), vis)
                     for j in range(G)])


def prefill_tile_select(Ql, Kl, g: int, G: int, start: int, end: int, fraction: float,
                        k_min: int, pooling: str = POST) -> Tuple[np.ndarray, np.ndarray]:
    """(selection, pooled vector) of one prefill tile of an anchor layer
    (runner.py:148-152,199-206) without materialising the full [Hq][N][N] P."""
    if pooling == POST:
        Pt = prefill_tile_rows(Ql, Kl, g, G, start, end)
        pooled = Pt[:, :, :end].mean(axis=(0, 1), dtype=np.float64)
    else:
        pooled = pooled_pre(Ql, Kl, g, G, start, end)
    return topk_sorted(pooled, k_budget(fraction, k_min, end)), pooled


# --------------------------------------------------------------------------
# offline calibration: head similarity / head maps (heads.py:50-143,
# pipeline.py:31-73) and the layer similarity matrix (metrics.py:105-335)
# --------------------------------------------------------------------------

def group_mean(P: np.ndarray, G: int) -> np.ndarray:
    """heads.py:50-59: per-kv-head distributions, the fp64 mean of the
    group's G query-head rows, stored as fp32 -> [Hkv][N][N]."""
    Hq, N, M = P.shape
    return P.reshape(Hq // G, G, N, M).mean(axis=1, dtype=np.float64).astype(np.float32)


def token_sets(D: np.ndarray, k: int):
    """Per-token Top-k of causal rows (ranking.py:14-25 + the row-r support
    mask of heads.py:92-94 / metrics.py:133-149): positions ordered by
    (value desc, index asc), the first min(k, r+1) valid.  D [..][N][N] ->
    (idx [..][N][take], valid [N][take])."""
    N = D.shape[-1]
    take = min(k, N)
    idx = np.argsort(-D, axis=-1, kind="stable")[..., :take]
    valid = np.arange(take)[None, :] < np.minimum(np.arange(N) + 1, take)[:, None]
    return idx, valid


def masked_mass(D: np.ndarray, idx: np.ndarray, valid: np.ndarray) -> np.ndarray:
    """fp64 sum of D[row][idx[row][t]] over valid t: [..][N][N] -> [..][N]."""
    got = np.take_along_axis(D.astype(np.float64), np.where(valid, idx, 0), axis=-1)
    return np.where(valid, got, 0.0).sum(axis=-1)


def _agg(scores: np.ndarray, how: str) -> float:
    if scores.size == 0:
        return 0.0
    return float(scores.mean(dtype=np.float64)) if how == "mean" else float(scores.min())


def head_similarity_dists(idx_a: np.ndarray, Db: np.ndarray, k: int, how: str = "mean") -> np.ndarray:
    """heads.py:67-108: hs[i][j] = token aggregate of mass(Db_j on anchor
    head i's per-token sets) / mass(Db_j on its own sets), fp32 per token."""
    Hkv = Db.shape[0]
    idx_b, valid = token_sets(Db, k)
    hs = np.zeros((Hkv, Hkv), np.float64)
    for j in range(Hkv):
        den = masked_mass(Db[j], idx_b[j], valid)
        ok = den != 0.0
        for i in range(Hkv):
            num = masked_mass(Db[j], idx_a[i], valid)
            hs[i, j] = _agg((num[ok] / den[ok]).astype(np.float32), how)
    return hs


def layer_group_dists(Q, K, V, layer: int) -> np.ndarray:
    P, _ = dense_layer(Q[layer], K[layer], V[layer])
    return group_mean(P, Q.shape[1] // K.shape[1])


def head_similarity(Q, K, V, a: int, b: int, k: int = 64, how: str = "mean") -> np.ndarray:
    """heads.py:111-126 for one trace."""
    Da = layer_group_dists(Q, K, V, a)
    Db = Da if a == b else layer_group_dists(Q, K, V, b)
    return head_similarity_dists(token_sets(Da, k)[0], Db, k, how)


def head_maps(Q, K, V, anchors: Sequence[int], k: int = 64) -> Dict[int, List[int]]:
    """pipeline.py:31-73 (remapped mode): for each reuse layer, argmax over
    anchor heads (first maximum) of its similarity column against the most
    recent anchor.  Returns {layer: map}."""
    L = Q.shape[0]
    anchors = sorted(set(anchors))
    out = {}
    for n, a in enumerate(anchors):
        end = anchors[n + 1] if n + 1 < len(anchors) else L
        if a + 1 >= end:
            continue
        idx_a = token_sets(layer_group_dists(Q, K, V, a), k)[0]
        for b in range(a + 1, end):
            hs = head_similarity_dists(idx_a, layer_group_dists(Q, K, V, b), k)
            out[b] = [int(x) for x in hs.argmax(axis=0)]
    return out


def planning_matrix(Q, K, V, k: int = 64, how: str = "mean", tile: int = 128, phase: str = "prefill"):
    """metrics.py:226-295: per-(kv head, tile) pooled distributions (fp64)
    and their Top-k sets per layer; S[a][b] aggregates, over tiles, the mean
    over reuse heads j of mass(b, j on a's set of head map[j]) / mass(b, j on
    its own set), the head map maximising the tile-mean per-head score.
    Returns (S fp32 [L][L], undefined count)."""
    L, Hq = Q.shape[0], Q.shape[1]
    Hkv, N = K.shape[1], Q.shape[2]
    G = Hq // Hkv
    tiles = prefill_tiles(N, tile) if phase == "prefill" else decode_tiles(N)
    dist, sets, den = [], [], []
    for layer in range(L):
        P, _ = dense_layer(Q[layer], K[layer], V[layer])
        dl, sl, nl = {}, {}, {}
        for g in range(Hkv):
            for s, e, t in tiles:
                w = pooled_post(P, g, G, s, e)
                chosen = np.argsort(-w, kind="stable")[:min(k, e)]
                dl[(g, t)], sl[(g, t)], nl[(g, t)] = w, np.sort(chosen), float(w[chosen].sum())
        dist.append(dl), sets.append(sl), den.append(nl)
    tids = [t for _, _, t in tiles]

    def score(i, a, j, b, t):
        d = den[b][(j, t)]
        return None if d == 0.0 else float(np.float32(float(dist[b][(j, t)][sets[a][(i, t)]].sum()) / d))

    S = np.zeros((L, L), np.float32)
    undefined = 0
    for b in range(L):
        for a in range(b + 1):
            hs = np.zeros((Hkv, Hkv))
            for i in range(Hkv):
                for j in range(Hkv):
                    v = [x for x in (score(i, a, j, b, t) for t in tids) if x is not None]
                    hs[i, j] = np.mean(v) if v else 0.0
            hm = hs.argmax(axis=0)
            per_tile = []
            for t in tids:
                v = [score(int(hm[j]), a, j, b, t) for j in range(Hkv)]
                kept = [x for x in v if x is not None]
                undefined += len(v) - len(kept)
                if kept:
                    per_tile.append(float(np.mean(kept)))
            if per_tile:
                S[a, b] = np.float32(np.mean(per_tile) if how == "mean" else np.min(per_tile))
    return S, undefined


def diagnostic_matrix(Q, K, V, k: int = 64, how: str = "mean"):
    """metrics.py:205-223: per-token distributions averaged over ALL query
    heads; S[a][b] aggregates mass(b on a's sets) / mass(b on b's sets)."""
    L = Q.shape[0]
    S = np.zeros((L, L), np.float32)
    undefined = 0
    kept_sets = []
    for b in range(L):
        P, _ = dense_layer(Q[b], K[b], V[b])
        Db = P.mean(axis=0, dtype=np.float64).astype(np.float32)
        idx_b, valid = token_sets(Db, k)
        den = masked_mass(Db, idx_b, valid)
        kept_sets.append(idx_b)
        ok = den != 0.0
        for a in range(b + 1):
            num = masked_mass(Db, kept_sets[a], valid)
            sc = np.zeros_like(num)
            sc[ok] = num[ok] / den[ok]
            sc = sc.astype(np.float32)
            undefined += int((~ok).sum())
            S[a, b] = np.float32(_agg(sc[ok], how)) if how == "mean" else _agg(sc[ok], how)
    return S, undefined
