"""Host-side types of the anchor/reuse API, field-compatible with the
reference package so its objects (and plan JSON files) drop in unchanged.

Mirrors: KBudgetPolicy / k_budget / Tile / TileSpec / make_tiles
(tiles.py:25-152), TopKIndexSet / TopkAttentionResult (attention.py:40-74),
HeadMap (heads.py:25-47), AnchorPlanCore (planner.py:24-42), AnchorPlan /
LayerReport / RunReport (runner.py:49-129), AttentionTrace (trace.py:11-113)
and the plan JSON schema v1 (traceio.py:315-407).  Reference objects are
accepted wherever these are (duck typing on the same field names).
"""

from __future__ import annotations

import hashlib
import json
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from .exceptions import FormatError, InvalidArgumentError, InvalidPlanError

PREFILL, DECODE = "prefill", "decode"
POOL_POST, POOL_PRE = "post", "pre"
MODE_REMAPPED, MODE_IDENTITY, MODE_ALL_HEADS_POOLED = "remapped", "identity", "all_heads_pooled"
KIND_ANCHOR0, KIND_ANCHOR, KIND_REUSE = "anchor0", "anchor", "reuse"
DEFAULT_TILE_SIZE, DEFAULT_TOPK_FRACTION, DEFAULT_K_MIN = 128, 0.1, 128


# ------------------------------------------------------------------ budgets
@dataclass(frozen=True)
class KBudgetPolicy:
    """k = min(max(floor(fraction * n), k_min), n) over n visible keys."""

    fraction: float = DEFAULT_TOPK_FRACTION
    k_min: int = DEFAULT_K_MIN

    def __post_init__(self):
        if not 0.0 < self.fraction <= 1.0:
            raise InvalidArgumentError(f"fraction must be in (0, 1], got {self.fraction}")
        if self.k_min < 1:
            raise InvalidArgumentError(f"k_min must be >= 1, got {self.k_min}")


def k_budget(policy, num_keys: int) -> int:
    """Floors the fp64 product before clamping (tiles.py:81-89); the same
    expression the C ABI evaluates (kscd_k_budget)."""
    if num_keys < 1:
        raise InvalidArgumentError(f"num_keys must be >= 1, got {num_keys}")
    return min(max(math.floor(policy.fraction * num_keys), policy.k_min), num_keys)


# -------------------------------------------------------------------- tiles
@dataclass(frozen=True)
class Tile:
    start: int
    end: int
    kv_head: int
    tile_id: int

    @property
    def causal_bound(self) -> int:
        return self.end


@dataclass
class TileSpec:
    phase: str
    tile_size: int
    tiles: List[Tile] = field(default_factory=list)

    def validate(self, seq_len: int, num_kv_heads: int):
        if self.phase not in (PREFILL, DECODE):
            raise InvalidArgumentError(f"unknown phase {self.phase!r}")
        for g in range(num_kv_heads):
            cursor = 0
            for s, e in sorted((t.start, t.end) for t in self.tiles if t.kv_head == g):
                if s != cursor or e <= s:
                    raise InvalidArgumentError(f"tiles for kv head {g} do not partition rows (at {s})")
                cursor = e
            if cursor != seq_len:
                raise InvalidArgumentError(f"tiles for kv head {g} cover {cursor} of {seq_len} rows")


def make_tiles(seq_len: int, phase: str, num_query_heads: int, num_kv_heads: int,
               tile_size: int = DEFAULT_TILE_SIZE) -> TileSpec:
    """Prefill: ceil(N/tile) row blocks per kv head; decode: one single-row
    tile per token per kv head with tile_size = Hq/Hkv (tiles.py:117-152)."""
    if tile_size < 1:
        raise InvalidArgumentError(f"tile_size must be >= 1, got {tile_size}")
    if num_query_heads % num_kv_heads:
        raise InvalidArgumentError(
            f"num_query_heads ({num_query_heads}) must be divisible by num_kv_heads ({num_kv_heads})")
    if phase == PREFILL:
        starts = range(0, seq_len, tile_size)
        return TileSpec(PREFILL, tile_size, [Tile(s, min(s + tile_size, seq_len), g, i)
                                             for g in range(num_kv_heads) for i, s in enumerate(starts)])
    if phase == DECODE:
        return TileSpec(DECODE, num_query_heads // num_kv_heads,
                        [Tile(t, t + 1, g, t) for g in range(num_kv_heads) for t in range(seq_len)])
    raise InvalidArgumentError(f"unknown phase {phase!r}")


# --------------------------------------------------------------- selections
@dataclass
class TopKIndexSet:
    kv_head: int
    tile_id: int
    indices: np.ndarray
    k: int

    def __post_init__(self):
        self.indices = np.asarray(self.indices, dtype=np.int64)

    def validate(self, causal_bound: Optional[int] = None):
        idx = self.indices
        if idx.size > 1 and not (np.diff(idx) > 0).all():
            raise InvalidArgumentError("indices must be unique and sorted")
        if (idx < 0).any():
            raise InvalidArgumentError("indices must be non-negative")
        if causal_bound is not None:
            if (idx >= causal_bound).any():
                raise InvalidArgumentError(f"index beyond causal bound {causal_bound} of the tile")
            if idx.size != min(self.k, causal_bound):
                raise InvalidArgumentError(
                    f"expected min(k={self.k}, attendable={causal_bound}) indices, got {idx.size}")


@dataclass
class TopkAttentionResult:
    Y: np.ndarray
    mass_recovered: np.ndarray
    fallback_rows: list = field(default_factory=list)


@dataclass
class HeadMap:
    """map[g] = anchor kv head whose Top-k set reuse kv head g borrows."""

    reuse_layer: int
    anchor_layer: int
    map: List[int]
    mode: str = MODE_REMAPPED

    def __post_init__(self):
        self.map = [int(m) for m in self.map]

    def validate(self, num_kv_heads: int):
        if self.mode not in (MODE_REMAPPED, MODE_IDENTITY, MODE_ALL_HEADS_POOLED):
            raise InvalidArgumentError(f"unknown head-map mode {self.mode!r}")
        if self.mode == MODE_ALL_HEADS_POOLED:
            return
        if len(self.map) != num_kv_heads:
            raise InvalidArgumentError(f"head map has {len(self.map)} entries for {num_kv_heads} kv heads")
        if any(not 0 <= m < num_kv_heads for m in self.map):
            raise InvalidArgumentError("head map entry out of range")


def identity_head_map(num_kv_heads: int, reuse_layer: int = -1, anchor_layer: int = -1) -> HeadMap:
    return HeadMap(reuse_layer, anchor_layer, list(range(num_kv_heads)), MODE_IDENTITY)


# --------------------------------------------------------------------- plans
@dataclass
class AnchorPlanCore:
    anchors: List[int]
    budget: int
    objective_value: float
    source_digest: str = ""

    def __post_init__(self):
        self.anchors = [int(a) for a in self.anchors]
        if len(self.anchors) != self.budget:
            raise InvalidArgumentError(f"{len(self.anchors)} anchors but budget {self.budget}")
        if not self.anchors or self.anchors[0] != 0:
            raise InvalidArgumentError("layer 0 must be the first anchor")
        if any(b <= a for a, b in zip(self.anchors, self.anchors[1:])):
            raise InvalidArgumentError("anchors must be strictly increasing")


@dataclass
class AnchorPlan:
    core: AnchorPlanCore
    head_maps: Dict[int, HeadMap] = field(default_factory=dict)
    pooling: str = POOL_POST
    k_policy: KBudgetPolicy = field(default_factory=KBudgetPolicy)
    tile_size: int = DEFAULT_TILE_SIZE
    mode: str = MODE_REMAPPED

    @property
    def anchors(self) -> List[int]:
        return self.core.anchors

    def latest_anchor(self, layer: int) -> int:
        prior = [a for a in self.anchors if a <= layer]
        if not prior:
            raise InvalidPlanError(f"no anchor precedes layer {layer}")
        return prior[-1]

    def validate(self, trace_or_layers, num_kv_heads: Optional[int] = None):
        """runner.py:71-95.  Accepts a trace or (num_layers, num_kv_heads)."""
        validate_plan(self, trace_or_layers, num_kv_heads)

    def digest(self) -> str:
        payload = {"anchors": self.anchors, "mode": self.mode, "pooling": self.pooling,
                   "tile_size": self.tile_size, "fraction": self.k_policy.fraction,
                   "k_min": self.k_policy.k_min,
                   "head_maps": {str(l): hm.map for l, hm in sorted(self.head_maps.items())}}
        return hashlib.sha256(json.dumps(payload, sort_keys=True).encode()).hexdigest()[:16]


def validate_plan(plan, trace_or_layers, num_kv_heads: Optional[int] = None) -> None:
    """AnchorPlan invariants against a trace shape (runner.py:71-95); works on
    reference AnchorPlan objects too."""
    if num_kv_heads is None:
        L, Hkv = trace_or_layers.num_layers, trace_or_layers.num_kv_heads
    else:
        L, Hkv = int(trace_or_layers), int(num_kv_heads)
    if plan.pooling not in (POOL_POST, POOL_PRE):
        raise InvalidPlanError(f"unknown pooling mode {plan.pooling!r}")
    if plan.mode not in (MODE_REMAPPED, MODE_ALL_HEADS_POOLED):
        raise InvalidPlanError(f"unknown plan mode {plan.mode!r}")
    anchors = list(plan.core.anchors)
    if anchors[-1] >= L:
        raise InvalidPlanError(f"anchor {anchors[-1]} out of range for {L} layers")
    if 0 not in anchors:
        raise InvalidPlanError("layer 0 must be an anchor")
    if plan.mode == MODE_REMAPPED:
        for layer in range(L):
            if layer in anchors:
                continue
            hm = plan.head_maps.get(layer)
            if hm is None:
                raise InvalidPlanError(f"reuse layer {layer} has no head map")
            latest = max(a for a in anchors if a <= layer)
            if hm.anchor_layer != latest:
                raise InvalidPlanError(
                    f"head map for layer {layer} references anchor {hm.anchor_layer}, expected {latest}")
            try:
                hm.validate(Hkv)
            except Exception as e:  # reference HeadMap raises its own InvalidArgumentError
                raise InvalidArgumentError(str(e)) from None


@dataclass
class LayerReport:
    layer: int
    kind: str
    output_rel_err_l2: float
    mass_recovered_mean: float
    fallback_rows: int = 0


@dataclass
class RunReport:
    per_layer: List[LayerReport]
    overall: Dict[str, float]
    config: Dict[str, str] = field(default_factory=dict)

    def kind_mean(self, kind: str, field_name: str) -> float:
        vals = [getattr(r, field_name) for r in self.per_layer if r.kind == kind]
        return float(np.mean(vals)) if vals else float("nan")


# -------------------------------------------------------------------- trace
@dataclass
class AttentionTrace:
    """Q [L][Hq][N][d], K/V [L][Hkv][N][d] (+ optional X/Y), trace.py:11-113."""

    num_layers: int
    num_query_heads: int
    num_kv_heads: int
    head_dim: int
    seq_len: int
    Q: np.ndarray
    K: np.ndarray
    V: np.ndarray
    X: Optional[np.ndarray] = None
    Y: Optional[np.ndarray] = None
    prompt_id: str = ""

    def __post_init__(self):
        self.validate()

    def validate(self) -> None:
        """trace.py:52-98: positive dims, GQA divisibility, tensor shapes,
        finite payloads, X/Y together with matching [L][N][model_dim]."""
        dims = dict(num_layers=self.num_layers, num_query_heads=self.num_query_heads,
                    num_kv_heads=self.num_kv_heads, head_dim=self.head_dim, seq_len=self.seq_len)
        for name, v in dims.items():
            if v < 1:
                raise InvalidArgumentError(f"{name} must be >= 1, got {v}")
        if self.num_query_heads % self.num_kv_heads:
            raise InvalidArgumentError(f"num_query_heads ({self.num_query_heads}) must be divisible by "
                                       f"num_kv_heads ({self.num_kv_heads})")
        L, Hq, Hkv, d, N = (self.num_layers, self.num_query_heads, self.num_kv_heads, self.head_dim,
                            self.seq_len)
        for name, shape in (("Q", (L, Hq, N, d)), ("K", (L, Hkv, N, d)), ("V", (L, Hkv, N, d))):
            arr = getattr(self, name)
            if tuple(arr.shape) != shape:
                raise InvalidArgumentError(f"{name} has shape {tuple(arr.shape)}, header implies {shape}")
            if not np.isfinite(arr).all():
                raise InvalidArgumentError(f"{name} contains non-finite values")
        if (self.X is None) != (self.Y is None):
            raise InvalidArgumentError("X and Y must be supplied together")
        if self.X is not None:
            for name in ("X", "Y"):
                arr = getattr(self, name)
                if arr.ndim != 3 or arr.shape[0] != L or arr.shape[1] != N:
                    raise InvalidArgumentError(f"{name} has shape {tuple(arr.shape)}, expected "
                                               f"[L={L}][N={N}][model_dim]")
                if not np.isfinite(arr).all():
                    raise InvalidArgumentError(f"{name} contains non-finite values")
            if self.X.shape != self.Y.shape:
                raise InvalidArgumentError(f"X shape {tuple(self.X.shape)} != Y shape {tuple(self.Y.shape)}")

    def equals(self, other) -> bool:
        """trace.py:100-120: bit-exact equality of header and tensors."""
        head = ("num_layers", "num_query_heads", "num_kv_heads", "head_dim", "seq_len", "prompt_id")
        if any(getattr(self, f) != getattr(other, f) for f in head) or self.has_xy() != other.has_xy():
            return False
        names = ("Q", "K", "V", "X", "Y") if self.has_xy() else ("Q", "K", "V")
        return all(np.array_equal(getattr(self, n), getattr(other, n)) for n in names)

    @property
    def group_size(self) -> int:
        return self.num_query_heads // self.num_kv_heads

    def kv_head_of(self, query_head: int) -> int:
        return query_head // self.group_size

    def has_xy(self) -> bool:
        return self.X is not None and self.Y is not None


# ---------------------------------------------------------- plan JSON (v1)
def plan_to_dict(plan) -> dict:
    return {
        "schema_version": 1, "kind": "kascade-plan", "anchors": list(plan.core.anchors),
        "budget": plan.core.budget, "objective_value": plan.core.objective_value,
        "source_digest": plan.core.source_digest, "mode": plan.mode, "pooling": plan.pooling,
        "tile_size": plan.tile_size,
        "k_policy": {"fraction": plan.k_policy.fraction, "k_min": plan.k_policy.k_min},
        "head_maps": [{"reuse_layer": hm.reuse_layer, "anchor_layer": hm.anchor_layer, "mode": hm.mode,
                       "map": list(hm.map)} for _, hm in sorted(plan.head_maps.items())],
    }


def plan_from_dict(d: dict) -> AnchorPlan:
    """Schema v1 of traceio.py:315-392 (same field names and checks)."""
    def need(obj, key, kinds, path):
        if not isinstance(obj, dict) or key not in obj:
            raise FormatError("missing required field", field_path=f"{path}.{key}")
        if not isinstance(obj[key], kinds):
            raise FormatError(f"field has type {type(obj[key]).__name__}", field_path=f"{path}.{key}")
        return obj[key]

    if need(d, "schema_version", int, "$") != 1:
        raise FormatError("unsupported plan schema version", field_path="$.schema_version")
    kp = need(d, "k_policy", dict, "$")
    maps = {}
    for i, e in enumerate(need(d, "head_maps", list, "$")):
        p = f"$.head_maps[{i}]"
        hm = HeadMap(need(e, "reuse_layer", int, p), need(e, "anchor_layer", int, p),
                     need(e, "map", list, p), need(e, "mode", str, p))
        maps[hm.reuse_layer] = hm
    try:
        core = AnchorPlanCore(need(d, "anchors", list, "$"), need(d, "budget", int, "$"),
                              float(need(d, "objective_value", (int, float), "$")),
                              need(d, "source_digest", str, "$"))
        return AnchorPlan(core=core, head_maps=maps, pooling=need(d, "pooling", str, "$"),
                          k_policy=KBudgetPolicy(float(need(kp, "fraction", (int, float), "$.k_policy")),
                                                 need(kp, "k_min", int, "$.k_policy")),
                          tile_size=need(d, "tile_size", int, "$"), mode=need(d, "mode", str, "$"))
    except InvalidArgumentError as e:
        raise FormatError(f"plan violates invariants: {e}", field_path="$") from None


def read_plan(path) -> AnchorPlan:
    with open(path, "r", encoding="utf-8") as f:
        try:
            return plan_from_dict(json.load(f))
        except json.JSONDecodeError as e:
            raise FormatError(f"plan file is not valid JSON: {e}") from None


def write_plan(path, plan) -> None:
    with open(path, "w", encoding="utf-8") as f:
        json.dump(plan_to_dict(plan), f, indent=2, sort_keys=True)
        f.write("\n")
