"""The reference's analytic cost model (costmodel.py), with B200 presets
(SURVEY.md 8(f) rank 4).

Two tables of per-layer kernel times feed the same arithmetic -- the
weighted pipeline time (costmodel.py:156-184), the per-preset report
(187-201) and the least-squares ratio fit and prediction (204-280):

* ``PUBLISHED_BENCH`` -- the paper's H100 Table 3 rows the reference
  bundles (costmodel.py:64-112), presets ``table3-{phase}-{seq}-k{pct}``.
  Every reference name defaults to this table, so a reference caller gets
  the reference's numbers (pinned by tests/golden/costmodel_ref.json).
* ``B200_BENCH`` -- rows MEASURED on B200 with this engine
  (scripts/table3_b200.py -> b200_presets.json): the dense baseline layer
  (this engine's Top-k = 100 % mode, standing in for both of the paper's
  baseline columns), anchor0, anchor and reuse layer times, presets
  ``b200-{phase}-{seq}-k{pct}``; pass ``table="b200"`` to the fit and the
  predictions.
"""

import json
import os
from dataclasses import dataclass, field
from functools import lru_cache
from typing import Dict, List

import numpy as np

from .exceptions import InvalidArgumentError

PHASE_DECODE = "decode"
PHASE_PREFILL = "prefill"

PIPELINE_LAYERS = 32       # layer count behind the published weights (costmodel.py:35)
PIPELINE_ANCHORS = 5       # anchor count behind the published weights (costmodel.py:36)

FIT_MIN_SEQ = 65536        # rows used for the ratio fit (costmodel.py:38)
VALID_MIN_SEQ = 16384      # below this the fitted model is flagged (costmodel.py:39)

TABLE_PUBLISHED, TABLE_B200 = "table3", "b200"
_HERE = os.path.dirname(os.path.abspath(__file__))


@dataclass(frozen=True)
class BenchRow:
    """One kernel microbenchmark row, times in ms per layer
    (costmodel.py:42-62; same fields and order).  ``table`` names the
    preset family; B200 rows carry their dense layer in both baseline
    columns and derive the ratio / pipeline columns from their times."""

    phase: str
    seq_len: int
    topk_pct: int
    fa3_ms: float
    tl_ms: float
    anchor0_ms: float
    anchor0_ratio: float
    anchor_ms: float
    anchor_ratio: float
    reuse_ms: float
    reuse_ratio: float
    kascade_ms: float
    speedup_fa3: float
    speedup_tl: float
    table: str = TABLE_PUBLISHED
    batch: int = 1

    @property
    def preset_name(self) -> str:
        return f"{self.table}-{self.phase}-{self.seq_len}-k{self.topk_pct}"

    @property
    def dense_ms(self) -> float:
        """The baseline column report_from_preset divides by."""
        return self.tl_ms

    @property
    def speedup(self) -> float:
        return self.speedup_tl


def _published() -> List[BenchRow]:
    with open(os.path.join(_HERE, "published_table3.json"), "r", encoding="utf-8") as f:
        data = json.load(f)
    return [BenchRow(**dict(zip(data["fields"], row))) for row in data["rows"]]


def _b200_row(phase, seq_len, topk_pct, dense_ms, anchor0_ms, anchor_ms, reuse_ms, batch=1) -> BenchRow:
    kascade = (anchor0_ms + (PIPELINE_ANCHORS - 1) * anchor_ms
               + (PIPELINE_LAYERS - PIPELINE_ANCHORS) * reuse_ms) / PIPELINE_LAYERS
    return BenchRow(phase, seq_len, topk_pct, dense_ms, dense_ms, anchor0_ms, anchor0_ms / dense_ms, anchor_ms,
                    anchor_ms / dense_ms, reuse_ms, reuse_ms / dense_ms, kascade, dense_ms / kascade,
                    dense_ms / kascade, table=TABLE_B200, batch=batch)


def _b200() -> List[BenchRow]:
    with open(os.path.join(_HERE, "b200_presets.json"), "r", encoding="utf-8") as f:
        data = json.load(f)
    return [_b200_row(r["phase"], int(r["seq_len"]), int(r["topk_pct"]), float(r["dense_ms"]),
                      float(r["anchor0_ms"]), float(r["anchor_ms"]), float(r["reuse_ms"]), int(r.get("batch", 1)))
            for r in data["rows"]]


PUBLISHED_BENCH: List[BenchRow] = _published()
B200_BENCH: List[BenchRow] = _b200()
_TABLES = {TABLE_PUBLISHED: PUBLISHED_BENCH, TABLE_B200: B200_BENCH}


def _table(table: str) -> List[BenchRow]:
    if table not in _TABLES:
        raise InvalidArgumentError(f"unknown preset table {table!r}; known: {', '.join(_TABLES)}")
    return _TABLES[table]


def preset_names(table: str = TABLE_PUBLISHED) -> List[str]:
    """costmodel.py:115-116 (``table="b200"`` for the measured B200 rows)."""
    return [row.preset_name for row in _table(table)]


def get_preset(name: str) -> BenchRow:
    """costmodel.py:119-125; resolves ``table3-...`` and ``b200-...`` names."""
    for rows in _TABLES.values():
        for row in rows:
            if row.preset_name == name:
                return row
    raise InvalidArgumentError(f"unknown preset {name!r}; known presets: "
                               f"{', '.join(preset_names(TABLE_PUBLISHED) + preset_names(TABLE_B200))}")


@dataclass
class CostParams:
    """costmodel.py:115-130."""

    phase: str
    num_layers: int = PIPELINE_LAYERS
    num_anchors: int = PIPELINE_ANCHORS
    topk_fraction: float = 0.1
    seq_len: int = 131072
    baseline_layer_time: float = 1.0

    def __post_init__(self):
        if self.num_anchors > self.num_layers or self.num_anchors < 1:
            raise InvalidArgumentError(f"num_anchors {self.num_anchors} outside [1, {self.num_layers}]")
        if self.baseline_layer_time <= 0:
            raise InvalidArgumentError("baseline_layer_time must be > 0")


@dataclass
class CostReport:
    """costmodel.py:133-141."""

    kascade_time: float
    speedup: float
    baseline_time: float
    per_kind: Dict[str, float]
    valid: bool = True
    note: str = ""


def weighted_pipeline_time(params: CostParams, per_kind_times: Dict[str, float]) -> CostReport:
    """time = (t_anchor0 + (M-1) t_anchor + (L-M) t_reuse) / L, speedup =
    baseline / time (costmodel.py:144-184)."""
    for kind in ("anchor0", "anchor", "reuse"):
        if kind not in per_kind_times or per_kind_times[kind] <= 0:
            raise InvalidArgumentError(f"per-kind time {kind!r} must be > 0")
    L, M = params.num_layers, params.num_anchors
    t0, ta, tr = per_kind_times["anchor0"], per_kind_times["anchor"], per_kind_times["reuse"]
    time = (t0 + (M - 1) * ta + (L - M) * tr) / L
    valid = params.seq_len >= VALID_MIN_SEQ
    return CostReport(kascade_time=time, speedup=params.baseline_layer_time / time,
                      baseline_time=params.baseline_layer_time,
                      per_kind={"anchor0": t0 / L, "anchor": (M - 1) * ta / L, "reuse": (L - M) * tr / L},
                      valid=valid, note="" if valid else f"fixed overheads dominate below seq {VALID_MIN_SEQ}")


def report_from_preset(name: str) -> CostReport:
    """costmodel.py:187-201: one row's per-kind times against its own
    dense-baseline column (tl_ms)."""
    row = get_preset(name)
    params = CostParams(phase=row.phase, topk_fraction=row.topk_pct / 100.0, seq_len=row.seq_len,
                        baseline_layer_time=row.dense_ms)
    return weighted_pipeline_time(params, {"anchor0": row.anchor0_ms, "anchor": row.anchor_ms,
                                           "reuse": row.reuse_ms})


@dataclass(frozen=True)
class RatioFit:
    phase: str
    c_gather: float
    c_select: float
    c_pass1: float
    max_residual: Dict[str, float] = field(default_factory=dict)


def fit_ratios_from(rows, phase: str) -> RatioFit:
    """The reference's least-squares constants (costmodel.py:213-241) over
    any rows carrying topk_pct / seq_len and the three per-kind ratios:
    reuse ~ f + c_gather, anchor0 ~ 1 + c_select, anchor ~ c_pass1 +
    c_select + reuse, fitted on the rows with seq_len >= 65536."""
    rows = [r for r in rows if r.phase == phase and r.seq_len >= FIT_MIN_SEQ]
    if not rows:
        raise InvalidArgumentError(f"unknown phase {phase!r}")
    fracs = np.array([r.topk_pct / 100.0 for r in rows])
    reuse = np.array([r.reuse_ratio for r in rows])
    anchor0 = np.array([r.anchor0_ratio for r in rows])
    anchor = np.array([r.anchor_ratio for r in rows])
    c_gather = float(np.mean(reuse - fracs))
    c_select = float(np.mean(anchor0 - 1.0))
    c_pass1 = float(np.mean(anchor - c_select - (fracs + c_gather)))
    resid = {"reuse": float(np.max(np.abs(reuse - (fracs + c_gather)))),
             "anchor0": float(np.max(np.abs(anchor0 - (1.0 + c_select)))),
             "anchor": float(np.max(np.abs(anchor - (c_pass1 + c_select + fracs + c_gather))))}
    return RatioFit(phase=phase, c_gather=c_gather, c_select=c_select, c_pass1=c_pass1, max_residual=resid)


@lru_cache(maxsize=None)
def fit_ratios(phase: str, table: str = TABLE_PUBLISHED) -> RatioFit:
    """costmodel.py:212-238: fit_ratios_from over one preset table."""
    return fit_ratios_from(_table(table), phase)


def predict_ratios(phase: str, topk_fraction: float, seq_len: int, table: str = TABLE_PUBLISHED) -> Dict[str, float]:
    """costmodel.py:244-258."""
    if not (0.0 < topk_fraction <= 1.0):
        raise InvalidArgumentError(f"topk_fraction must be in (0, 1], got {topk_fraction}")
    fit = fit_ratios(phase, table)
    reuse = topk_fraction + fit.c_gather
    return {"anchor0": 1.0 + fit.c_select, "anchor": fit.c_pass1 + fit.c_select + reuse, "reuse": reuse,
            "valid": float(seq_len >= VALID_MIN_SEQ)}


def predict_report(phase: str, topk_fraction: float, seq_len: int, num_layers: int = PIPELINE_LAYERS,
                   num_anchors: int = PIPELINE_ANCHORS, baseline_layer_time: float = 1.0,
                   table: str = TABLE_PUBLISHED) -> CostReport:
    """costmodel.py:261-280."""
    ratios = predict_ratios(phase, topk_fraction, seq_len, table)
    params = CostParams(phase=phase, num_layers=num_layers, num_anchors=num_anchors, topk_fraction=topk_fraction,
                        seq_len=seq_len, baseline_layer_time=baseline_layer_time)
    times = {kind: ratios[kind] * baseline_layer_time for kind in ("anchor0", "anchor", "reuse")}
    return weighted_pipeline_time(params, times)
