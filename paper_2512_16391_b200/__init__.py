"""B200-native Kascade anchor/reuse attention engine (arxiv 2512.16391).

Drop-in for the hot path of the reference package ``kascade``: the same
host types and exception taxonomy, a batched PyTorch API (``ops``), layer
executors (``engine``) and the reference-signature functions over traces
(``compat``), all running on hand-written sm_100a kernels behind the C ABI
in ``include/kascade_b200.h``.  There is no CPU fallback.
"""

from .exceptions import (FormatError, InvalidArgumentError, InvalidPlanError, KascadeError, NumericError,
                         UndefinedScoreError, UnsupportedOperationError)
from .host_types import (AnchorPlan, AnchorPlanCore, AttentionTrace, HeadMap, KBudgetPolicy, LayerReport,
                         RunReport, Tile, TileSpec, TopkAttentionResult, TopKIndexSet, identity_head_map,
                         k_budget, make_tiles, plan_from_dict, plan_to_dict, read_plan, write_plan)

__version__ = "0.1.0"


def __getattr__(name):
    # lazy: importing the package must not require torch/CUDA (plan tooling)
    if name in ("ops", "engine", "compat"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    if name in ("dense_attention", "topk_attention", "oracle_topk_indices", "run_kascade", "run_dense",
                "compare", "softmax_row", "AttentionDistribution", "pool_presoftmax", "pool_postsoftmax",
                "layer_distribution", "mass_coverage", "sim_score", "pooled_all_heads_topk"):
        from . import compat
        return getattr(compat, name)
    if name in ("compute_head_map", "compute_head_maps", "head_similarity", "similarity_matrix", "SimilarityMatrix",
                "LayerImportance", "layer_importance", "apply_importance", "select_anchors", "build_plan",
                "exhaustive_select", "objective"):
        from . import calibration
        return getattr(calibration, name)
    if name in ("BenchRow", "CostParams", "CostReport", "get_preset", "predict_ratios", "predict_report",
                "preset_names", "weighted_pipeline_time", "report_from_preset", "fit_ratios"):
        from . import costmodel
        return getattr(costmodel, name)
    if name in ("SynthConfig", "generate_synthetic"):
        from . import synth
        return getattr(synth, name)
    if name in ("read_trace", "write_trace"):
        from . import kscd_io
        return getattr(kscd_io, name)
    raise AttributeError(name)
