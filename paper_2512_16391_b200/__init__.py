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
                "compare", "softmax_row"):
        from . import compat
        return getattr(compat, name)
    raise AttributeError(name)
