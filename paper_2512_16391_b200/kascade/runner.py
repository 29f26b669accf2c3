"""kascade.runner (runner.py): the anchor/reuse pipeline over a trace, on the B200 engine."""
from ..compat import compare, run_dense, run_kascade
from ..host_types import (KIND_ANCHOR, KIND_ANCHOR0, KIND_REUSE, POOL_POST, POOL_PRE, AnchorPlan, LayerReport,
                          RunReport)

__all__ = ["POOL_POST", "POOL_PRE", "KIND_ANCHOR0", "KIND_ANCHOR", "KIND_REUSE", "AnchorPlan", "LayerReport",
           "RunReport", "run_dense", "run_kascade", "compare"]
