"""kascade.metrics (metrics.py): coverage, reuse similarity matrices and layer importance."""
from ..calibration import (MODE_DIAGNOSTIC, MODE_PLANNING, PLANNING_K, TOKEN_AGG_MEAN, TOKEN_AGG_MIN, LayerImportance,
                           SimilarityMatrix, apply_importance, layer_importance, similarity_matrix)
from ..compat import _token_topk, layer_distribution, mass_coverage, sim_score  # noqa: F401  (_token_topk: tests)

__all__ = ["TOKEN_AGG_MEAN", "TOKEN_AGG_MIN", "PLANNING_K", "MODE_DIAGNOSTIC", "MODE_PLANNING", "SimilarityMatrix",
           "LayerImportance", "mass_coverage", "layer_distribution", "sim_score", "similarity_matrix",
           "layer_importance", "apply_importance"]
