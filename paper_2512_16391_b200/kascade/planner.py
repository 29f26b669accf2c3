"""kascade.planner (planner.py): the anchor-selection DP and its exhaustive check."""
from ..calibration import DEFAULT_ANCHOR_BUDGET, EXHAUSTIVE_LIMIT, exhaustive_select, objective, select_anchors
from ..host_types import AnchorPlanCore

__all__ = ["DEFAULT_ANCHOR_BUDGET", "EXHAUSTIVE_LIMIT", "AnchorPlanCore", "objective", "select_anchors",
           "exhaustive_select"]
