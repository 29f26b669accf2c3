"""kascade.pipeline (pipeline.py): head maps for a plan and the end-to-end planner."""
from ..calibration import build_plan, compute_head_maps

__all__ = ["compute_head_maps", "build_plan"]
