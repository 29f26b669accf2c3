"""kascade.ranking (ranking.py): value-ordered Top-k index tables (stable device sort)."""
from ..compat import topk_table

__all__ = ["topk_table"]
