"""kascade.heads (heads.py): head maps and head-level reuse scores (masked sums on the device)."""
from ..calibration import PLANNING_K, TOKEN_AGG_MEAN, TOKEN_AGG_MIN, compute_head_map, head_similarity
from ..compat import group_distributions, head_similarity_from_dists, pooled_all_heads_topk, topk_tables
from ..host_types import MODE_ALL_HEADS_POOLED, MODE_IDENTITY, MODE_REMAPPED, HeadMap, identity_head_map

__all__ = ["MODE_REMAPPED", "MODE_IDENTITY", "MODE_ALL_HEADS_POOLED", "HeadMap", "group_distributions", "topk_tables",
           "head_similarity_from_dists", "head_similarity", "compute_head_map", "identity_head_map",
           "pooled_all_heads_topk", "PLANNING_K", "TOKEN_AGG_MEAN", "TOKEN_AGG_MIN"]
