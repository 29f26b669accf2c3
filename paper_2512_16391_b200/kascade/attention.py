"""kascade.attention (attention.py) on the B200 kernels: dense and Top-k sparse attention, exact Top-k."""
from ..compat import AttentionDistribution, dense_attention, oracle_topk_indices, softmax_row, topk_attention
from ..host_types import TopkAttentionResult, TopKIndexSet

__all__ = ["AttentionDistribution", "TopKIndexSet", "TopkAttentionResult", "dense_attention", "oracle_topk_indices",
           "softmax_row", "topk_attention"]
