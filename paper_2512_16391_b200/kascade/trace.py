"""kascade.trace (trace.py): the in-memory attention trace."""
from ..host_types import AttentionTrace

__all__ = ["AttentionTrace"]
