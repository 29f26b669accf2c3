"""kascade.tiles (tiles.py): query tiles, the Top-k budget rule and tile pooling."""
from ..compat import pool_postsoftmax, pool_presoftmax
from ..host_types import (DECODE, DEFAULT_K_MIN, DEFAULT_TILE_SIZE, DEFAULT_TOPK_FRACTION, PREFILL, KBudgetPolicy,
                          Tile, TileSpec, k_budget, make_tiles)

__all__ = ["PREFILL", "DECODE", "DEFAULT_TILE_SIZE", "DEFAULT_TOPK_FRACTION", "DEFAULT_K_MIN", "Tile", "TileSpec",
           "KBudgetPolicy", "k_budget", "pool_presoftmax", "pool_postsoftmax", "make_tiles"]
