"""Freeze the reference's small path utilities (tiles.py:92-114,
metrics.py:80-131, heads.py:155-171) on seeded inputs for
tests/test_utils_gpu.py.  Dev container only (imports /root/reference).

    python tests/golden/make_utils_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from kascade import heads, metrics, tiles  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(123)
    out = {}
    q_tile = rng.standard_normal((37, 128)).astype(np.float32)
    out["q_tile"], out["pre"] = q_tile, tiles.pool_presoftmax(q_tile)
    rows = []
    for n in (5, 9, 9, 3, 12):
        w = rng.random(n)
        rows.append((w / w.sum()).astype(np.float32))
    for i, r in enumerate(rows):
        out[f"row{i}"] = r
    out["post"] = tiles.pool_postsoftmax(rows)
    P = rng.random((4, 40, 40)).astype(np.float32)
    P = np.tril(P)
    P = (P / P.sum(axis=-1, keepdims=True)).astype(np.float32)
    out["P"], out["layer_dist"] = P, metrics.layer_distribution(P)
    out["cov_mean"] = metrics.mass_coverage(P, 7)
    out["cov_rows"] = metrics.mass_coverage(P, 7, per_row=True)
    pb = rows[3]
    pb = np.concatenate([rows[4], np.zeros(0, np.float32)])
    ia, ib = np.array([0, 3, 5, 11]), np.array([1, 3, 4, 11])
    out["pb"], out["ia"], out["ib"], out["sim"] = pb, ia, ib, np.array(metrics.sim_score(pb, ia, ib))
    gd = rng.random((3, 50)).astype(np.float32)
    sel = heads.pooled_all_heads_topk(gd, 9, tile_id=4)
    out["gd"], out["pooled_sel"] = gd, sel.indices
    np.savez_compressed(os.path.join(HERE, "utils_ref.npz"), **out)


if __name__ == "__main__":
    main()
