"""Freeze what the reference's module layout exposes and a few of its
host/device utilities, for the ``paper_2512_16391_b200.kascade`` namespace
(tests/test_kascade_namespace.py, tests/test_utils_gpu.py).  Dev container
only (imports /root/reference/pkg/src read-only).

    python tests/golden/make_namespace_golden.py
"""
import importlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True
import kascade  # noqa: E402
from kascade import heads, metrics, ranking, traceio  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
MODULES = ("attention", "cli", "costmodel", "errors", "heads", "metrics", "parallel", "pipeline", "planner",
           "ranking", "runner", "tiles", "trace", "traceio")


def public(mod):
    """Public names ``mod`` itself defines (top-level def / class / assignment)."""
    import ast
    tree = ast.parse(open(mod.__file__).read())
    out = set()
    for node in tree.body:
        if isinstance(node, (ast.FunctionDef, ast.ClassDef)):
            out.add(node.name)
        elif isinstance(node, ast.Assign):
            out.update(t.id for t in node.targets if isinstance(t, ast.Name))
        elif isinstance(node, ast.AnnAssign) and isinstance(node.target, ast.Name):
            out.add(node.target.id)
    return sorted(n for n in out if not n.startswith("_"))


def main():
    names = {"__root__": sorted(n for n in dir(kascade) if not n.startswith("_"))}
    for m in MODULES:
        mod = importlib.import_module(f"kascade.{m}")
        names[m] = public(mod)
    S = metrics.SimilarityMatrix(S=np.triu(np.arange(16, dtype=np.float32).reshape(4, 4) / 7.0), k_used=8,
                                 token_aggregation="mean", mode="planning")
    imp = metrics.LayerImportance(w=np.array([0.25, 1.0 / 3.0, 2.0, 1e-9]), source_prompt_count=2)
    cov = [np.array([0.5, 0.123456789]), np.array([1.0, 2.0 / 3.0])]
    out = {"names": names, "similarity_csv": traceio.similarity_csv(S), "importance_csv": traceio.importance_csv(imp),
           "coverage_csv": traceio.coverage_csv(cov), "S": S.S.tolist(), "w": imp.w.tolist(),
           "cov": [c.tolist() for c in cov]}
    json.dump(out, open(os.path.join(HERE, "namespace_ref.json"), "w"), indent=1)

    # device utilities with the reference's signatures (ranking / heads / metrics)
    rng = np.random.default_rng(321)
    # continuous values for the partial tables: with exact ties at the k-th
    # value the reference's set comes from numpy's argpartition (introselect),
    # which is implementation-defined; the full sort (take >= n) is stable
    arr = rng.standard_normal((3, 6, 33)).astype(np.float32)
    ties = rng.integers(0, 5, size=(3, 6, 33)).astype(np.float32)
    P = np.tril(rng.random((6, 30, 30))).astype(np.float32)
    P = (P / P.sum(-1, keepdims=True)).astype(np.float32)
    Hkv = 3
    Pa = np.stack([P[2 * g:2 * g + 2].mean(0, dtype=np.float64) for g in range(Hkv)]).astype(np.float32)
    P2 = np.tril(rng.random((6, 30, 30))).astype(np.float32)
    P2 = (P2 / P2.sum(-1, keepdims=True)).astype(np.float32)
    Pb = np.stack([P2[2 * g:2 * g + 2].mean(0, dtype=np.float64) for g in range(Hkv)]).astype(np.float32)
    tok_idx, tok_valid, tok_den = metrics._token_topk(Pa[1], 7)
    z = {"arr": arr, "table": ranking.topk_table(arr, 9), "table_all": ranking.topk_table(arr, 40),
         "ties": ties, "ties_all": ranking.topk_table(ties, 33),
         "Pa": Pa, "Pb": Pb, "tables": heads.topk_tables(Pa, 5),
         "hs_mean": heads.head_similarity_from_dists(Pa, Pb, 5, "mean"),
         "hs_min": heads.head_similarity_from_dists(Pa, Pb, 5, "min"),
         "hs_idx": heads.head_similarity_from_dists(None, Pb, 5, "mean", idx_a=heads.topk_tables(Pa, 5)),
         "tok_idx": tok_idx, "tok_valid": tok_valid, "tok_den": tok_den}
    np.savez_compressed(os.path.join(HERE, "namespace_ref.npz"), **z)


if __name__ == "__main__":
    main()
