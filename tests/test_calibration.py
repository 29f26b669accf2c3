"""Host arithmetic of the GPU calibration module:
the anchor DP, the importance weights and the score aggregation, pinned to
the reference's outputs (tests/golden/calib_plan.npz) and to brute force.
CPU only; the device steps are tests/test_calibration_gpu.py."""
import itertools

import numpy as np
import pytest

from conftest import golden
from paper_2512_16391_b200 import calibration as cal
from paper_2512_16391_b200.exceptions import InvalidArgumentError, UnsupportedOperationError


def _brute(mat, M):
    L = mat.shape[0]
    best, arg = -np.inf, None
    for rest in itertools.combinations(range(1, L), M - 1):
        a = [0, *rest]
        v = cal.objective(mat, a)
        if v > best:                      # strict: keeps the lexicographically first optimum
            best, arg = v, a
    return arg, best


@pytest.mark.parametrize("seed,L,M", [(0, 6, 3), (1, 8, 4), (2, 7, 1), (3, 9, 9), (4, 10, 5)])
def test_select_anchors_is_the_optimum_with_lexicographic_ties(seed, L, M):
    rng = np.random.default_rng(seed)
    mat = np.triu(rng.random((L, L)).astype(np.float32))
    if seed == 4:                          # plant exact ties
        mat = np.triu(np.ones((L, L), np.float32))
    core = cal.select_anchors(mat, M)
    ref, best = _brute(mat.astype(np.float64), M)
    assert core.anchors == ref and abs(core.objective_value - best) < 1e-12


def test_select_anchors_on_reference_planning_matrix():
    z = golden("calib_plan")
    core = cal.select_anchors(z["S"], 3)
    assert core.anchors == z["anchors"].tolist()
    assert core.objective_value == float(z["objective"])
    with pytest.raises(InvalidArgumentError):
        cal.select_anchors(z["S"], 0)
    with pytest.raises(InvalidArgumentError):
        cal.objective(z["S"], [1, 2])


def test_layer_importance_matches_reference():
    z = golden("calib_plan")

    class T:
        num_layers, num_query_heads, num_kv_heads, prompt_id = 6, 4, 2, "xy"
        X, Y = z["X"], z["Y"]

    imp = cal.layer_importance(T())
    np.testing.assert_allclose(imp.w, z["w"], rtol=0, atol=1e-12)
    assert imp.skipped_tokens == int(z["skipped"])
    S = cal.SimilarityMatrix(S=z["S"], k_used=16, token_aggregation="min", mode="planning")
    np.testing.assert_array_equal(cal.apply_importance(S, imp).S, z["S_weighted"])

    class NoXY(T):
        X = None
    with pytest.raises(UnsupportedOperationError):
        cal.layer_importance(NoXY())


def test_score_aggregation_rules():
    num = np.array([[[1.0, 2.0, 0.5]], [[0.0, 0.0, 0.0]]])     # [I=2][J=1][rows=3]
    den = np.array([[2.0, 0.0, 1.0]])                          # row 1 undefined
    hs = cal._aggregate_scores(num, den, "mean")
    assert hs.shape == (2, 1)
    assert hs[0, 0] == np.float32(0.5) / 2 + np.float32(0.5) / 2 and hs[1, 0] == 0.0
    assert cal._aggregate_scores(num, den, "min")[0, 0] == 0.5
    with pytest.raises(InvalidArgumentError):
        cal.head_similarity_from_dists(None, None, None, token_agg="median")


def test_gen_cli_matches_reference_bytes(tmp_path, capsys):
    """`gen` (cli.py:117-148) writes the reference's exact bytes (X/Y and
    per-layer kv-head permutations included)."""
    import hashlib
    import json
    import os
    from conftest import GOLDEN
    from paper_2512_16391_b200 import cli
    want = json.load(open(os.path.join(GOLDEN, "cli_analyze.json")))["gen_sha256"]
    out = tmp_path / "g.kscd"
    assert cli.main(["gen", "--layers", "3", "--q-heads", "4", "--kv-heads", "2", "--dim", "8", "--tokens", "10",
                     "--permute-heads", "--seed", "5", "--xy", "--out", str(out)]) == 0
    assert hashlib.sha256(out.read_bytes()).hexdigest() == want
    assert capsys.readouterr().out.startswith(f"wrote {out}: layers=3 q_heads=4 kv_heads=2 dim=8 tokens=10 xy=1")


def test_report_cli(tmp_path, capsys):
    import json
    import os
    from conftest import GOLDEN
    from paper_2512_16391_b200 import cli
    case = json.load(open(os.path.join(GOLDEN, "cli_cases.json")))["cases"]["t128_prefill_remapped"]
    p = tmp_path / "r.json"
    p.write_text(json.dumps(case["report"]))
    assert cli.main(["report", str(p)]) == 0
    assert capsys.readouterr().out == case["stdout"]
    q = tmp_path / "other.json"
    q.write_text('{"b": 1, "a": [2]}')
    assert cli.main(["report", str(q)]) == 0
    assert json.loads(capsys.readouterr().out) == {"a": [2], "b": 1}


@pytest.mark.parametrize("seed,L,M", [(5, 7, 3), (6, 9, 4), (7, 6, 6)])
def test_exhaustive_select_agrees_with_dp(seed, L, M):
    rng = np.random.default_rng(seed)
    mat = np.triu(rng.random((L, L)).astype(np.float32))
    ex, dp = cal.exhaustive_select(mat, M), cal.select_anchors(mat, M)
    assert ex.anchors == dp.anchors and abs(ex.objective_value - dp.objective_value) < 1e-12
    with pytest.raises(UnsupportedOperationError):
        cal.exhaustive_select(np.zeros((40, 40)), 12)
