"""The reference's small path utilities (pool_presoftmax / pool_postsoftmax,
layer_distribution, mass_coverage, sim_score, pooled_all_heads_topk,
AttentionDistribution) on the device, against the reference's own outputs
(tests/golden/utils_ref.npz).  Needs a B200."""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")


def test_utilities_match_reference(cuda_ok):
    import paper_2512_16391_b200 as k
    z = golden("utils_ref")
    np.testing.assert_allclose(k.pool_presoftmax(z["q_tile"]), z["pre"], rtol=0, atol=1e-7)
    rows = [z[f"row{i}"] for i in range(5)]
    np.testing.assert_allclose(k.pool_postsoftmax(rows), z["post"], rtol=0, atol=1e-7)
    np.testing.assert_allclose(k.layer_distribution(z["P"]), z["layer_dist"], rtol=0, atol=1e-7)
    np.testing.assert_allclose(k.mass_coverage(z["P"], 7), z["cov_mean"], rtol=0, atol=1e-6)
    np.testing.assert_allclose(k.mass_coverage(z["P"], 7, per_row=True), z["cov_rows"], rtol=0, atol=1e-6)
    assert k.sim_score(z["pb"], z["ia"], z["ib"]) == pytest.approx(float(z["sim"]), abs=1e-7)
    sel = k.pooled_all_heads_topk(z["gd"], 9, tile_id=4)
    np.testing.assert_array_equal(sel.indices, z["pooled_sel"])
    assert sel.kv_head == -1 and sel.tile_id == 4


def test_utility_errors(cuda_ok):
    import paper_2512_16391_b200 as k
    with pytest.raises(k.InvalidArgumentError):
        k.pool_postsoftmax([])
    with pytest.raises(k.InvalidArgumentError):
        k.pool_presoftmax(np.zeros((0, 4)))
    with pytest.raises(k.InvalidArgumentError):
        k.mass_coverage(np.ones((2, 2)), 0)
    with pytest.raises(k.InvalidArgumentError):
        k.sim_score(np.ones(4), [0, 1], [0])
    with pytest.raises(k.UndefinedScoreError):
        k.sim_score(np.zeros(4), [0, 1], [2, 3])
    d = k.AttentionDistribution(np.array([0.5, 0.5]), np.array([3, 1]))
    with pytest.raises(k.InvalidArgumentError):
        d.validate()
    k.AttentionDistribution(np.array([0.25, 0.75]), np.array([1, 3])).validate()
