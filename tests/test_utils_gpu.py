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


def test_namespace_device_utilities_match_reference(cuda_ok):
    """ranking.topk_table, heads.topk_tables / head_similarity_from_dists /
    group_distributions and metrics._token_topk with the reference's
    signatures (tests/golden/namespace_ref.npz)."""
    from paper_2512_16391_b200.kascade import heads, metrics, ranking
    z = golden("namespace_ref")
    np.testing.assert_array_equal(ranking.topk_table(z["arr"], 9), z["table"])
    np.testing.assert_array_equal(ranking.topk_table(z["arr"], 40), z["table_all"])
    np.testing.assert_array_equal(ranking.topk_table(z["ties"], 33), z["ties_all"])   # stable: index ascending
    # partial tables with ties at the k-th value keep the smallest indices
    # (the reference's argpartition picks an implementation-defined subset;
    # every masked sum over the set is the same either way)
    part = ranking.topk_table(z["ties"], 9)
    np.testing.assert_array_equal(part, z["ties_all"][..., :9])
    np.testing.assert_array_equal(heads.topk_tables(z["Pa"], 5), z["tables"])
    for key, kw in (("hs_mean", {"token_agg": "mean"}), ("hs_min", {"token_agg": "min"})):
        np.testing.assert_allclose(heads.head_similarity_from_dists(z["Pa"], z["Pb"], 5, **kw), z[key],
                                   rtol=0, atol=1e-7)
    np.testing.assert_allclose(heads.head_similarity_from_dists(None, z["Pb"], 5, "mean", idx_a=z["tables"]),
                               z["hs_idx"], rtol=0, atol=1e-7)
    idx, valid, den = metrics._token_topk(z["Pa"][1], 7)
    np.testing.assert_array_equal(idx, z["tok_idx"])
    np.testing.assert_array_equal(valid, z["tok_valid"])
    np.testing.assert_allclose(den, z["tok_den"], rtol=1e-12)


def test_namespace_group_distributions_match_oracle(cuda_ok):
    """heads.group_distributions: the group mean of dense P, fp64 -> fp32."""
    from oracle import kascade_oracle as orc
    from paper_2512_16391_b200 import AttentionTrace
    from paper_2512_16391_b200.kascade import heads
    Q, K, V = (orc.bf16_round(x) for x in orc.random_qkv(9, 1, 4, 2, 64, 40))
    t = AttentionTrace(1, 4, 2, 64, 40, Q, K, V)
    P, _ = orc.dense_layer(Q[0], K[0], V[0])
    want = np.stack([P[2 * g:2 * g + 2].mean(axis=0, dtype=np.float64) for g in range(2)]).astype(np.float32)
    np.testing.assert_allclose(heads.group_distributions(t, 0), want, rtol=0, atol=2e-6)
    np.testing.assert_allclose(heads.group_distributions(t, 0, P=P), want, rtol=0, atol=1e-7)
