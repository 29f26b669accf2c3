"""The reference's trace-level API on the B200 kernels: the reference's own
test assertions (pkg/tests/test_attention.py, test_runner.py) at d = 128 on
bf16-representable traces, plus the frozen golden vectors.  Needs a B200."""

import numpy as np
import pytest

from conftest import bf16, golden
from oracle import kascade_oracle as orc
from parity import assert_outputs_close, topk_swaps

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")


def trace(Q, K, V, pid="t"):
    from paper_2512_16391_b200 import AttentionTrace
    L, Hq, N, d = Q.shape
    return AttentionTrace(L, Hq, K.shape[1], d, N, Q, K, V, prompt_id=pid)


def rand_trace(seed, L=1, Hq=4, Hkv=2, N=24):
    Q, K, V = orc.random_qkv(seed, L, Hq, Hkv, 128, N)
    return trace(*(orc.bf16_round(x) for x in (Q, K, V)))


# ----------------------------------------------------------- dense_attention
def test_dense_matches_reference_golden(cuda_ok):
    from paper_2512_16391_b200 import compat
    z = golden("dense_small")
    t = trace(bf16(z["Q"]), bf16(z["K"]), bf16(z["V"]))
    P, Y = compat.dense_attention(t, 0)
    assert_outputs_close(Y, z["Y"])
    np.testing.assert_allclose(P, z["P"], atol=2e-5)
    Pn, Yn = compat.dense_attention(t, 0, causal=False)
    assert_outputs_close(Yn, z["Yn"])
    np.testing.assert_allclose(Pn, z["Pn"], atol=2e-5)


def test_dense_single_token_and_causal_zeros(cuda_ok):
    from paper_2512_16391_b200 import compat
    t = rand_trace(1, N=1)
    P, Y = compat.dense_attention(t, 0)
    for h in range(t.num_query_heads):
        assert P[h, 0, 0] == pytest.approx(1.0, abs=1e-6)
        np.testing.assert_allclose(Y[h, 0], t.V[0, t.kv_head_of(h), 0], atol=1e-2)
    t = rand_trace(2, N=16)
    P, _ = compat.dense_attention(t, 0)
    assert (np.triu(P[0], k=1) == 0.0).all()
    np.testing.assert_allclose(P.sum(axis=2), 1.0, atol=1e-5)


def test_dense_gqa_heads_share_kv(cuda_ok):
    from paper_2512_16391_b200 import compat
    t = rand_trace(6)
    t.Q[0, 1] = t.Q[0, 0]
    P, Y = compat.dense_attention(t, 0)
    np.testing.assert_array_equal(P[0], P[1])
    np.testing.assert_array_equal(Y[0], Y[1])


def test_dense_layer_out_of_range(cuda_ok):
    from paper_2512_16391_b200 import InvalidArgumentError, compat
    t = rand_trace(3, L=2)
    with pytest.raises(InvalidArgumentError):
        compat.dense_attention(t, 2)


# ------------------------------------------------------- oracle_topk_indices
def test_topk_contract(cuda_ok):
    from paper_2512_16391_b200 import InvalidArgumentError, compat
    assert compat.oracle_topk_indices(np.array([0.7, 0.1, 0.2]), 1).indices.tolist() == [0]
    assert compat.oracle_topk_indices(np.full(4, 0.25), 2).indices.tolist() == [0, 1]
    assert compat.oracle_topk_indices(np.array([0.2, 0.8]), 5).indices.tolist() == [0, 1]
    with pytest.raises(InvalidArgumentError):
        compat.oracle_topk_indices(np.array([1.0]), 0)

    class Dist:
        weights = np.array([0.1, 0.6, 0.3])
        key_positions = np.array([4, 9, 17])
    assert compat.oracle_topk_indices(Dist(), 2).indices.tolist() == [9, 17]
    rng = np.random.default_rng(0)
    for _ in range(5):
        p = rng.random(64).astype(np.float32)
        assert compat.oracle_topk_indices(p, 8).indices.tolist() == orc.topk_sorted(p, 8).tolist()


# ------------------------------------------------------------ topk_attention
def _full_budget(t, tiles):
    from paper_2512_16391_b200 import TopKIndexSet
    return {(x.kv_head, x.tile_id): TopKIndexSet(x.kv_head, x.tile_id, np.arange(x.causal_bound), x.causal_bound)
            for x in tiles.tiles}


@pytest.mark.parametrize("tile", [24, 128])
def test_full_budget_equals_dense(cuda_ok, tile):
    from paper_2512_16391_b200 import compat, make_tiles
    N = 24 if tile == 24 else 300
    t = rand_trace(4, N=N)
    tiles = make_tiles(N, "prefill", 4, 2, tile_size=min(tile, N))
    res = compat.topk_attention(t, 0, _full_budget(t, tiles), tiles)
    _, Y = compat.dense_attention(t, 0)
    np.testing.assert_allclose(res.Y, Y, atol=1e-2)
    np.testing.assert_allclose(res.mass_recovered, 1.0, atol=1e-4)
    assert not res.fallback_rows


def test_sparse_golden_with_fallback(cuda_ok):
    from paper_2512_16391_b200 import compat, make_tiles, TopKIndexSet
    z = golden("sparse_small")
    t = trace(bf16(z["Q"]), bf16(z["K"]), bf16(z["V"]))
    tiles = make_tiles(72, "prefill", 4, 2, tile_size=16)
    for key in ("", "2"):
        idx, cnt = z["idx" + key], z["cnt" + key]
        sels = {(g, i): TopKIndexSet(g, i, idx[g, i, :cnt[g, i]], int(cnt[g, i])) for g in range(2)
                for i in range(idx.shape[1])}
        res = compat.topk_attention(t, 0, sels, tiles)
        assert_outputs_close(res.Y, z["Y" + key])
        np.testing.assert_allclose(res.mass_recovered, z["mass" + key], atol=1e-3)
        assert sorted(res.fallback_rows) == [tuple(r) for r in z["fallback" + key].tolist()]


def test_selection_errors(cuda_ok):
    from paper_2512_16391_b200 import InvalidArgumentError, TopKIndexSet, compat, make_tiles
    t = rand_trace(12, N=8)
    tiles = make_tiles(8, "prefill", 4, 2, tile_size=4)
    sel = _full_budget(t, tiles)
    sel[(0, 0)] = TopKIndexSet(0, 0, np.array([7]), 1)
    with pytest.raises(InvalidArgumentError):
        compat.topk_attention(t, 0, sel, tiles)
    with pytest.raises(InvalidArgumentError):
        compat.topk_attention(t, 0, {}, tiles)


def test_mass_monotone_under_set_inclusion(cuda_ok):
    from paper_2512_16391_b200 import TopKIndexSet, compat, make_tiles
    t = rand_trace(10, Hq=2, Hkv=1, N=20)
    tiles = make_tiles(20, "prefill", 2, 1, tile_size=20)
    P, _ = compat.dense_attention(t, 0)
    pooled = P.mean(axis=0)[-1]
    base = orc.topk_sorted(pooled, 4)
    grown = np.union1d(base, orc.topk_sorted(pooled, 9))
    small = compat.topk_attention(t, 0, {(0, 0): TopKIndexSet(0, 0, base, 4)}, tiles)
    big = compat.topk_attention(t, 0, {(0, 0): TopKIndexSet(0, 0, grown, len(grown))}, tiles)
    assert (big.mass_recovered >= small.mass_recovered - 1e-5).all()


# --------------------------------------------------------------- run_kascade
def _maps(hm, anchors):
    from paper_2512_16391_b200 import HeadMap
    return {l: HeadMap(l, max(a for a in anchors if a <= l), m) for l, m in enumerate(hm.tolist()) if m[0] >= 0}


def test_run_kascade_remapped_golden_tile64(cuda_ok):
    from paper_2512_16391_b200 import AnchorPlan, AnchorPlanCore, KBudgetPolicy, compat
    z = golden("kascade_prefill")
    t = trace(bf16(z["Q"]), bf16(z["K"]), bf16(z["V"]))
    anchors = z["anchors"].tolist()
    plan = AnchorPlan(AnchorPlanCore(anchors, len(anchors), 0.0), head_maps=_maps(z["head_maps"], anchors),
                      k_policy=KBudgetPolicy(float(z["fraction"]), int(z["k_min"])), tile_size=int(z["tile"]))
    outs, rep = compat.run_kascade(t, plan)
    assert_outputs_close(outs, z["outs"])
    assert rep.per_layer[0].output_rel_err_l2 == 0.0
    np.testing.assert_allclose([r.mass_recovered_mean for r in rep.per_layer], z["mass"], atol=2e-3)
    np.testing.assert_allclose([r.output_rel_err_l2 for r in rep.per_layer], z["rel"], atol=2e-2)


def test_run_kascade_variants_golden(cuda_ok):
    from paper_2512_16391_b200 import AnchorPlan, AnchorPlanCore, KBudgetPolicy, compat, identity_head_map
    z = golden("variants")
    t = trace(bf16(z["Q"]), bf16(z["K"]), bf16(z["V"]))
    core = AnchorPlanCore([0, 1], 2, 0.0)
    pol = KBudgetPolicy(0.5, 4)
    outs, _ = compat.run_kascade(t, AnchorPlan(core, mode="all_heads_pooled", k_policy=pol, tile_size=16))
    assert_outputs_close(outs, z["outs_allheads"])
    plan = AnchorPlan(core, head_maps={2: identity_head_map(2, 2, 1)}, pooling="pre", k_policy=pol, tile_size=16)
    outs, _ = compat.run_kascade(t, plan)
    assert_outputs_close(outs, z["outs_pre"])


def test_run_kascade_config1_prefill_fast_path(cuda_ok):
    import json, os
    from conftest import GOLDEN
    from paper_2512_16391_b200 import AnchorPlan, AnchorPlanCore, KBudgetPolicy, compat
    a = json.load(open(os.path.join(GOLDEN, "golden.json")))["synth_sha256"]["config1"]["args"]
    Q, K, V = orc.synth_qkv(a["L"], a["Hq"], a["Hkv"], a["d"], a["N"], seed=a["seed"], rho=a["rho"])
    t = trace(*(orc.bf16_round(x) for x in (Q, K, V)))
    z = golden("config1")
    plan = AnchorPlan(AnchorPlanCore([0, 2], 2, 0.0), head_maps=_maps(z["head_maps"], [0, 2]),
                      k_policy=KBudgetPolicy(0.1, 128), tile_size=128)
    outs, rep = compat.run_kascade(t, plan)
    assert_outputs_close(outs[:, :, -128:], z["pre_last_tile"])
    np.testing.assert_allclose([r.mass_recovered_mean for r in rep.per_layer], z["pre_mass"], atol=2e-3)


def test_run_kascade_decode_phase_and_degenerate_plan(cuda_ok):
    from paper_2512_16391_b200 import AnchorPlan, AnchorPlanCore, KBudgetPolicy, compat, identity_head_map
    t = rand_trace(28, L=2, N=12)
    plan = AnchorPlan(AnchorPlanCore([0], 1, 0.0), head_maps={1: identity_head_map(2, 1, 0)},
                      k_policy=KBudgetPolicy(0.5, 2), tile_size=128)
    _, rep = compat.run_kascade(t, plan, phase="decode")
    assert rep.config["phase"] == "decode"
    assert rep.overall["mean_mass_recovered"] > 0.5
    # every layer an anchor at full budget = dense (test_runner.py:74-81)
    t = rand_trace(22, L=3, N=32)
    full = AnchorPlan(AnchorPlanCore([0, 1, 2], 3, 0.0), k_policy=KBudgetPolicy(1.0, 32), tile_size=32)
    outs, rep = compat.run_kascade(t, full)
    dense = compat.run_dense(t)
    assert np.abs(outs - dense).max() <= 2e-2
    for r in rep.per_layer:
        assert r.mass_recovered_mean == pytest.approx(1.0, abs=1e-4)


def test_remapped_equals_per_layer_oracle_on_permuted_copies(cuda_ok):
    # test_runner.py:132-147 at d = 128: exact head-permuted copies
    from paper_2512_16391_b200 import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy, compat
    perm = [1, 2, 0]
    Q, K, V = orc.synth_qkv(3, 6, 3, 128, 64, seed=35, rho=1.0, perms=[[0, 1, 2], perm, perm])
    t = trace(*(orc.bf16_round(x) for x in (Q, K, V)))
    pol = KBudgetPolicy(0.2, 4)
    oracle_plan = AnchorPlan(AnchorPlanCore([0, 1, 2], 3, 0.0), k_policy=pol, tile_size=16)
    maps = {l: HeadMap(l, 0, perm) for l in (1, 2)}
    ident = {l: HeadMap(l, 0, [0, 1, 2], "identity") for l in (1, 2)}
    remapped = AnchorPlan(AnchorPlanCore([0], 1, 0.0), head_maps=maps, k_policy=pol, tile_size=16)
    identity = AnchorPlan(AnchorPlanCore([0], 1, 0.0), head_maps=ident, k_policy=pol, tile_size=16)
    o_out, _ = compat.run_kascade(t, oracle_plan)
    r_out, _ = compat.run_kascade(t, remapped)
    i_out, _ = compat.run_kascade(t, identity)
    assert np.abs(r_out - o_out).max() <= 2e-2
    assert np.abs(i_out - o_out).max() > 2e-2


def test_invalid_plans(cuda_ok):
    from paper_2512_16391_b200 import AnchorPlan, AnchorPlanCore, InvalidPlanError, compat, identity_head_map
    t = rand_trace(29, L=3)
    with pytest.raises(InvalidPlanError):
        compat.run_kascade(t, AnchorPlan(AnchorPlanCore([0], 1, 0.0)))
    with pytest.raises(InvalidPlanError):
        compat.run_kascade(t, AnchorPlan(AnchorPlanCore([0, 5], 2, 0.0)))
    maps = {1: identity_head_map(2, reuse_layer=1, anchor_layer=2)}
    with pytest.raises(InvalidPlanError):
        compat.run_kascade(t, AnchorPlan(AnchorPlanCore([0, 2], 2, 0.0), head_maps=maps))
    # a malformed head map raises HeadMap.validate's InvalidArgumentError
    # unchanged, as runner.py:236 -> heads.py:37-47 does
    from paper_2512_16391_b200 import HeadMap, InvalidArgumentError
    for bad in ([0, 1, 0], [0, 2]):
        maps = {1: HeadMap(1, 0, bad), 2: HeadMap(2, 0, [0, 1])}
        with pytest.raises(InvalidArgumentError) as ei:
            compat.run_kascade(t, AnchorPlan(AnchorPlanCore([0], 1, 0.0), head_maps=maps))
        assert not isinstance(ei.value, InvalidPlanError)


# ---------------------------------------------------------- head_dim < 128
@pytest.mark.parametrize("d", [16, 64])
def test_small_head_dim_matches_reference_golden(cuda_ok, d):
    """The reference's tests use d in {4..64}: the engine zero-pads rows to
    128 and passes 1/sqrt(d) (make_smalld_golden.py)."""
    from paper_2512_16391_b200 import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy, compat
    z = golden("smalld")
    t = trace(bf16(z[f"Q{d}"]), bf16(z[f"K{d}"]), bf16(z[f"V{d}"]))
    P, Y = compat.dense_attention(t, 0)
    assert Y.shape == (4, 48, d)
    assert_outputs_close(Y, z[f"Y{d}"])
    np.testing.assert_allclose(P, z[f"P{d}"], atol=2e-5)
    core = AnchorPlanCore([0, 1], 2, 0.0)
    maps = {2: HeadMap(2, 1, [1, 0])}
    pol = KBudgetPolicy(0.25, 4)
    outs, rep = compat.run_kascade(t, AnchorPlan(core, head_maps=maps, k_policy=pol, tile_size=16))
    assert_outputs_close(outs, z[f"outs{d}"])
    np.testing.assert_allclose([r.mass_recovered_mean for r in rep.per_layer], z[f"mass{d}"], atol=2e-3)
    outs, _ = compat.run_kascade(t, AnchorPlan(core, head_maps=maps, pooling="pre", k_policy=pol, tile_size=16))
    assert_outputs_close(outs, z[f"outs_pre{d}"])
    outs, rep = compat.run_kascade(t, AnchorPlan(core, head_maps=maps, k_policy=pol, tile_size=16), phase="decode")
    assert_outputs_close(outs, z[f"outs_dec{d}"])
    np.testing.assert_allclose([r.mass_recovered_mean for r in rep.per_layer], z[f"mass_dec{d}"], atol=2e-3)


def test_small_head_dim_fast_prefill_path_matches_oracle(cuda_ok):
    """d = 64 through the tcgen05 prefill kernels (tile 128, post pooling)
    against the oracle on the same bf16 inputs."""
    from paper_2512_16391_b200 import AnchorPlan, AnchorPlanCore, HeadMap, KBudgetPolicy, compat
    Q, K, V = orc.random_qkv(77, 3, 4, 2, 64, 300)
    Q, K, V = (orc.bf16_round(x) for x in (Q, K, V))
    t = trace(Q, K, V)
    plan = AnchorPlan(AnchorPlanCore([0, 1], 2, 0.0), head_maps={2: HeadMap(2, 1, [1, 0])},
                      k_policy=KBudgetPolicy(0.25, 16), tile_size=128)
    outs, _ = compat.run_kascade(t, plan)
    ref, _ = orc.run_kascade(Q, K, V, [0, 1], {2: [1, 0]}, 0.25, 16, tile_size=128)
    assert_outputs_close(outs, ref)


def test_head_dim_above_128_rejected(cuda_ok):
    from paper_2512_16391_b200 import UnsupportedOperationError, compat
    Q, K, V = orc.random_qkv(5, 1, 2, 1, 160, 8)
    with pytest.raises(UnsupportedOperationError):
        compat.dense_attention(trace(Q, K, V), 0)


def test_topk_attention_non_causal_matches_oracle(cuda_ok):
    """causal=False (attention.py:233: every row sees the whole selection,
    selections may reach past the tile) against the oracle, with the
    mass recovered from the non-causal dense normaliser."""
    from paper_2512_16391_b200 import TopKIndexSet, compat, make_tiles
    t = rand_trace(31, Hq=4, Hkv=2, N=80)
    tiles = make_tiles(80, "prefill", 4, 2, tile_size=32)
    rng = np.random.default_rng(5)
    sels = {}
    for tl in tiles.tiles:
        idx = np.sort(rng.choice(80, size=12, replace=False))          # keys past the tile too
        sels[(tl.kv_head, tl.tile_id)] = TopKIndexSet(tl.kv_head, tl.tile_id, idx, 12)
    res = compat.topk_attention(t, 0, sels, tiles, causal=False)
    P, _ = orc.dense_layer(t.Q[0], t.K[0], t.V[0], causal=False)
    Y, mass, fb = orc.sparse_layer(t.Q[0], t.K[0], t.V[0], {k: v.indices for k, v in sels.items()},
                                   [(tl.start, tl.end, tl.tile_id) for tl in tiles.tiles if tl.kv_head == 0],
                                   causal=False, dense_P=P)
    assert_outputs_close(res.Y, Y)
    np.testing.assert_allclose(res.mass_recovered, mass, atol=1e-3)
    assert res.fallback_rows == [] and fb == []
