"""The reference's acceptance properties (pkg/tests/test_acceptance.py:
pooling, remapping and sparsity) re-checked on the B200 engine, at the
reference's own shapes (head_dim 32 / 64, served by zero-padding rows to
128).  The inputs are the reference generator's traces (synth.py, byte-identical),
rounded to bf16 as every engine input is.  Needs a B200."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")


def _bf16_trace(t):
    from oracle import kascade_oracle as orc
    from paper_2512_16391_b200 import AttentionTrace
    return AttentionTrace(t.num_layers, t.num_query_heads, t.num_kv_heads, t.head_dim, t.seq_len,
                          *(orc.bf16_round(x) for x in (t.Q, t.K, t.V)), prompt_id=t.prompt_id)


def test_post_softmax_pooling_at_least_as_good_as_pre(cuda_ok):
    """test_acceptance.py:141-165: over 20 seeded heavy-tailed traces (tile
    128, k = 10 %), the mean output error of post-softmax pooling is at most
    that of pre-softmax pooling."""
    import paper_2512_16391_b200 as k
    errs = {"post": [], "pre": []}
    for seed in range(20):
        t = _bf16_trace(k.generate_synthetic(k.SynthConfig(
            num_layers=6, num_query_heads=4, num_kv_heads=2, head_dim=32, seq_len=512, seed=200 + seed,
            layer_correlation=0.9, heavy_tail_temperature=4.0)))
        anchors = [0, 2, 4]
        maps = k.compute_head_maps(t, anchors, k=64)
        for pooling in ("post", "pre"):
            plan = k.AnchorPlan(k.AnchorPlanCore(anchors, 3, 0.0), head_maps=dict(maps), pooling=pooling,
                                k_policy=k.KBudgetPolicy(0.1, 16), tile_size=128)
            _, rep = k.run_kascade(t, plan)
            errs[pooling].append(rep.overall["mean_output_rel_err_l2"])
    post, pre = np.mean(errs["post"]), np.mean(errs["pre"])
    assert post <= pre, (post, pre)


def test_remapping_recovers_mass_on_permuted_traces(cuda_ok):
    """test_acceptance.py:168-195: on head-permuted rho = 1 traces the
    calibrated head maps are the permutation, remapped decode recovers
    >= 0.999 of the attention mass, and the identity map strictly less."""
    import paper_2512_16391_b200 as k
    perms = [[3, 0, 1, 2], [1, 3, 0, 2], [2, 1, 3, 0]]
    remapped, identity = [], []
    for seed, perm in enumerate(perms):
        L = 3
        t = _bf16_trace(k.generate_synthetic(k.SynthConfig(
            num_layers=L, num_query_heads=8, num_kv_heads=4, head_dim=32, seq_len=256, seed=300 + seed,
            layer_correlation=1.0, heavy_tail_temperature=5.0, query_correlation=0.95,
            head_permutations=[[0, 1, 2, 3]] + [perm] * (L - 1))))
        maps = k.compute_head_maps(t, [0], k=32)
        assert all(list(hm.map) == perm for hm in maps.values())
        id_maps = k.compute_head_maps(t, [0], head_map_mode="identity")
        for used, sink in ((maps, remapped), (id_maps, identity)):
            plan = k.AnchorPlan(k.AnchorPlanCore([0], 1, 0.0), head_maps=used, k_policy=k.KBudgetPolicy(0.1, 64),
                                tile_size=128)
            _, rep = k.run_kascade(t, plan, phase="decode")
            sink.append(rep.overall["reuse_mean_mass_recovered"])
    re_mean, id_mean = float(np.mean(remapped)), float(np.mean(identity))
    assert re_mean >= 0.999, re_mean
    assert id_mean < re_mean


def test_sparsity_reproduction_heavy_tail(cuda_ok):
    """test_acceptance.py:198-221: heavy-tailed generator at N = 2048, k =
    10 %: the Top-k covers >= 0.95 of the mass on >= 90 % of the rows of
    layers > 0 (P and coverage on the device), spot-checked against a
    per-row sort."""
    import paper_2512_16391_b200 as k
    t = _bf16_trace(k.generate_synthetic(k.SynthConfig(
        num_layers=3, num_query_heads=4, num_kv_heads=2, head_dim=64, seq_len=2048, seed=400,
        layer_correlation=0.9, heavy_tail_temperature=4.0)))
    kk = 204
    rng = np.random.default_rng(0)
    fractions = []
    for layer in (1, 2):
        P, _ = k.dense_attention(t, layer)
        per_row = k.mass_coverage(P, kk, per_row=True)
        for _ in range(40):
            h, row = int(rng.integers(0, 4)), int(rng.integers(0, 2048))
            vals = np.sort(P[h, row].astype(np.float64))[::-1][:kk]
            assert per_row[h, row] == pytest.approx(vals.sum(), abs=1e-6)
        fractions.append(float((per_row >= 0.95).mean()))
    assert np.mean(fractions) >= 0.90, fractions
