"""Pin the CPU oracle (oracle/kascade_oracle.py) to vectors produced by the
reference implementation itself (tests/golden/make_golden.py).  CPU only."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, bf16, golden
from oracle import kascade_oracle as orc


def _sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_generator_bytes_match_reference():
    meta = json.load(open(os.path.join(GOLDEN, "golden.json")))
    for name, ent in meta["synth_sha256"].items():
        a = ent["args"]
        Q, K, V = orc.synth_qkv(a["L"], a["Hq"], a["Hkv"], a["d"], a["N"], seed=a["seed"],
                                rho=a["rho"], perms=a.get("perms"))
        assert _sha(Q, K, V) == ent["sha256"], name


def test_topk_contract_matches_reference():
    z = golden("topk")
    for i in range(int(z["n"])):
        got = orc.topk_sorted(z[f"w{i}"], int(z[f"k{i}"]))
        np.testing.assert_array_equal(got, z[f"idx{i}"])


@pytest.mark.parametrize("n,expect", [(64, 64), (1000, 128), (1280, 128), (4096, 409)])
def test_k_budget_published_rule(n, expect):
    # pkg/tests/test_tiles.py:18-23 pins these four lengths
    assert orc.k_budget(0.1, 128, n) == expect


def test_softmax_known_answer():
    # pkg/tests/test_attention.py:42-46 (frozen from longdouble)
    out = orc.softmax_vec(np.array([1.0, 2.0, 3.0]))
    np.testing.assert_allclose(out, [0.09003057317038046, 0.24472847105479767, 0.6652409557748219],
                               atol=1e-7)


def test_dense_layer_matches_reference():
    z = golden("dense_small")
    Q, K, V = bf16(z["Q"]), bf16(z["K"]), bf16(z["V"])
    P, Y = orc.dense_layer(Q[0], K[0], V[0])
    np.testing.assert_allclose(P, z["P"], rtol=0, atol=1e-7)
    np.testing.assert_allclose(Y, z["Y"], rtol=0, atol=1e-6)
    Pn, Yn = orc.dense_layer(Q[0], K[0], V[0], causal=False)
    np.testing.assert_allclose(Pn, z["Pn"], rtol=0, atol=1e-7)
    np.testing.assert_allclose(Yn, z["Yn"], rtol=0, atol=1e-6)


def test_sparse_layer_with_fallback_matches_reference():
    z = golden("sparse_small")
    Q, K, V = bf16(z["Q"]), bf16(z["K"]), bf16(z["V"])
    N, tile = Q.shape[2], int(z["tile"])
    tiles = orc.prefill_tiles(N, tile)
    P, _ = orc.dense_layer(Q[0], K[0], V[0])
    pooled = orc.layer_pooled(Q[0], K[0], P, tiles, 2, orc.POST)
    sels = orc.select(pooled, {t: e for (_, e, t) in tiles}, float(z["fraction"]), int(z["k_min"]))
    for g in range(2):
        for (_, _, t) in tiles:
            c = z["cnt"][g, t]
            np.testing.assert_array_equal(sels[(g, t)], z["idx"][g, t, :c])
    Y, mass, fb = orc.sparse_layer(Q[0], K[0], V[0], sels, tiles, dense_P=P)
    np.testing.assert_allclose(Y, z["Y"], rtol=0, atol=1e-6)
    np.testing.assert_allclose(mass, z["mass"], rtol=0, atol=1e-6)
    assert sorted(fb) == [tuple(r) for r in z["fallback"].tolist()]
    hand = {(g, t): z["idx2"][g, t, :z["cnt2"][g, t]].astype(np.int64) for g in range(2) for (_, _, t) in tiles}
    Y2, mass2, fb2 = orc.sparse_layer(Q[0], K[0], V[0], hand, tiles, dense_P=P)
    np.testing.assert_allclose(Y2, z["Y2"], rtol=0, atol=1e-6)
    np.testing.assert_allclose(mass2, z["mass2"], rtol=0, atol=1e-6)
    assert sorted(fb2) == [tuple(r) for r in z["fallback2"].tolist()]
    assert len(fb2) > 0  # the fixture exercises the diagonal fallback


def _maps(hm):
    return {l: list(m) for l, m in enumerate(hm.tolist()) if m[0] >= 0}


def test_run_kascade_prefill_remapped_matches_reference():
    z = golden("kascade_prefill")
    Q, K, V = bf16(z["Q"]), bf16(z["K"]), bf16(z["V"])
    maps = _maps(z["head_maps"])
    assert any(m != sorted(m) for m in maps.values())  # non-identity remap exercised
    outs, rep = orc.run_kascade(Q, K, V, z["anchors"].tolist(), maps, float(z["fraction"]),
                                int(z["k_min"]), tile_size=int(z["tile"]))
    np.testing.assert_allclose(outs, z["outs"], rtol=0, atol=1e-6)
    np.testing.assert_allclose([r["rel"] for r in rep], z["rel"], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose([r["mass"] for r in rep], z["mass"], rtol=1e-6)


def test_mode_variants_match_reference():
    z = golden("variants")
    Q, K, V = bf16(z["Q"]), bf16(z["K"]), bf16(z["V"])
    outs, _ = orc.run_kascade(Q, K, V, [0, 1], {}, 0.5, 4, tile_size=16, mode=orc.ALL_HEADS_POOLED)
    np.testing.assert_allclose(outs, z["outs_allheads"], rtol=0, atol=1e-6)
    outs, _ = orc.run_kascade(Q, K, V, [0, 1], {2: [0, 1]}, 0.5, 4, tile_size=16, pooling=orc.PRE)
    np.testing.assert_allclose(outs, z["outs_pre"], rtol=0, atol=1e-6)


@pytest.mark.parametrize("d", [16, 64])
def test_small_head_dim_matches_reference(d):
    """The reference's own small-d traces (make_smalld_golden.py)."""
    z = golden("smalld")
    Q, K, V = bf16(z[f"Q{d}"]), bf16(z[f"K{d}"]), bf16(z[f"V{d}"])
    P, Y = orc.dense_layer(Q[0], K[0], V[0])
    np.testing.assert_allclose(P, z[f"P{d}"], rtol=0, atol=1e-6)
    np.testing.assert_allclose(Y, z[f"Y{d}"], rtol=0, atol=1e-6)
    for key, kw in ((f"outs{d}", {}), (f"outs_pre{d}", {"pooling": orc.PRE}), (f"outs_dec{d}", {"phase": "decode"})):
        outs, rep = orc.run_kascade(Q, K, V, [0, 1], {2: [1, 0]}, 0.25, 4, tile_size=16, **kw)
        np.testing.assert_allclose(outs, z[key], rtol=0, atol=1e-6)
        if key.startswith("outs_dec"):
            np.testing.assert_allclose([r["mass"] for r in rep], z[f"mass_dec{d}"], rtol=1e-6)
        elif not key.startswith("outs_pre"):
            np.testing.assert_allclose([r["mass"] for r in rep], z[f"mass{d}"], rtol=1e-6)


@pytest.fixture(scope="module")
def config1():
    meta = json.load(open(os.path.join(GOLDEN, "golden.json")))
    a = meta["synth_sha256"]["config1"]["args"]
    Q, K, V = orc.synth_qkv(a["L"], a["Hq"], a["Hkv"], a["d"], a["N"], seed=a["seed"], rho=a["rho"])
    return [orc.bf16_round(x) for x in (Q, K, V)], golden("config1")


def test_decode_step_driver_bit_equal_to_reference_decode(config1):
    (Q, K, V), z = config1
    maps = _maps(z["head_maps"])
    Y, sels, _ = orc.decode_step(Q[:, :, -1], K, V, z["anchors"].tolist(), maps, 0.1, 128)
    for l in range(4):
        for g in range(2):
            np.testing.assert_array_equal(sels[l][g], z["dec_sel"][l, g])
    np.testing.assert_array_equal(Y, z["dec_Y"])


def test_prefill_tile_driver_matches_reference(config1):
    (Q, K, V), z = config1
    N, tile = Q.shape[2], 128
    maps = _maps(z["head_maps"])
    last = N // tile - 1
    for ai, a in enumerate(z["anchors"].tolist()):
        for g in range(2):
            for t in (0, 5, last):
                sel, _ = orc.prefill_tile_select(Q[a], K[a], g, 4, t * tile, (t + 1) * tile, 0.1, 128)
                np.testing.assert_array_equal(sel, z["pre_idx"][ai, g, t, :sel.size])
    # last tile outputs of every layer through the per-tile driver
    for l in range(4):
        anchor = max(a for a in z["anchors"].tolist() if a <= l)
        for g in range(2):
            src = maps[l][g] if l in maps else g
            sel, _ = orc.prefill_tile_select(Q[anchor], K[anchor], src, 4, N - tile, N, 0.1, 128)
            if l == 0:
                Pt = orc.prefill_tile_rows(Q[0], K[0], g, 4, N - tile, N)
                y = np.stack([Pt[j] @ V[0, g] for j in range(4)])
                np.testing.assert_allclose(y, z["pre_last_tile"][0, g * 4:(g + 1) * 4], atol=1e-6)
                continue
            y, _, _ = orc.sparse_tile(Q[l], K[l], V[l], g, 4, N - tile, N, sel)
            np.testing.assert_allclose(y, z["pre_last_tile"][l, g * 4:(g + 1) * 4], rtol=0, atol=1e-6)


# ---------------------------------------------------------------- calibration
# Offline calibration: head similarity, head maps and
# the layer similarity matrix in both modes, frozen from the reference
# (heads.py:67-143, pipeline.py:31-73, metrics.py:205-335) by make_golden.py.

@pytest.fixture(scope="module")
def calib():
    z5 = golden("kascade_prefill")
    qkv = tuple(bf16(z5[n]) for n in ("Q", "K", "V"))
    return qkv, golden("calibration")


@pytest.mark.parametrize("agg", ["mean", "min"])
def test_head_similarity_matches_reference(calib, agg):
    (Q, K, V), z = calib
    for a, b in ((0, 1), (0, 3), (2, 3), (1, 1)):
        np.testing.assert_allclose(orc.head_similarity(Q, K, V, a, b, k=16, how=agg), z[f"hs_{agg}_{a}_{b}"],
                                   rtol=0, atol=1e-6)


def test_head_maps_match_reference(calib, config1):
    (Q, K, V), z = calib
    maps = orc.head_maps(Q, K, V, [0, 2], k=16)
    got = np.array([maps.get(l, [-1, -1]) for l in range(4)], np.int32)
    np.testing.assert_array_equal(got, z["maps_A"])
    (Q1, K1, V1), _ = config1
    maps1 = orc.head_maps(Q1, K1, V1, [0, 2], k=64)
    np.testing.assert_array_equal(np.array([maps1.get(l, [-1, -1]) for l in range(4)], np.int32), z["maps1"])
    np.testing.assert_allclose(orc.head_similarity(Q1, K1, V1, 0, 1, k=64), z["hs1_0_1"], rtol=0, atol=1e-6)


@pytest.mark.parametrize("agg", ["mean", "min"])
def test_similarity_matrices_match_reference(calib, agg):
    (Q, K, V), z = calib
    S, und = orc.planning_matrix(Q, K, V, k=16, how=agg, tile=64)
    np.testing.assert_allclose(S, z[f"S_planning_{agg}"], rtol=0, atol=1e-6)
    assert und == int(z[f"und_planning_{agg}"])
    S, und = orc.diagnostic_matrix(Q, K, V, k=16, how=agg)
    np.testing.assert_allclose(S, z[f"S_diagnostic_{agg}"], rtol=0, atol=1e-6)
    assert und == int(z[f"und_diagnostic_{agg}"])
    if agg == "min":
        S, und = orc.planning_matrix(Q, K, V, k=16, how="min", tile=64, phase="decode")
        np.testing.assert_allclose(S, z["S_planning_decode_min"], rtol=0, atol=1e-6)
        assert und == int(z["und_planning_decode_min"])
