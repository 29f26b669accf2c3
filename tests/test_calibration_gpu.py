"""GPU offline calibration against the reference's
own outputs: head similarity, head maps, the planning / diagnostic layer
similarity matrices and the whole build_plan pass, frozen by
tests/golden/make_golden.py (section 9) and make_calib_plan_golden.py.

The device path computes P with bf16 tensor-core products (the reference:
numpy fp32 on the same bf16-representable inputs), so scores agree to
~1e-6; head maps and anchor sets must be identical.  Needs a B200."""
import json
import os
import time

import numpy as np
import pytest

from conftest import GOLDEN, bf16, golden
from oracle import kascade_oracle as orc

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")

ATOL = 2e-4     # scores are ratios in [0, 1]; measured differences are ~1e-6


def trace(Q, K, V, pid="t"):
    from paper_2512_16391_b200 import AttentionTrace
    L, Hq, N, d = Q.shape
    return AttentionTrace(L, Hq, K.shape[1], d, N, Q, K, V, prompt_id=pid)


@pytest.fixture(scope="module")
def tA():
    z5 = golden("kascade_prefill")
    return trace(*(bf16(z5[n]) for n in ("Q", "K", "V")), pid="A")


@pytest.fixture(scope="module")
def t1():
    meta = json.load(open(os.path.join(GOLDEN, "golden.json")))
    a = meta["synth_sha256"]["config1"]["args"]
    Q, K, V = orc.synth_qkv(a["L"], a["Hq"], a["Hkv"], a["d"], a["N"], seed=a["seed"], rho=a["rho"])
    return trace(*(orc.bf16_round(x) for x in (Q, K, V)), pid="config1")


@pytest.mark.parametrize("agg", ["mean", "min"])
def test_head_similarity_matches_reference(cuda_ok, tA, agg):
    from paper_2512_16391_b200 import calibration as cal
    z = golden("calibration")
    for a, b in ((0, 1), (0, 3), (2, 3), (1, 1)):
        got = cal.head_similarity(tA, a, b, k=16, token_agg=agg)
        np.testing.assert_allclose(got, z[f"hs_{agg}_{a}_{b}"], rtol=0, atol=ATOL)


def test_head_maps_match_reference(cuda_ok, tA, t1):
    from paper_2512_16391_b200 import calibration as cal
    z = golden("calibration")
    maps = cal.compute_head_maps(tA, [0, 2], k=16)
    got = np.array([maps[l].map if l in maps else [-1, -1] for l in range(4)], np.int32)
    np.testing.assert_array_equal(got, z["maps_A"])
    assert all(maps[l].anchor_layer == (0 if l < 2 else 2) for l in maps)
    t0 = time.perf_counter()
    maps1 = cal.compute_head_maps(t1, [0, 2], k=64)
    dt = time.perf_counter() - t0
    got1 = np.array([maps1[l].map if l in maps1 else [-1, -1] for l in range(4)], np.int32)
    np.testing.assert_array_equal(got1, z["maps1"])
    np.testing.assert_allclose(cal.head_similarity(t1, 0, 1, k=64), z["hs1_0_1"], rtol=0, atol=ATOL)
    ref_s = json.load(open(os.path.join(GOLDEN, "golden.json")))["ref_seconds_config1_head_maps"]
    print(f"config-1 head maps: GPU {dt:.3f} s vs reference {ref_s} s (8-core host)")
    idm = cal.compute_head_maps(tA, [0, 2], head_map_mode="identity")
    assert sorted(idm) == [1, 3] and all(m.map == [0, 1] for m in idm.values())


@pytest.mark.parametrize("agg", ["mean", "min"])
def test_similarity_matrices_match_reference(cuda_ok, tA, agg):
    from paper_2512_16391_b200 import calibration as cal
    z = golden("calibration")
    S = cal.similarity_matrix(tA, k=16, token_agg=agg, mode="planning", tile_size=64)
    np.testing.assert_allclose(S.S, z[f"S_planning_{agg}"], rtol=0, atol=ATOL)
    assert S.undefined_scores == int(z[f"und_planning_{agg}"]) and S.mode == "planning"
    S = cal.similarity_matrix(tA, k=16, token_agg=agg, mode="diagnostic")
    np.testing.assert_allclose(S.S, z[f"S_diagnostic_{agg}"], rtol=0, atol=ATOL)
    assert S.undefined_scores == int(z[f"und_diagnostic_{agg}"])
    if agg == "min":
        S = cal.similarity_matrix(tA, k=16, token_agg="min", mode="planning", tile_size=64, phase="decode")
        np.testing.assert_allclose(S.S, z["S_planning_decode_min"], rtol=0, atol=ATOL)
        assert S.undefined_scores == int(z["und_planning_decode_min"])


def test_config1_planning_matrix(cuda_ok, t1):
    from paper_2512_16391_b200 import calibration as cal
    z = golden("calibration")
    t0 = time.perf_counter()
    S = cal.similarity_matrix(t1, k=64, token_agg="min", mode="planning", tile_size=128)
    dt = time.perf_counter() - t0
    np.testing.assert_allclose(S.S, z["S1_planning_min"], rtol=0, atol=ATOL)
    assert S.undefined_scores == int(z["und1"])
    ref_s = json.load(open(os.path.join(GOLDEN, "golden.json")))["ref_seconds_config1_planning_matrix"]
    print(f"config-1 planning matrix: GPU {dt:.3f} s vs reference {ref_s} s (8-core host)")


def test_build_plan_matches_reference(cuda_ok):
    from paper_2512_16391_b200 import calibration as cal
    z = golden("calib_plan")
    t = trace(*(bf16(z[n]) for n in ("Q", "K", "V")), pid="calib-plan")
    S = cal.similarity_matrix(t, k=16, token_agg="min", mode="planning", tile_size=64)
    np.testing.assert_allclose(S.S, z["S"], rtol=0, atol=ATOL)
    assert S.undefined_scores == int(z["und"])
    plan = cal.build_plan(t, budget=3, k=16, tile_size=64, use_importance=False)
    assert plan.anchors == z["anchors"].tolist()
    got = np.array([plan.head_maps[l].map if l in plan.head_maps else [-1, -1] for l in range(6)], np.int32)
    np.testing.assert_array_equal(got, z["maps"])
    assert any(m.map != [0, 1] for m in plan.head_maps.values())   # the remap is exercised
    # the plan drives the engine directly
    from paper_2512_16391_b200 import compat
    outs, rep = compat.run_kascade(t, plan)
    assert outs.shape == (6, 4, 256, 128) and np.isfinite(outs).all()


def test_calibration_errors(cuda_ok, tA):
    from paper_2512_16391_b200 import calibration as cal
    from paper_2512_16391_b200.exceptions import InvalidArgumentError
    with pytest.raises(InvalidArgumentError):
        cal.similarity_matrix(tA, k=0)
    with pytest.raises(InvalidArgumentError):
        cal.similarity_matrix(tA, mode="bogus")
    with pytest.raises(InvalidArgumentError):
        cal.compute_head_maps(tA, [0, 2], head_map_mode="bogus")
    with pytest.raises(InvalidArgumentError):
        cal.compute_head_map(np.zeros((2, 3)))


def test_plan_cli_matches_reference_cli(cuda_ok, tmp_path, capsys):
    """`python -m paper_2512_16391_b200 plan` vs the reference's `kascade
    plan` on the CLI golden trace (same arguments, streamed from the KSCD
    file): identical anchors, head maps and policy; objective to 1e-4."""
    from paper_2512_16391_b200 import cli
    from test_kscd_io import cli_trace
    path, _ = cli_trace(tmp_path)
    meta = json.load(open(os.path.join(GOLDEN, "cli_plan_built_meta.json")))
    out = tmp_path / "plan.json"
    assert cli.main(["plan", "--trace", str(path), *meta["argv"], "--out", str(out)]) == 0
    text = capsys.readouterr().out
    assert text.split(" -> ")[0].split(" objective=")[0] == meta["stdout"].split(" objective=")[0]
    got, want = json.load(open(out)), json.load(open(os.path.join(GOLDEN, "cli_plan_built.json")))
    assert abs(got.pop("objective_value") - want.pop("objective_value")) < 1e-4
    got.pop("source_digest", None), want.pop("source_digest", None)
    assert got == want


@pytest.mark.parametrize("mode", ["diagnostic", "planning"])
def test_analyze_cli_matches_reference_cli(cuda_ok, tmp_path, capsys, mode):
    """`python -m paper_2512_16391_b200 analyze` vs the reference's `kascade
    analyze` (cli.py:151-192) on the CLI golden trace: the same files, rows
    and keys; coverage and similarity values within the P tolerance."""
    from paper_2512_16391_b200 import cli
    from test_kscd_io import cli_trace
    path, _ = cli_trace(tmp_path)
    ref = json.load(open(os.path.join(GOLDEN, "cli_analyze.json")))[mode]
    od = tmp_path / "out"
    assert cli.main(["analyze", "--trace", str(path), *ref["argv"], "--out-dir", str(od)]) == 0
    assert capsys.readouterr().out.split(" -> ")[0] == ref["stdout"]
    assert sorted(os.listdir(od)) == sorted(ref["files"])
    for name, text in ref["files"].items():
        got = (od / name).read_text().splitlines()
        want = text.splitlines()
        assert got[0] == want[0] and len(got) == len(want), name
        for g, w in zip(got[1:], want[1:]):
            gk, gv = g.rsplit(",", 1)
            wk, wv = w.rsplit(",", 1)
            assert gk == wk
            assert abs(float(gv) - float(wv)) <= ATOL, (name, g, w)
