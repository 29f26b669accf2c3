"""B200 cost-model presets: the restated arithmetic
is pinned to the reference cost model's own outputs (tests/golden/
costmodel_ref.json, frozen by make_costmodel_golden.py from costmodel.py),
and the measured B200 rows load and report consistently.  CPU only."""
import json
import os
from types import SimpleNamespace

import pytest

from paper_2512_16391_b200 import cli, costmodel as cm
from paper_2512_16391_b200.exceptions import InvalidArgumentError

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "costmodel_ref.json")))


def _close(a, b, tol=1e-12):
    assert abs(a - b) <= tol * max(1.0, abs(b)), (a, b)


def _same_report(got, ref):
    _close(got.kascade_time, ref["kascade_time"])
    _close(got.speedup, ref["speedup"])
    _close(got.baseline_time, ref["baseline_time"])
    assert got.valid == ref["valid"]
    for k, v in ref["per_kind"].items():
        _close(got.per_kind[k], v)


@pytest.mark.parametrize("case", range(len(GOLD["weighted"])))
def test_weighted_pipeline_time_matches_reference(case):
    ph, L, M, fr, n, base, (a0, a, r) = GOLD["weighted"][case]["args"]
    p = cm.CostParams(phase=ph, num_layers=L, num_anchors=M, topk_fraction=fr, seq_len=n, baseline_layer_time=base)
    _same_report(cm.weighted_pipeline_time(p, {"anchor0": a0, "anchor": a, "reuse": r}),
                 GOLD["weighted"][case]["report"])


@pytest.mark.parametrize("phase", ["decode", "prefill"])
def test_ratio_fit_matches_reference_on_h100_rows(phase):
    rows = [SimpleNamespace(**r) for r in GOLD["rows"]]
    fit = cm.fit_ratios_from(rows, phase)
    ref = GOLD["fits"][phase]
    _close(fit.c_gather, ref["c_gather"])
    _close(fit.c_select, ref["c_select"])
    _close(fit.c_pass1, ref["c_pass1"])
    for k, v in ref["max_residual"].items():
        _close(fit.max_residual[k], v)


def test_preset_report_formula_matches_reference():
    # report_from_preset = weighted_pipeline_time(row times, baseline column)
    for r in GOLD["rows"]:
        name = f"table3-{r['phase']}-{r['seq_len']}-k{r['topk_pct']}"
        p = cm.CostParams(phase=r["phase"], topk_fraction=r["topk_pct"] / 100, seq_len=r["seq_len"],
                          baseline_layer_time=r["tl_ms"])
        got = cm.weighted_pipeline_time(p, {"anchor0": r["anchor0_ms"], "anchor": r["anchor_ms"],
                                            "reuse": r["reuse_ms"]})
        _same_report(got, GOLD["presets"][name])


def test_published_table_is_the_reference_default():
    """Reference names give the reference's numbers (costmodel_ref.json)."""
    assert len(cm.PUBLISHED_BENCH) == len(GOLD["rows"])
    for row, ref in zip(cm.PUBLISHED_BENCH, GOLD["rows"]):
        for k, v in ref.items():
            assert getattr(row, k) == v, (row.preset_name, k)
    assert cm.preset_names() == [f"table3-{r['phase']}-{r['seq_len']}-k{r['topk_pct']}" for r in GOLD["rows"]]
    for name, ref in GOLD["presets"].items():
        _same_report(cm.report_from_preset(name), ref)
    for phase in ("decode", "prefill"):
        fit, ref = cm.fit_ratios(phase), GOLD["fits"][phase]
        _close(fit.c_gather, ref["c_gather"])
        _close(fit.c_select, ref["c_select"])
        _close(fit.c_pass1, ref["c_pass1"])
    for case in GOLD["predict"]:
        _same_report(cm.predict_report(*case["args"]), case["report"])
    assert cm.get_preset("table3-decode-131072-k10").kascade_ms == 2.83


def test_b200_presets_load_and_report():
    names = cm.preset_names("b200")
    assert len(names) == len(set(names)) >= 30
    assert "b200-decode-131072-k10" in names and "b200-prefill-131072-k10" in names
    for name in names:
        row = cm.get_preset(name)
        rep = cm.report_from_preset(name)
        assert row.table == "b200" and row.dense_ms > 0 and row.reuse_ms > 0
        assert abs(rep.kascade_time - row.kascade_ms) < 1e-9
        assert abs(rep.speedup - row.speedup) < 1e-9
        assert abs(row.reuse_ratio - row.reuse_ms / row.dense_ms) < 1e-12
    # the sparse reuse layer is cheaper than dense at every measured point
    assert all(r.reuse_ms < r.dense_ms for r in cm.B200_BENCH)
    fit = cm.fit_ratios("decode", "b200")
    assert fit.c_gather != cm.fit_ratios("decode").c_gather
    assert cm.predict_report("decode", 0.1, 131072, table="b200").speedup > 1.0
    with pytest.raises(InvalidArgumentError):
        cm.get_preset("b200-decode-1-k99")
    with pytest.raises(InvalidArgumentError):
        cm.preset_names("h100")


def test_predict_and_validation():
    rep = cm.predict_report("decode", 0.1, 131072)
    assert rep.valid and rep.speedup > 1.0
    assert not cm.predict_report("prefill", 0.1, 8192).valid
    with pytest.raises(InvalidArgumentError):
        cm.predict_ratios("decode", 0.0, 131072)
    with pytest.raises(InvalidArgumentError):
        cm.fit_ratios("training")
    with pytest.raises(InvalidArgumentError):
        cm.CostParams(phase="decode", num_layers=4, num_anchors=5)


def test_cost_cli(tmp_path, capsys):
    out = tmp_path / "c.json"
    for case in GOLD["cli"]:                       # the reference CLI's stdout, verbatim
        assert cli.main(list(case["argv"])) == case["rc"]
        assert capsys.readouterr().out == case["stdout"], case["argv"]
    assert cli.main(["cost", "--preset", "b200-decode-131072-k10", "--out", str(out)]) == 0
    text = capsys.readouterr().out
    assert text.startswith("b200-decode-131072-k10: time=") and "measured B200" in text
    data = json.load(open(out))
    assert data[0]["name"] == "b200-decode-131072-k10" and data[0]["speedup"] > 1
    assert cli.main(["cost", "--ratios", "1.2,0.9,0.1", "--baseline-time", "1"]) == 0
    assert cli.main(["cost", "--ratios", "1,2"]) == 2
    assert cli.main(["cost", "--preset", "nope"]) == 2
    capsys.readouterr()
    assert cli.main(["cost", "--list-presets"]) == 0
    assert capsys.readouterr().out.splitlines()[0] == "table3-decode-8192-k10"
    assert cli.main(["cost", "--list-presets", "--table", "b200"]) == 0
    assert capsys.readouterr().out.splitlines()[0].startswith("b200-")
    assert cli.main(["cost", "--predict", "--phase", "prefill", "--csv"]) == 0
    assert cli.main(["cost", "--predict", "--table", "b200"]) == 0
    assert "predict-b200-decode-131072-k0.1" in capsys.readouterr().out
