"""The reference's module layout (``paper_2512_16391_b200.kascade``):
every public name each reference module defines exists here
(tests/golden/namespace_ref.json, frozen from the reference), ``install()``
makes ``import kascade`` resolve to it, and the host-side pieces behave
like the reference's (CSV forms verbatim, trace validation / equality,
plan equality, the thread-pool map).  CPU only."""
import importlib
import json
import os
import sys

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "namespace_ref.json")))


def test_every_reference_name_resolves():
    from paper_2512_16391_b200 import kascade
    for module, names in GOLD["names"].items():
        mod = kascade if module == "__root__" else importlib.import_module(f"paper_2512_16391_b200.kascade.{module}")
        missing = [n for n in names if not hasattr(mod, n)]
        assert not missing, (module, missing)


def test_install_aliases_kascade(monkeypatch):
    from paper_2512_16391_b200 import kascade as ns
    for key in [k for k in sys.modules if k == "kascade" or k.startswith("kascade.")]:
        monkeypatch.delitem(sys.modules, key)
    ns.install()
    try:
        import kascade
        from kascade.costmodel import PUBLISHED_BENCH
        from kascade.runner import POOL_POST, run_kascade
        assert kascade is ns and kascade.__version__ == "0.1.0"
        assert POOL_POST == "post" and len(PUBLISHED_BENCH) == 39
        from paper_2512_16391_b200 import compat
        assert run_kascade is compat.run_kascade
    finally:
        for key in [k for k in sys.modules if k == "kascade" or k.startswith("kascade.")]:
            del sys.modules[key]


def test_csv_forms_match_reference():
    from paper_2512_16391_b200.kascade import LayerImportance, SimilarityMatrix, traceio
    S = SimilarityMatrix(S=np.array(GOLD["S"], dtype=np.float32), k_used=8, token_aggregation="mean",
                         mode="planning")
    assert traceio.similarity_csv(S) == GOLD["similarity_csv"]
    imp = LayerImportance(w=np.array(GOLD["w"]), source_prompt_count=2)
    assert traceio.importance_csv(imp) == GOLD["importance_csv"]
    assert traceio.coverage_csv([np.array(c) for c in GOLD["cov"]]) == GOLD["coverage_csv"]


def test_trace_validation_and_equality():
    from paper_2512_16391_b200.kascade import AttentionTrace, InvalidArgumentError
    rng = np.random.default_rng(0)
    Q, K, V = (rng.standard_normal(s).astype(np.float32) for s in ((2, 4, 5, 8), (2, 2, 5, 8), (2, 2, 5, 8)))
    t = AttentionTrace(2, 4, 2, 8, 5, Q, K, V, prompt_id="p")
    assert t.equals(AttentionTrace(2, 4, 2, 8, 5, Q.copy(), K.copy(), V.copy(), prompt_id="p"))
    assert not t.equals(AttentionTrace(2, 4, 2, 8, 5, Q, K, V, prompt_id="q"))
    bad = Q.copy()
    bad[1, 2, 3, 4] = np.nan
    with pytest.raises(InvalidArgumentError, match="non-finite"):
        AttentionTrace(2, 4, 2, 8, 5, bad, K, V)
    X = np.zeros((2, 5, 16), np.float32)
    with pytest.raises(InvalidArgumentError, match="expected"):
        AttentionTrace(2, 4, 2, 8, 5, Q, K, V, X=X, Y=np.zeros((2, 4, 16), np.float32))
    with pytest.raises(InvalidArgumentError, match="together"):
        AttentionTrace(2, 4, 2, 8, 5, Q, K, V, X=X)
    with pytest.raises(InvalidArgumentError, match="divisible"):
        AttentionTrace(2, 3, 2, 8, 5, Q[:, :3], K, V)


def test_plans_equal_and_report_dicts(tmp_path):
    from paper_2512_16391_b200.kascade import AnchorPlan, AnchorPlanCore, LayerReport, RunReport, traceio
    a = AnchorPlan(AnchorPlanCore([0, 2], 2, 0.5))
    traceio.write_plan(tmp_path / "p.json", a)
    assert traceio.plans_equal(a, traceio.read_plan(tmp_path / "p.json"))
    assert not traceio.plans_equal(a, AnchorPlan(AnchorPlanCore([0, 3], 2, 0.5)))
    rep = RunReport(per_layer=[LayerReport(0, "anchor0", 0.0, 1.0), LayerReport(1, "reuse", 0.01, 0.9, 3)],
                    overall={"x": 1.0}, config={"phase": "prefill"})
    back = traceio.report_from_dict(traceio.report_to_dict(rep))
    assert back.per_layer == rep.per_layer and back.overall == rep.overall and back.config == rep.config


def test_parallel_map_keeps_order(monkeypatch):
    from paper_2512_16391_b200.kascade import parallel
    monkeypatch.setenv("KASCADE_THREADS", "4")
    assert parallel.thread_count() == 4
    assert parallel.parallel_map(lambda x: x * x, range(50)) == [x * x for x in range(50)]
    monkeypatch.setenv("KASCADE_THREADS", "zero")
    assert parallel.thread_count() == 1
