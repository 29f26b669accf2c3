"""Reference-style usage through ``import kascade`` after
``paper_2512_16391_b200.kascade.install()``: the reference's own workflow
(generate a synthetic trace, build a plan, run the anchor/reuse pipeline in
both phases, write / read the report) on the B200 engine, at the small head
dims the reference's tests use, checked against the oracle.  Needs a B200."""
import sys

import numpy as np
import pytest

from oracle import kascade_oracle as orc
from parity import assert_outputs_close_rel

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")


@pytest.fixture()
def kascade():
    from paper_2512_16391_b200.kascade import install
    saved = {k: v for k, v in sys.modules.items() if k == "kascade" or k.startswith("kascade.")}
    install()
    import kascade as k
    yield k
    for key in [k for k in sys.modules if k == "kascade" or k.startswith("kascade.")]:
        del sys.modules[key]
    sys.modules.update(saved)


@pytest.mark.parametrize("d", [16, 64, 128])
def test_reference_workflow_through_install(cuda_ok, kascade, tmp_path, d):
    from kascade.runner import POOL_POST
    from kascade.traceio import read_report, write_report
    cfg = kascade.SynthConfig(num_layers=4, num_query_heads=4, num_kv_heads=2, head_dim=d, seq_len=96, seed=3,
                              layer_correlation=0.9, head_permutations=[[0, 1], [1, 0], [1, 0], [0, 1]])
    trace = kascade.generate_synthetic(cfg)
    trace = kascade.AttentionTrace(trace.num_layers, trace.num_query_heads, trace.num_kv_heads, d, trace.seq_len,
                                   *(orc.bf16_round(x) for x in (trace.Q, trace.K, trace.V)), prompt_id="w")
    plan = kascade.build_plan([trace], budget=2, k=16, tile_size=32,
                              k_policy=kascade.KBudgetPolicy(fraction=0.25, k_min=8))
    assert plan.core.anchors[0] == 0 and plan.pooling == POOL_POST
    maps = {l: list(hm.map) for l, hm in plan.head_maps.items()}
    for phase in ("prefill", "decode"):
        outs, rep = kascade.run_kascade(trace, plan, phase=phase)
        want, _ = orc.run_kascade(trace.Q, trace.K, trace.V, list(plan.core.anchors), maps, 0.25, 8,
                                  tile_size=32, phase=phase)
        assert outs.shape == (4, 4, 96, d)
        assert_outputs_close_rel(outs, want)
        assert rep.per_layer[0].output_rel_err_l2 == 0.0
        write_report(tmp_path / f"{phase}.json", rep)
        back = read_report(tmp_path / f"{phase}.json")
        assert [r.kind for r in back.per_layer] == [r.kind for r in rep.per_layer]
    dense = kascade.run_dense(trace)
    for layer in range(4):
        _, Y = orc.dense_layer(trace.Q[layer], trace.K[layer], trace.V[layer])
        assert_outputs_close_rel(dense[layer], Y)
