"""Model traces: KSCD files written by the reference's
own exporter from its reference transformer (RoPE, GQA, RMSNorm; see
tests/golden/make_exporter_golden.py), run through the B200 engine's `run`
CLI -- mmap -> pinned -> bf16 device loader, the engine's selections and
sparse attention -- and checked against the reports the reference's
`run_kascade` produced on the same files (both phases, both plan modes;
head_dim 64 on the tile-128 performance path, head_dim 128 on 32-row tiles)."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

CASES = json.load(open(os.path.join(GOLDEN, "exporter_cases.json")))["cases"]
REL_ATOL = 2e-2      # per-layer rel-L2 (sparse vs dense) of the engine vs the reference's
MASS_ATOL = 2e-3


def test_exporter_traces_are_the_generated_ones():
    """CPU: the committed files are the generator's bytes, and the engine's
    KSCD reader sees the exporter's shapes."""
    from paper_2512_16391_b200 import kscd_io
    for name, c in CASES.items():
        path = os.path.join(GOLDEN, c["trace"])
        assert hashlib.sha256(open(path, "rb").read()).hexdigest() == c["sha256"], name
        t = kscd_io.TraceFile(path)
        assert (t.num_layers, t.num_query_heads, t.num_kv_heads, t.head_dim, t.seq_len) == \
            (c["layers"], c["q_heads"], c["kv_heads"], c["head_dim"], c["tokens"])


@pytest.mark.gpu
@pytest.mark.parametrize("name,run", [(n, r) for n in sorted(CASES) for r in sorted(CASES[n]["runs"])])
def test_engine_run_matches_reference_on_model_traces(tmp_path, cuda_ok, name, run):
    from paper_2512_16391_b200 import cli
    c = CASES[name]
    phase, mode = run.split("_", 1)
    out = tmp_path / "r.json"
    argv = ["run", "--trace", os.path.join(GOLDEN, c["trace"]), "--plan", os.path.join(GOLDEN, c["plan"]),
            "--phase", phase, "--mode", mode.replace("_", "-"), "--out", str(out)]
    assert cli.main(argv) == 0
    got, want = json.loads(out.read_text()), c["runs"][run]
    assert [r["kind"] for r in got["per_layer"]] == [r["kind"] for r in want["per_layer"]]
    g_rel = [r["output_rel_err_l2"] for r in got["per_layer"]]
    w_rel = [r["output_rel_err_l2"] for r in want["per_layer"]]
    print(f"{name} {run}: rel-L2 engine {np.round(g_rel, 4).tolist()} reference {np.round(w_rel, 4).tolist()}")
    np.testing.assert_allclose(g_rel, w_rel, atol=REL_ATOL)
    np.testing.assert_allclose([r["mass_recovered_mean"] for r in got["per_layer"]],
                               [r["mass_recovered_mean"] for r in want["per_layer"]], atol=MASS_ATOL)
    assert [r["fallback_rows"] for r in got["per_layer"]] == [r["fallback_rows"] for r in want["per_layer"]]
