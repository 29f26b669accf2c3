"""`python -m paper_2512_16391_b200 run` on the GPU against the reference's
own `kascade run` reports (tests/golden/cli_cases.json): the trace is
streamed from the mmap through the device loader, selections and sparse
attention run on the B200 kernels, and the per-layer fidelity numbers must
match the reference's within the report tolerances below."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2512_16391_b200 import cli

from test_kscd_io import GOLDEN, cases, cli_trace

pytestmark = pytest.mark.gpu

REL_ATOL = 2e-2     # rel-L2 of bf16 engine outputs vs the reference's fp32 outputs
MASS_ATOL = 2e-3


@pytest.mark.parametrize("case", sorted(cases()["cases"]))
def test_run_matches_reference_report(tmp_path, cuda_ok, case):
    path, c = cli_trace(tmp_path)
    spec = c["cases"][case]
    out = tmp_path / "r.json"
    argv = ["run", "--trace", str(path), "--plan", os.path.join(GOLDEN, spec["plan"]), "--phase", spec["phase"],
            "--out", str(out)]
    if spec["mode"]:
        argv += ["--mode", spec["mode"]]
    assert cli.main(argv) == spec["exit"]
    got, want = json.loads(out.read_text()), spec["report"]
    assert [r["kind"] for r in got["per_layer"]] == [r["kind"] for r in want["per_layer"]]
    np.testing.assert_allclose([r["output_rel_err_l2"] for r in got["per_layer"]],
                               [r["output_rel_err_l2"] for r in want["per_layer"]], atol=REL_ATOL)
    np.testing.assert_allclose([r["mass_recovered_mean"] for r in got["per_layer"]],
                               [r["mass_recovered_mean"] for r in want["per_layer"]], atol=MASS_ATOL)
    assert [r["fallback_rows"] for r in got["per_layer"]] == [r["fallback_rows"] for r in want["per_layer"]]
    assert got["config"]["mode"] == want["config"]["mode"]


def test_fail_above_exit_codes(tmp_path, cuda_ok):
    path, _ = cli_trace(tmp_path)
    plan = os.path.join(GOLDEN, "cli_plan_t128.json")
    assert cli.main(["run", "--trace", str(path), "--plan", plan, "--fail-above", "1e-9"]) == cli.EXIT_THRESHOLD
    assert cli.main(["run", "--trace", str(path), "--plan", plan, "--fail-above", "1e9"]) == cli.EXIT_OK


def test_module_entry_point(tmp_path, cuda_ok):
    path, c = cli_trace(tmp_path)
    plan = os.path.join(GOLDEN, "cli_plan_t128.json")
    r = subprocess.run([sys.executable, "-m", "paper_2512_16391_b200", "run", "--trace", str(path), "--plan", plan],
                       capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr
    assert r.stdout.splitlines()[0] == c["cases"]["t128_prefill_remapped"]["stdout"].splitlines()[0]
    assert "anchor0" in r.stdout


def test_cli_workflow_small_head_dim(cuda_ok, tmp_path):
    """gen -> plan -> run (both phases) -> analyze -> report at head_dim 16,
    the reference CLI tests' scale (rows zero-padded to 128 on the device)."""
    from paper_2512_16391_b200 import cli
    t, p, r = tmp_path / "t.kscd", tmp_path / "p.json", tmp_path / "r.json"
    assert cli.main(["gen", "--layers", "4", "--q-heads", "4", "--kv-heads", "2", "--dim", "16", "--tokens", "96",
                     "--seed", "3", "--permute-heads", "--xy", "--out", str(t)]) == 0
    assert cli.main(["plan", "--trace", str(t), "--out", str(p), "--budget", "2", "--k", "16", "--tile-size", "32",
                     "--fraction", "0.25", "--k-min", "8"]) == 0
    assert cli.main(["run", "--trace", str(t), "--plan", str(p), "--out", str(r)]) == 0
    assert cli.main(["run", "--trace", str(t), "--plan", str(p), "--phase", "decode", "--fail-above", "0.5"]) == 0
    assert cli.main(["analyze", "--trace", str(t), "--out-dir", str(tmp_path / "an"), "--importance"]) == 0
    assert (tmp_path / "an" / "similarity.csv").read_text().startswith("row,col,value\n")
    assert cli.main(["report", str(r)]) == 0
