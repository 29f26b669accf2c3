"""KSCD v1 trace I/O, run reports and the `run` CLI front end, pinned to the
reference (tests/golden/cli_cases.json and conformance_v1.kscd come from
tests/golden/make_golden.py, which runs the reference's own writer, reader
and CLI).  CPU only; the GPU side of the CLI is in test_cli_gpu.py."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import kascade_oracle as orc
from paper_2512_16391_b200 import cli, kscd_io
from paper_2512_16391_b200.exceptions import FormatError
from paper_2512_16391_b200.host_types import AttentionTrace

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CONFORMANCE = os.path.join(GOLDEN, "conformance_v1.kscd")
CONFORMANCE_SHA256 = "2edfef34ff69dfe516906e770d4dddb182a3798ad15cf5868d70fac047af60ae"   # test_traceio.py:40


def cases():
    with open(os.path.join(GOLDEN, "cli_cases.json")) as f:
        return json.load(f)


def random_trace(seed, L=2, Hq=4, Hkv=2, d=8, N=6, xy=False, model_dim=5, pid="t"):
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((L, Hq, N, d)).astype(np.float32)
    K = rng.standard_normal((L, Hkv, N, d)).astype(np.float32)
    V = rng.standard_normal((L, Hkv, N, d)).astype(np.float32)
    X = Y = None
    if xy:
        X = rng.standard_normal((L, N, model_dim)).astype(np.float32)
        Y = rng.standard_normal((L, N, model_dim)).astype(np.float32)
    return AttentionTrace(L, Hq, Hkv, d, N, Q, K, V, X, Y, prompt_id=pid)


def same(a, b):
    for name in ("Q", "K", "V", "X", "Y"):
        x, y = getattr(a, name), getattr(b, name)
        if (x is None) != (y is None) or (x is not None and not np.array_equal(x, y)):
            return False
    return a.prompt_id == b.prompt_id


def cli_trace(tmp_path):
    """The CLI golden trace, regenerated with the oracle generator and our
    writer; its bytes must equal the reference writer's."""
    c = cases()
    a = c["trace_args"]
    Q, K, V = orc.synth_qkv(a["L"], a["Hq"], a["Hkv"], a["d"], a["N"], seed=a["seed"], rho=a["rho"],
                            perms=a["perms"])
    Q, K, V = (orc.bf16_round(x) for x in (Q, K, V))
    t = AttentionTrace(a["L"], a["Hq"], a["Hkv"], a["d"], a["N"], Q, K, V, prompt_id=c["trace_prompt_id"])
    path = tmp_path / "cli.kscd"
    kscd_io.write_trace(path, t)
    return path, c


class TestConformance:
    def test_fixture_sha(self):
        with open(CONFORMANCE, "rb") as f:
            assert hashlib.sha256(f.read()).hexdigest() == CONFORMANCE_SHA256

    def test_header_and_values(self):
        t = kscd_io.read_trace(CONFORMANCE)
        assert (t.num_layers, t.num_query_heads, t.num_kv_heads, t.head_dim, t.seq_len) == (2, 2, 1, 4, 3)
        assert t.prompt_id == "conformance-v1" and t.has_xy() and t.X.shape == (2, 3, 8)
        np.testing.assert_array_equal(t.Q[0, 0, 0], np.float32([-2.8182718753814697, -2.204554319381714,
                                                                6.762521743774414, 2.337858200073242]))

    def test_writer_reproduces_bytes(self, tmp_path):
        out = tmp_path / "re.kscd"
        kscd_io.write_trace(out, kscd_io.read_trace(CONFORMANCE))
        with open(CONFORMANCE, "rb") as f:
            assert out.read_bytes() == f.read()

    def test_cli_trace_bytes_match_reference_writer(self, tmp_path):
        path, c = cli_trace(tmp_path)
        assert hashlib.sha256(path.read_bytes()).hexdigest() == c["trace_sha256"]


class TestRoundTrip:
    @pytest.mark.parametrize("xy", [False, True])
    def test_bit_exact(self, tmp_path, xy):
        t = random_trace(1, xy=xy)
        kscd_io.write_trace(tmp_path / "t.kscd", t)
        assert same(kscd_io.read_trace(tmp_path / "t.kscd"), t)

    def test_many_shapes(self, tmp_path):
        rng = np.random.default_rng(2)
        for i in range(20):
            Hkv = int(rng.integers(1, 4))
            t = random_trace(100 + i, L=int(rng.integers(1, 4)), Hq=Hkv * int(rng.integers(1, 4)), Hkv=Hkv,
                             d=int(rng.integers(1, 9)), N=int(rng.integers(1, 9)), xy=bool(rng.integers(0, 2)),
                             model_dim=int(rng.integers(1, 12)))
            kscd_io.write_trace(tmp_path / f"t{i}.kscd", t)
            assert same(kscd_io.read_trace(tmp_path / f"t{i}.kscd"), t)

    def test_unicode_prompt(self, tmp_path):
        t = random_trace(3, pid="prompt é中文 42")
        kscd_io.write_trace(tmp_path / "u.kscd", t)
        assert kscd_io.read_trace(tmp_path / "u.kscd").prompt_id == t.prompt_id

    def test_layer_views_are_zero_copy_slices(self, tmp_path):
        t = random_trace(4, L=3, Hq=4, Hkv=2, d=8, N=5)
        kscd_io.write_trace(tmp_path / "v.kscd", t)
        tf = kscd_io.TraceFile(str(tmp_path / "v.kscd"))
        for layer in range(3):
            q, k, v = tf.layer_numpy(layer)
            assert np.array_equal(q, t.Q[layer]) and np.array_equal(k, t.K[layer]) and np.array_equal(v, t.V[layer])
        assert (tf.num_layers, tf.num_query_heads, tf.num_kv_heads, tf.head_dim, tf.seq_len) == (3, 4, 2, 8, 5)

    def test_non_finite_rejected(self, tmp_path):
        t = random_trace(5)
        t.K[1, 0, 2, 3] = np.nan
        kscd_io.write_trace(tmp_path / "n.kscd", t)
        with pytest.raises(FormatError, match="K contains non-finite"):
            kscd_io.read_trace(tmp_path / "n.kscd")


@pytest.mark.parametrize("name", sorted(cases()["format_errors"]))
def test_format_errors_match_reference(tmp_path, name):
    """Corrupted copies of the conformance trace: same FormatError message
    and byte offset as the reference reader (traceio.py:75-156)."""
    with open(CONFORMANCE, "rb") as f:
        good = f.read()
    corrupt = {"magic": b"NOPE" + good[4:], "version": good[:4] + (999).to_bytes(2, "little") + good[6:],
               "dtype": good[:26] + bytes([7]) + good[27:], "truncated": good[:-5], "header": b"KSCD\x01",
               "trailing": good + b"xx", "heads": good[:10] + (3).to_bytes(4, "little") + good[14:],
               "zero_dim": good[:6] + (0).to_bytes(4, "little") + good[10:],
               "prompt_utf8": good[:28] + b"\xff" + good[29:]}
    path = tmp_path / f"{name}.kscd"
    path.write_bytes(corrupt[name])
    want = cases()["format_errors"][name]
    if want is None:
        kscd_io.read_trace(path)
        return
    with pytest.raises(FormatError) as err:
        kscd_io.read_trace(path)
    assert str(err.value) == want["message"]
    assert err.value.offset == want["offset"]


class TestReports:
    @pytest.mark.parametrize("case", sorted(cases()["cases"]))
    def test_format_report_matches_reference_stdout(self, tmp_path, case):
        c = cases()["cases"][case]
        p = tmp_path / "r.json"
        p.write_text(json.dumps(c["report"]))
        rep = kscd_io.read_report(p)
        assert kscd_io.format_report(rep) == c["stdout"]
        assert kscd_io.report_to_dict(rep) == c["report"]

    def test_write_read_round_trip(self, tmp_path):
        c = cases()["cases"]["t128_prefill_remapped"]
        p, q = tmp_path / "a.json", tmp_path / "b.json"
        p.write_text(json.dumps(c["report"]))
        kscd_io.write_report(q, kscd_io.read_report(p))
        assert json.loads(q.read_text()) == c["report"]

    def test_bad_json(self, tmp_path):
        (tmp_path / "x.json").write_text("{not json")
        with pytest.raises(FormatError):
            kscd_io.read_report(tmp_path / "x.json")


class TestCliHost:
    """Exit-code contract (cli.py:20-23) for paths that fail before any
    kernel launch."""

    def test_usage_error(self, capsys):
        assert cli.main(["run", "--trace", "x.kscd"]) == cli.EXIT_USAGE
        assert cli.main(["frobnicate"]) == cli.EXIT_USAGE

    def test_missing_trace_is_data_error(self, tmp_path):
        plan = os.path.join(GOLDEN, "cli_plan_t128.json")
        assert cli.main(["run", "--trace", str(tmp_path / "nope.kscd"), "--plan", plan]) == cli.EXIT_DATA

    def test_corrupt_trace_is_data_error(self, tmp_path, capsys):
        (tmp_path / "bad.kscd").write_bytes(b"KSCD\x01")
        plan = os.path.join(GOLDEN, "cli_plan_t128.json")
        assert cli.main(["run", "--trace", str(tmp_path / "bad.kscd"), "--plan", plan]) == cli.EXIT_DATA
        assert "header" in capsys.readouterr().err

    def test_plan_trace_mismatch_is_data_error(self, tmp_path):
        t = random_trace(6, L=2, Hq=8, Hkv=2, d=128, N=8)
        kscd_io.write_trace(tmp_path / "small.kscd", t)
        plan = os.path.join(GOLDEN, "cli_plan_t128.json")      # anchors {0,2} on a 2-layer trace
        assert cli.main(["run", "--trace", str(tmp_path / "small.kscd"), "--plan", plan]) == cli.EXIT_DATA
