"""Freeze the reference's full offline planning pass (pipeline.build_plan:
planning similarity matrix -> DP anchor selection -> head maps,
pipeline.py:76-118) and its layer importance (metrics.py:338-377) on small
synthetic traces, for the GPU calibration tests (tests/test_calibration*.py).
Dev container only (imports /root/reference/pkg/src read-only).

    python tests/golden/make_calib_plan_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from kascade import metrics, pipeline  # noqa: E402
from kascade.trace import AttentionTrace  # noqa: E402
from kascade.traceio import SynthConfig, generate_synthetic  # noqa: E402
from oracle import kascade_oracle as orc  # noqa: E402


def main():
    L, Hq, Hkv, d, N = 6, 4, 2, 128, 256
    rng = np.random.default_rng(61)
    perms = [[0, 1], [1, 0], [0, 1], [0, 1], [1, 0], [0, 1]]   # alternating: non-identity maps
    t = generate_synthetic(SynthConfig(num_layers=L, num_query_heads=Hq, num_kv_heads=Hkv, head_dim=d, seq_len=N,
                                       seed=61, layer_correlation=0.8, head_permutations=perms,
                                       prompt_id="calib-plan"))
    Q, K, V = (orc.bf16_round(x) for x in (t.Q, t.K, t.V))
    t = AttentionTrace(num_layers=L, num_query_heads=Hq, num_kv_heads=Hkv, head_dim=d, seq_len=N, Q=Q, K=K, V=V,
                       prompt_id="calib-plan")
    out = {"Q": orc.bf16_bits(Q), "K": orc.bf16_bits(K), "V": orc.bf16_bits(V)}
    S = metrics.similarity_matrix(t, k=16, token_agg="min", mode="planning", tile_size=64)
    out["S"], out["und"] = S.S, np.array(S.undefined_scores)
    plan = pipeline.build_plan(t, budget=3, k=16, tile_size=64, use_importance=False)
    out["anchors"] = np.array(plan.anchors, np.int32)
    out["maps"] = np.array([plan.head_maps[l].map if l in plan.head_maps else [-1] * Hkv for l in range(L)], np.int32)
    out["objective"] = np.array(plan.core.objective_value)
    # layer importance on small hidden states
    xr = np.random.default_rng(7)
    X = xr.standard_normal((L, N, 24)).astype(np.float32)
    Y = (0.5 * X + xr.standard_normal((L, N, 24))).astype(np.float32)
    X[2, 5] = 0.0                                       # a skipped token (norm below the floor)
    tx = AttentionTrace(num_layers=L, num_query_heads=Hq, num_kv_heads=Hkv, head_dim=d, seq_len=N, Q=Q, K=K, V=V,
                        X=X, Y=Y, prompt_id="calib-xy")
    imp = metrics.layer_importance(tx)
    out["X"], out["Y"], out["w"], out["skipped"] = X, Y, imp.w, np.array(imp.skipped_tokens)
    out["S_weighted"] = metrics.apply_importance(S, imp).S
    np.savez_compressed(os.path.join(HERE, "calib_plan.npz"), **out)
    print("anchors", plan.anchors, "maps", out["maps"].tolist())

    # `kascade plan` (cli.py:195-213) on the CLI golden trace (cli_cases.json)
    import contextlib
    import io
    import json
    import tempfile
    from kascade import cli as ref_cli
    from kascade import traceio as ref_io
    c = json.load(open(os.path.join(HERE, "cli_cases.json")))
    a = c["trace_args"]
    Q, K, V = orc.synth_qkv(a["L"], a["Hq"], a["Hkv"], a["d"], a["N"], seed=a["seed"], rho=a["rho"], perms=a["perms"])
    Q, K, V = (orc.bf16_round(x) for x in (Q, K, V))
    tc = AttentionTrace(num_layers=a["L"], num_query_heads=a["Hq"], num_kv_heads=a["Hkv"], head_dim=a["d"],
                        seq_len=a["N"], Q=Q, K=K, V=V, prompt_id=c["trace_prompt_id"])
    with tempfile.TemporaryDirectory() as td:
        tpath, ppath = os.path.join(td, "t.kscd"), os.path.join(HERE, "cli_plan_built.json")
        ref_io.write_trace(tpath, tc)
        argv = ["plan", "--trace", tpath, "--budget", "2", "--k", "32", "--tile-size", "64", "--fraction", "0.1",
                "--k-min", "16", "--out", ppath]
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            code = ref_cli.main(argv)
        assert code == 0
        meta = {"argv": argv[3:], "stdout": buf.getvalue().replace(ppath, "OUT")}
        json.dump(meta, open(os.path.join(HERE, "cli_plan_built_meta.json"), "w"), indent=1)
        print(buf.getvalue())


if __name__ == "__main__":
    main()


def analyze_golden():
    """`kascade analyze` (cli.py:151-192) on the CLI golden trace, both
    similarity modes, plus `gen` output bytes' hash with --permute-heads."""
    import contextlib
    import hashlib
    import io
    import json
    import tempfile
    from kascade import cli as ref_cli
    from kascade import traceio as ref_io
    c = json.load(open(os.path.join(HERE, "cli_cases.json")))
    a = c["trace_args"]
    Q, K, V = orc.synth_qkv(a["L"], a["Hq"], a["Hkv"], a["d"], a["N"], seed=a["seed"], rho=a["rho"], perms=a["perms"])
    Q, K, V = (orc.bf16_round(x) for x in (Q, K, V))
    tc = AttentionTrace(num_layers=a["L"], num_query_heads=a["Hq"], num_kv_heads=a["Hkv"], head_dim=a["d"],
                        seq_len=a["N"], Q=Q, K=K, V=V, prompt_id=c["trace_prompt_id"])
    out = {}
    with tempfile.TemporaryDirectory() as td:
        tpath = os.path.join(td, "t.kscd")
        ref_io.write_trace(tpath, tc)
        for mode, extra in (("diagnostic", []), ("planning", ["--tile-size", "64", "--token-agg", "min"])):
            od = os.path.join(td, mode)
            argv = ["analyze", "--trace", tpath, "--k", "16", "--mode", mode, "--importance", "--out-dir", od] + extra
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(io.StringIO()):
                assert ref_cli.main(argv) == 0
            out[mode] = {"argv": ["--k", "16", "--mode", mode, "--importance"] + extra,
                         "stdout": buf.getvalue().split(" -> ")[0],
                         "files": {f: open(os.path.join(od, f)).read() for f in sorted(os.listdir(od))}}
        gp = os.path.join(td, "g.kscd")
        with contextlib.redirect_stdout(io.StringIO()):
            ref_cli.main(["gen", "--layers", "3", "--q-heads", "4", "--kv-heads", "2", "--dim", "8", "--tokens", "10",
                          "--permute-heads", "--seed", "5", "--xy", "--out", gp])
        out["gen_sha256"] = hashlib.sha256(open(gp, "rb").read()).hexdigest()
    json.dump(out, open(os.path.join(HERE, "cli_analyze.json"), "w"), indent=1)


if __name__ == "__main__" and os.environ.get("KSCD_ANALYZE_ONLY"):
    analyze_golden()
