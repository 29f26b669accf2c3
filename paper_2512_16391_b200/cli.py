"""``python -m paper_2512_16391_b200 gen|analyze|plan|run|cost|report``: the
reference CLI (cli.py:33-112) on this package -- ``run`` on the B200 engine,
``analyze`` / ``plan`` on the GPU calibration (calibration.py), ``cost`` over
the paper's Table 3 or the measured B200 presets (costmodel.py), ``gen`` / ``report`` with the same trace,
plan and report formats.  Exit codes as in the reference (cli.py:20-23).

    python -m paper_2512_16391_b200 run --trace t.kscd --plan p.json \\
        [--phase prefill|decode] [--mode remapped|all-heads-pooled] [--out report.json] [--fail-above X]
    python -m paper_2512_16391_b200 plan --trace a.kscd [b.kscd ...] --out plan.json [--budget 5] [--k 64]
        [--token-agg min|mean] [--tile-size 128] [--pooling post|pre] [--mode remapped|all-heads-pooled]
        [--fraction 0.1] [--k-min 128] [--no-importance]
    python -m paper_2512_16391_b200 cost [--preset table3-decode-131072-k10 ...] [--list-presets] [--table b200]
        [--ratios a0,a,r | --predict] [--phase] [--fraction] [--seq-len] [--layers] [--anchors]
        [--baseline-time] [--csv] [--out results.json]

Exit codes follow the reference (cli.py:20-23): 0 ok, 1 usage, 2 data or
format error, 3 threshold exceeded.
"""

import argparse
import sys

EXIT_OK, EXIT_USAGE, EXIT_DATA, EXIT_THRESHOLD = 0, 1, 2, 3


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise SystemExit(EXIT_USAGE)


def build_parser():
    p = _Parser(prog="kascade-b200", description=__doc__)
    sub = p.add_subparsers(dest="command", required=True)
    gen = sub.add_parser("gen", help="generate a synthetic trace file")
    gen.add_argument("--layers", type=int, required=True)
    gen.add_argument("--q-heads", type=int, required=True)
    gen.add_argument("--kv-heads", type=int, required=True)
    gen.add_argument("--dim", type=int, required=True)
    gen.add_argument("--tokens", type=int, required=True)
    gen.add_argument("--rho", type=float, default=1.0, help="cross-layer key correlation in [0, 1]")
    gen.add_argument("--seed", type=int, default=0)
    gen.add_argument("--temperature", type=float, default=4.0, help="query sharpness")
    gen.add_argument("--query-correlation", type=float, default=0.85)
    gen.add_argument("--layer0-temperature-scale", type=float, default=1.0)
    gen.add_argument("--permute-heads", action="store_true",
                     help="random kv-head permutation per layer (layer 0 stays identity)")
    gen.add_argument("--xy", action="store_true", help="include attention-block input/output hidden states")
    gen.add_argument("--prompt-id", default="")
    gen.add_argument("--out", required=True)
    analyze = sub.add_parser("analyze", help="coverage, similarity and importance reports (GPU)")
    analyze.add_argument("--trace", nargs="+", required=True)
    analyze.add_argument("--k", type=int, default=64)
    analyze.add_argument("--token-agg", choices=["mean", "min"], default="mean")
    analyze.add_argument("--mode", choices=["diagnostic", "planning"], default="diagnostic")
    analyze.add_argument("--tile-size", type=int, default=128)
    analyze.add_argument("--importance", action="store_true")
    analyze.add_argument("--out-dir", default=".")
    report = sub.add_parser("report", help="render a saved report file as text")
    report.add_argument("file")
    run = sub.add_parser("run", help="execute the anchor/reuse pipeline on the GPU and report fidelity vs dense")
    run.add_argument("--trace", required=True)
    run.add_argument("--plan", required=True)
    run.add_argument("--phase", choices=["prefill", "decode"], default="prefill")
    run.add_argument("--mode", choices=["remapped", "all-heads-pooled"], default=None)
    run.add_argument("--out", default=None)
    run.add_argument("--fail-above", type=float, default=None)
    run.add_argument("--engine", choices=["b200"], default="b200",
                     help="accepted for parity with `kascade run --engine b200`; there is no other engine")
    plan = sub.add_parser("plan", help="select anchors and head maps on the GPU, write a plan file")
    plan.add_argument("--trace", nargs="+", required=True)
    plan.add_argument("--budget", type=int, default=5)
    plan.add_argument("--k", type=int, default=64)
    plan.add_argument("--token-agg", choices=["mean", "min"], default="min")
    plan.add_argument("--tile-size", type=int, default=128)
    plan.add_argument("--pooling", choices=["post", "pre"], default="post")
    plan.add_argument("--mode", choices=["remapped", "all-heads-pooled"], default="remapped")
    plan.add_argument("--fraction", type=float, default=0.1)
    plan.add_argument("--k-min", type=int, default=128)
    plan.add_argument("--no-importance", action="store_true",
                      help="skip importance weighting even when X/Y are present")
    plan.add_argument("--out", required=True)
    cost = sub.add_parser("cost", help="weighted-average pipeline time and speedup (B200 presets)")
    cost.add_argument("--preset", action="append", default=None,
                      help="preset name, e.g. table3-decode-131072-k10 or b200-decode-131072-k10 (repeatable)")
    cost.add_argument("--list-presets", action="store_true")
    cost.add_argument("--table", choices=["table3", "b200"], default="table3",
                      help="preset table for --list-presets, --predict and the default listing: the paper's "
                           "H100 Table 3 (reference default) or the rows measured on B200")
    cost.add_argument("--ratios", default=None, help="anchor0,anchor,reuse per-layer times")
    cost.add_argument("--predict", action="store_true", help="use the ratio model fitted on --table's rows")
    cost.add_argument("--phase", choices=["decode", "prefill"], default="decode")
    cost.add_argument("--fraction", type=float, default=0.1)
    cost.add_argument("--seq-len", type=int, default=131072)
    cost.add_argument("--layers", type=int, default=32)
    cost.add_argument("--anchors", type=int, default=5)
    cost.add_argument("--baseline-time", type=float, default=1.0)
    cost.add_argument("--csv", action="store_true", help="emit CSV instead of text")
    cost.add_argument("--out", default=None, help="write JSON results here")
    return p


def _cost_rows(args):
    """cli.py:236-273; ``--table b200`` selects the measured B200 rows for
    the listing and the fitted prediction."""
    from . import costmodel
    from .exceptions import KascadeError
    rows = []
    if args.preset:
        for name in args.preset:
            rows.append((name, costmodel.report_from_preset(name), costmodel.get_preset(name)))
    elif args.ratios:
        parts = [float(x) for x in args.ratios.split(",")]
        if len(parts) != 3:
            raise KascadeError("--ratios needs anchor0,anchor,reuse")
        params = costmodel.CostParams(phase=args.phase, num_layers=args.layers, num_anchors=args.anchors,
                                      topk_fraction=args.fraction, seq_len=args.seq_len,
                                      baseline_layer_time=args.baseline_time)
        rows.append(("custom", costmodel.weighted_pipeline_time(
            params, {"anchor0": parts[0], "anchor": parts[1], "reuse": parts[2]}), None))
    elif args.predict:
        rep = costmodel.predict_report(args.phase, args.fraction, args.seq_len, num_layers=args.layers,
                                       num_anchors=args.anchors, baseline_layer_time=args.baseline_time,
                                       table=args.table)
        tag = "" if args.table == costmodel.TABLE_PUBLISHED else f"{args.table}-"
        rows.append((f"predict-{tag}{args.phase}-{args.seq_len}-k{args.fraction}", rep, None))
    else:
        for name in costmodel.preset_names(args.table):
            rows.append((name, costmodel.report_from_preset(name), costmodel.get_preset(name)))
    return rows


def _tabulated(row):
    """The row's own pipeline time / speedup columns: printed as published
    for Table 3 rows (cli.py:284-297), 6 significant digits for B200 rows."""
    from . import costmodel
    if row.table == costmodel.TABLE_PUBLISHED:
        return f"{row.kascade_ms}", f"{row.speedup_tl}"
    return f"{row.kascade_ms:.6g}", f"{row.speedup_tl:.6g}"


def cmd_cost(args) -> int:
    """cli.py:276-320 (same text, CSV and JSON forms)."""
    import json
    from . import costmodel
    if args.list_presets:
        for name in costmodel.preset_names(args.table):
            print(name)
        return EXIT_OK
    rows = _cost_rows(args)
    if args.csv:
        print("name,kascade_time,baseline_time,speedup,published_time,published_speedup")
        for name, rep, row in rows:
            pub_t, pub_s = _tabulated(row) if row else ("", "")
            print(f"{name},{rep.kascade_time:.6g},{rep.baseline_time:.6g},{rep.speedup:.6g},{pub_t},{pub_s}")
    else:
        for name, rep, row in rows:
            line = f"{name}: time={rep.kascade_time:.4g} baseline={rep.baseline_time:.4g} speedup={rep.speedup:.3f}"
            if row:
                pub_t, pub_s = _tabulated(row)
                label = "published" if row.table == costmodel.TABLE_PUBLISHED else "measured B200"
                line += f" ({label} time={pub_t} speedup={pub_s})"
            if not rep.valid:
                line += f" [!] {rep.note}"
            print(line)
    if args.out:
        payload = [{"name": name, "kascade_time": rep.kascade_time, "baseline_time": rep.baseline_time,
                    "speedup": rep.speedup, "per_kind": rep.per_kind, "valid": rep.valid,
                    "published_time": row.kascade_ms if row else None,
                    "published_speedup": row.speedup_tl if row else None} for name, rep, row in rows]
        with open(args.out, "w", encoding="utf-8") as f:
            json.dump(payload, f, indent=2)
            f.write("\n")
    return EXIT_OK


def cmd_gen(args) -> int:
    """cli.py:117-148."""
    import os
    import numpy as np
    from . import kscd_io
    from .synth import SynthConfig, generate_synthetic
    perms = None
    if args.permute_heads:
        rng = np.random.default_rng(args.seed ^ 0x9E3779B9)
        perms = [list(range(args.kv_heads))] + [list(rng.permutation(args.kv_heads)) for _ in range(args.layers - 1)]
    trace = generate_synthetic(SynthConfig(
        num_layers=args.layers, num_query_heads=args.q_heads, num_kv_heads=args.kv_heads, head_dim=args.dim,
        seq_len=args.tokens, seed=args.seed, layer_correlation=args.rho, head_permutations=perms,
        heavy_tail_temperature=args.temperature, query_correlation=args.query_correlation,
        layer0_temperature_scale=args.layer0_temperature_scale, include_xy=args.xy, prompt_id=args.prompt_id))
    kscd_io.write_trace(args.out, trace)
    size = os.path.getsize(args.out)
    print(f"wrote {args.out}: layers={trace.num_layers} q_heads={trace.num_query_heads} "
          f"kv_heads={trace.num_kv_heads} dim={trace.head_dim} tokens={trace.seq_len} "
          f"xy={int(trace.has_xy())} bytes={size}")
    return EXIT_OK


def cmd_analyze(args) -> int:
    """cli.py:151-192 with P, coverage and the similarity matrix on the GPU."""
    from pathlib import Path
    import numpy as np
    from . import calibration, compat, kscd_io
    traces = [kscd_io.TraceFile(p) for p in args.trace]
    out_dir = Path(args.out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    coverage = [np.mean([compat.mass_coverage(calibration.layer_probs(t, layer).cpu().numpy(), args.k)
                         for t in traces], axis=0) for layer in range(traces[0].num_layers)]
    (out_dir / "coverage.csv").write_text(kscd_io.coverage_csv(coverage))
    S = calibration.similarity_matrix(traces, k=args.k, token_agg=args.token_agg, mode=args.mode,
                                      tile_size=args.tile_size)
    (out_dir / "similarity.csv").write_text(kscd_io.similarity_csv(S))
    if args.importance:
        if all(t.X is not None and t.Y is not None for t in traces):
            imp = calibration.layer_importance(traces)
        else:
            print("warning: trace(s) lack attention input/output hidden states; using uniform importance weights",
                  file=sys.stderr)
            imp = calibration.LayerImportance(w=np.ones(traces[0].num_layers), source_prompt_count=len(traces))
        (out_dir / "importance.csv").write_text(kscd_io.importance_csv(imp))
    print(f"analyzed {len(traces)} trace(s): k={args.k} mode={args.mode} token_agg={args.token_agg} "
          f"undefined_scores={S.undefined_scores} -> {out_dir}")
    return EXIT_OK


def cmd_report(args) -> int:
    """cli.py:323-330."""
    import json
    from . import kscd_io
    with open(args.file, "r", encoding="utf-8") as f:
        data = json.load(f)
    if isinstance(data, dict) and data.get("kind") == "kascade-run-report":
        print(kscd_io.format_report(kscd_io.read_report(args.file)), end="")
    else:
        print(json.dumps(data, indent=2, sort_keys=True))
    return EXIT_OK


def cmd_plan(args) -> int:
    """cli.py:195-213 with the similarity matrix and head maps on the GPU."""
    from . import calibration, kscd_io
    from .host_types import KBudgetPolicy, write_plan
    traces = [kscd_io.TraceFile(p) for p in args.trace]
    plan = calibration.build_plan(traces, budget=args.budget, k=args.k, token_agg=args.token_agg,
                                  tile_size=args.tile_size, pooling=args.pooling,
                                  mode=args.mode.replace("-", "_"),
                                  k_policy=KBudgetPolicy(args.fraction, args.k_min),
                                  use_importance=not args.no_importance)
    write_plan(args.out, plan)
    print(f"anchors={plan.core.anchors} objective={plan.core.objective_value:.6g} "
          f"mode={plan.mode} pooling={plan.pooling} -> {args.out}")
    return EXIT_OK


def cmd_run(args) -> int:
    from . import compat, kscd_io
    from .host_types import read_plan
    trace = kscd_io.TraceFile(args.trace)      # header validated now; layers stream to the GPU
    plan = read_plan(args.plan)
    if args.mode is not None:
        plan.mode = args.mode.replace("-", "_")
    _, report = compat.run_kascade(trace, plan, phase=args.phase)
    if args.out:
        kscd_io.write_report(args.out, report)
    print(kscd_io.format_report(report), end="")
    if args.fail_above is not None:
        worst = report.overall["max_output_rel_err_l2"]
        if worst > args.fail_above:
            print(f"FAIL: max relative error {worst:.3e} exceeds {args.fail_above:.3e}", file=sys.stderr)
            return EXIT_THRESHOLD
    return EXIT_OK


def main(argv=None) -> int:
    """Every engine error (bad trace, bad plan, invalid argument, CUDA
    failure) and every OSError maps to exit 2, as in the reference main
    (cli.py:341-361); argparse errors return 1."""
    from .exceptions import KascadeError
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        return int(e.code or 0)
    if args.command == "gen" and args.q_heads % args.kv_heads != 0:     # usage error (cli.py:346-352)
        parser.print_usage(sys.stderr)
        sys.stderr.write(f"{parser.prog}: error: --q-heads ({args.q_heads}) must be divisible "
                         f"by --kv-heads ({args.kv_heads})\n")
        return EXIT_USAGE
    try:
        return {"gen": cmd_gen, "analyze": cmd_analyze, "cost": cmd_cost, "plan": cmd_plan, "run": cmd_run,
                "report": cmd_report}[args.command](args)
    except (KascadeError, OSError) as e:
        sys.stderr.write(f"{build_parser().prog}: {e}\n")
        return EXIT_DATA


if __name__ == "__main__":
    raise SystemExit(main())
