"""``python -m paper_2512_16391_b200 run``: the reference CLI's ``run``
subcommand (cli.py:80-89,216-233) on the B200 engine.

    python -m paper_2512_16391_b200 run --trace t.kscd --plan p.json \\
        [--phase prefill|decode] [--mode remapped|all-heads-pooled] [--out report.json] [--fail-above X]

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
    run = sub.add_parser("run", help="execute the anchor/reuse pipeline on the GPU and report fidelity vs dense")
    run.add_argument("--trace", required=True)
    run.add_argument("--plan", required=True)
    run.add_argument("--phase", choices=["prefill", "decode"], default="prefill")
    run.add_argument("--mode", choices=["remapped", "all-heads-pooled"], default=None)
    run.add_argument("--out", default=None)
    run.add_argument("--fail-above", type=float, default=None)
    run.add_argument("--engine", choices=["b200"], default="b200",
                     help="accepted for parity with `kascade run --engine b200`; there is no other engine")
    return p


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
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as e:
        return int(e.code or 0)
    try:
        return cmd_run(args)
    except (KascadeError, OSError) as e:
        sys.stderr.write(f"{build_parser().prog}: {e}\n")
        return EXIT_DATA


if __name__ == "__main__":
    raise SystemExit(main())
