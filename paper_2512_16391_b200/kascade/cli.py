"""kascade.cli (cli.py): the command line (gen, analyze, plan, run, cost, report)."""
from ..cli import (EXIT_DATA, EXIT_OK, EXIT_THRESHOLD, EXIT_USAGE, build_parser, cmd_analyze, cmd_cost, cmd_gen,
                   cmd_plan, cmd_report, cmd_run, main)

__all__ = ["main", "build_parser", "EXIT_OK", "EXIT_USAGE", "EXIT_DATA", "EXIT_THRESHOLD", "cmd_gen", "cmd_analyze",
           "cmd_plan", "cmd_run", "cmd_cost", "cmd_report"]
