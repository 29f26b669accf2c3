"""python -m paper_2512_16391_b200.kascade: the reference CLI (kascade gen|analyze|plan|run|cost|report)."""
import sys

from ..cli import main

sys.exit(main())
