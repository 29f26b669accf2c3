"""The reference package's module layout (``kascade`` 0.1.0) over this engine.

Every module of the reference that a caller imports from exists here with
the same public names, each bound to the B200 implementation (device
kernels through the C ABI; host-side types, plan/trace/report formats and
the cost model restated).  Two ways to switch:

    from paper_2512_16391_b200 import kascade          # explicit
    from paper_2512_16391_b200.kascade import install
    install()                                          # `import kascade` now resolves here

``install()`` registers this package and its submodules under the name
``kascade`` in ``sys.modules``, so code written against the reference --
``from kascade.runner import POOL_POST`` included -- runs unchanged.
"""

import importlib
import sys

__version__ = "0.1.0"

SUBMODULES = ("attention", "cli", "costmodel", "errors", "heads", "metrics", "parallel", "pipeline", "planner",
              "ranking", "runner", "tiles", "trace", "traceio")
# modules whose public names the reference re-exports at the top level
_ROOT_EXPORTS = ("attention", "costmodel", "errors", "heads", "metrics", "pipeline", "planner", "runner", "tiles",
                 "trace", "traceio")

for _name in SUBMODULES:
    _mod = importlib.import_module(f".{_name}", __name__)
    globals()[_name] = _mod
    if _name in _ROOT_EXPORTS:
        for _sym in _mod.__all__:
            globals()[_sym] = getattr(_mod, _sym)
del _name, _mod, _sym


def install(alias: str = "kascade") -> None:
    """Make ``import kascade`` (and every ``kascade.<module>``) resolve to
    this package in the current interpreter."""
    me = sys.modules[__name__]
    sys.modules[alias] = me
    for sub in SUBMODULES:
        sys.modules[f"{alias}.{sub}"] = importlib.import_module(f".{sub}", __name__)
