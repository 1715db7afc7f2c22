"""pytest plugin: import this package under the reference's name `dropsim`.

    PYTHONDONTWRITEBYTECODE=1 python -m pytest -p tests.dropsim_alias -p no:cacheprovider \
        /root/reference/pkg/tests/test_memory.py ...

so the reference's own unit / acceptance tests run unchanged against this
package (model mode: the engine's host path).  Test infrastructure only.
"""

import importlib
import sys

_MODULES = ("core", "memory", "planner", "exchange", "engine", "costmodel", "formulation",
            "config", "metrics", "traceio")


def _install() -> None:
    pkg = importlib.import_module("paper_2412_18169_b200")
    sys.modules["dropsim"] = pkg
    for m in _MODULES:
        mod = importlib.import_module(f"paper_2412_18169_b200.{m}")
        sys.modules[f"dropsim.{m}"] = mod
        setattr(pkg, m, mod)


_install()
