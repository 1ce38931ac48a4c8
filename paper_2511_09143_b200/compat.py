"""`migsim` import alias: lets code written against the reference package
(`import migsim.commsim`, `from migsim.scheduler import fm_select`, ...) run
on this package unchanged.  Used to run the reference's own hot-path tests
against this implementation (tests/test_reference_suite.py)."""

from __future__ import annotations

import importlib
import sys

_MODULES = ("commsim", "errors", "mig", "scheduler", "simcore", "workload", "cli")


def install_migsim_alias() -> None:
    pkg = importlib.import_module("paper_2511_09143_b200")
    sys.modules["migsim"] = pkg
    for name in _MODULES:
        mod = importlib.import_module(f"paper_2511_09143_b200.{name}")
        sys.modules[f"migsim.{name}"] = mod
        setattr(pkg, name, mod)
