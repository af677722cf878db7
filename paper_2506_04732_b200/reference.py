"""Locate the reference host package ``ttss`` (pkg/src/ttss).

The drop-in keeps the reference's host API as it is: problem setup (grids,
collocation blocks, coefficient sampling, operator chains), the train
containers, the config/report dataclasses and the exception classes all come
from ``ttss`` itself.  This package replaces only the hot path (the solve,
the step loop and the train arithmetic on it) with the CUDA engine.

Search order: an importable ``ttss``; ``$T2S2_TTSS_PATH``; the offline
install of the reference at ``<repo>/baseline/_ref`` (``python -m pip
install --no-index --no-build-isolation --no-deps --target baseline/_ref
<copy of /root/reference/pkg>``, which ``__graft_entry__.build()`` performs).
"""

from __future__ import annotations

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASELINE_REF = os.path.join(ROOT, "baseline", "_ref")

_mod = None


def ttss():
    """The imported ``ttss`` package (raises ImportError with a recipe)."""
    global _mod
    if _mod is not None:
        return _mod
    try:
        _mod = importlib.import_module("ttss")
        return _mod
    except ImportError:
        pass
    for path in (os.environ.get("T2S2_TTSS_PATH"), BASELINE_REF):
        if path and os.path.isdir(os.path.join(path, "ttss")):
            if path not in sys.path:
                sys.path.append(path)
            _mod = importlib.import_module("ttss")
            return _mod
    raise ImportError(
        "the reference host package `ttss` is not importable: install it (pip install "
        "<reference>/pkg) or run __graft_entry__.build(), which installs it into "
        f"{BASELINE_REF}")


def module(name):
    """``ttss.<name>`` (tensor_train, tt_solver, time_integration, ...)."""
    ttss()
    return importlib.import_module(f"ttss.{name}")
