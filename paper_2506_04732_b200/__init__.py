"""B200-native T^2S^2 hot path.

A drop-in for the tensor-train hot path of the reference's ``ttss`` package
(pkg/src/ttss): the alternating solve (tt_solver.solve / residual), the
implicit step loop (time_integration._march) and the train arithmetic on
it (tensor_train.tt_round / tt_norm / tt_dot / tt_add / tt_apply / tt_full)
run in the CUDA engine ``lib/libt2s2.so`` (sm_100a, fp64) behind the C ABI
of ``include/t2s2.h``.  Everything else — problem setup, containers,
configs, reports, exceptions — is the reference's own code, imported from
``ttss`` (see ``reference.py``); ``dropin.install()`` swaps the hot-path
functions inside an unmodified ``ttss``.

Importing this package does not touch the GPU; the first numerical call
loads the engine and raises ``NativeUnavailable`` if it cannot.
"""

from ._native import NativeUnavailable  # noqa: F401
from .errors import CapExceededError, MarchStepError, ShapeError  # noqa: F401

__all__ = ["tt", "solver", "march", "dropin", "sweep", "workloads", "NativeUnavailable",
           "ShapeError", "MarchStepError", "CapExceededError"]


def __getattr__(name):  # lazy: submodules pull in ttss and ctypes prototypes when used
    if name in ("tt", "solver", "march", "dropin", "sweep", "workloads"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
