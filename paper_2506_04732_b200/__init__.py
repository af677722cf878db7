"""B200-native T^2S^2 hot path.

A drop-in for the tensor-train linear algebra of the reference's
``pkg/src/ttss`` (tensor_train / tt_solver / time_integration): the host API
keeps the reference's names and arguments, and every numerical kernel of the
implicit step runs in the CUDA engine ``lib/libt2s2.so`` (sm_100a, fp64).
Problem setup (1-D Legendre collocation blocks, separable coefficients,
operator chains) is host-side, as in the reference.

Importing this package does not touch the GPU; the first numerical call
loads the engine and raises ``NativeUnavailable`` if it cannot.
"""

from . import assembly, coefficients, collocation, spectral, tt  # noqa: F401
from ._native import NativeUnavailable  # noqa: F401
from .errors import CapExceededError, MarchStepError, ShapeError  # noqa: F401

__all__ = ["assembly", "coefficients", "collocation", "spectral", "tt", "solver", "march",
           "NativeUnavailable", "ShapeError", "MarchStepError", "CapExceededError"]


def __getattr__(name):  # lazy: solver/march pull in ctypes prototypes only when used
    if name in ("solver", "march"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
