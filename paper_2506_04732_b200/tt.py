"""Tensor-train arithmetic of the hot path, computed by the CUDA engine.

The train containers are the reference's own ``ttss.tensor_train.TTVector``
/ ``TTOperator`` (tensor_train.py:63-133): every function here takes and
returns them, so reference code and this module exchange trains freely.
Structural constructors that only place given numbers into cores (separable
sums, identities, diagonal operators, block sums, operator composition,
scaling of the first core, the TTS2 container) are the reference's own
functions, re-exported unchanged — they are problem setup, not hot path.

Device-computed here: rounding (vector and operator), norm, dot product,
exact sum, operator application and dense reconstruction.  There is no CPU
implementation of any of them in this package; without the engine they
raise ``NativeUnavailable``.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import CapExceededError, ShapeError
from .reference import module as _ref

_rtt = _ref("tensor_train")

TTVector = _rtt.TTVector
TTOperator = _rtt.TTOperator
DENSE_CAP = _rtt.DENSE_CAP
# structural constructors (problem setup): the reference's own code
tt_scale = _rtt.tt_scale
tt_op_scale = _rtt.tt_op_scale
tt_rank_one = _rtt.tt_rank_one
tt_from_separable = _rtt.tt_from_separable
tt_diag_operator = _rtt.tt_diag_operator
tt_identity_operator = _rtt.tt_identity_operator
tt_op_add = _rtt.tt_op_add
tt_op_compose = _rtt.tt_op_compose
storage_size = _rtt.storage_size
compression_ratio = _rtt.compression_ratio
save_tt = _rtt.save_tt
load_tt = _rtt.load_tt

__all__ = [
    "TTVector", "TTOperator",
    "tt_round", "tt_op_round", "tt_add", "tt_dot", "tt_norm", "tt_apply", "tt_full",
    "tt_op_full", "tt_random", "to_device", "from_device",
    "tt_scale", "tt_op_scale", "tt_rank_one", "tt_from_separable", "tt_diag_operator",
    "tt_identity_operator", "tt_op_add", "tt_op_compose", "storage_size",
    "compression_ratio", "save_tt", "load_tt", "DENSE_CAP",
]


# -- host <-> device ------------------------------------------------------------


def _is_op(t):
    return t.cores[0].ndim == 4


def to_device(t):
    """Upload a train (any object with ``.cores``); returns a DeviceTrain."""
    return _native.DeviceTrain.upload(t.cores, _is_op(t))


def from_device(h):
    """Download a DeviceTrain into the reference's container."""
    cores, is_op = h.download()
    return TTOperator(cores) if is_op else TTVector(cores)


def _unary(t, fn):
    h = to_device(t)
    try:
        return fn(h)
    finally:
        h.free()


def _owned(out):
    o = _native.DeviceTrain(out)
    try:
        return from_device(o)
    finally:
        o.free()


# -- device-computed operations ---------------------------------------------------


def tt_round(v, tol, max_rank=None):
    """Recompress to relative accuracy ``tol`` (tensor_train.py:327)."""
    if tol < 0:
        raise ValueError("tolerance must be >= 0")
    L = _native.lib()

    def run(h):
        out = _native._P()
        _native.check(L.t2s2_round(_native.context(), h.handle, float(tol),
                                   int(max_rank or 0), out))
        return _owned(out)

    return _unary(v, run)


def tt_op_round(a, tol, max_rank=None):
    """Operator recompression through the merged-mode view (tensor_train.py:616)."""
    return tt_round(a, tol, max_rank)


def tt_norm(a):
    """Frobenius norm (tensor_train.py:319)."""
    L = _native.lib()

    def run(h):
        out = _native._D()
        _native.check(L.t2s2_norm(_native.context(), h.handle, out))
        return float(out.value)

    return _unary(a, run)


def tt_dot(a, b):
    """Inner product (tensor_train.py:296)."""
    if a.mode_sizes != b.mode_sizes:
        raise ShapeError(f"mode mismatch {a.mode_sizes} vs {b.mode_sizes}")
    L = _native.lib()
    ha, hb = to_device(a), to_device(b)
    try:
        out = _native._D()
        _native.check(L.t2s2_dot(_native.context(), ha.handle, hb.handle, out))
        return float(out.value)
    finally:
        ha.free()
        hb.free()


def _binary(a, b, call):
    ha, hb = to_device(a), to_device(b)
    try:
        out = _native._P()
        _native.check(call(ha.handle, hb.handle, out))
        return _owned(out)
    finally:
        ha.free()
        hb.free()


def tt_add(a, b):
    """Exact sum; internal ranks add (tensor_train.py:253)."""
    if not _is_op(a) and a.mode_sizes != b.mode_sizes:
        raise ShapeError(f"mode mismatch {a.mode_sizes} vs {b.mode_sizes}")
    L = _native.lib()
    return _binary(a, b, lambda x, y, o: L.t2s2_add(_native.context(), x, y, 1.0, 1.0, o))


def tt_apply(op, v):
    """Operator-vector product; bond ranks multiply (tensor_train.py:359)."""
    if op.col_sizes != v.mode_sizes:
        raise ShapeError(f"operator columns {op.col_sizes} vs vector {v.mode_sizes}")
    L = _native.lib()
    return _binary(op, v, lambda x, y, o: L.t2s2_apply(_native.context(), x, y, o))


def tt_full(v, cap=DENSE_CAP):
    """Dense reconstruction (tensor_train.py:186), computed on the device."""
    total = int(np.prod([float(n) for n in v.mode_sizes]))
    if total > cap:
        raise CapExceededError(f"dense materialization of {total} entries exceeds cap {cap}")
    L = _native.lib()

    def run(h):
        out = np.empty(total, dtype=np.float64)
        _native.check(L.t2s2_full(_native.context(), h.handle, out.ctypes.data_as(_native._DP),
                                  total))
        return out.reshape(v.mode_sizes)

    return _unary(v, run)


def tt_op_full(a, cap=DENSE_CAP):
    """Dense matrix (prod rows, prod cols) of an operator (tensor_train.py:622)."""
    rows, cols = a.row_sizes, a.col_sizes
    total = int(np.prod([float(m) for m in rows])) * int(np.prod([float(n) for n in cols]))
    if total > cap:
        raise CapExceededError(f"dense materialization of {total} entries exceeds cap {cap}")
    merged = TTVector([c.reshape(c.shape[0], c.shape[1] * c.shape[2], c.shape[3])
                       for c in a.cores])
    dense = tt_full(merged, cap=cap).reshape([x for m, n in zip(rows, cols) for x in (m, n)])
    d = len(rows)
    dense = dense.transpose(list(range(0, 2 * d, 2)) + list(range(1, 2 * d, 2)))
    return dense.reshape(int(np.prod(rows)), int(np.prod(cols)))


def tt_random(modes, rank, rng, norm=1.0):
    """Random train with uniform internal rank scaled to ``norm``; the same
    draws as tensor_train.tt_random, normalised with the device norm."""
    d = len(modes)
    rk = [1] + [rank] * (d - 1) + [1]
    v = TTVector([rng.standard_normal((rk[l], modes[l], rk[l + 1])) for l in range(d)])
    nrm = tt_norm(v)
    return tt_scale(v, norm / nrm) if nrm > 0 else v
