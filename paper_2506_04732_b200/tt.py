"""Tensor trains: host containers plus device-computed arithmetic.

``TTVector`` / ``TTOperator`` carry numpy cores exactly like the reference's
classes (pkg/src/ttss/tensor_train.py:63-133), so problem setup code reads
the same.  Structural constructors that only place given numbers into cores
(separable sums, identities, diagonal operators, block sums, Kronecker
composition of operator cores) run on the host as part of problem setup.
Every numerical algorithm of the hot path — orthogonalisation, rounding,
norms, dot products, operator application, dense reconstruction, the solver
and the time march — runs in the CUDA engine through ``_native``; there is no
CPU implementation of them in this package.
"""

from __future__ import annotations

import io
import struct

import numpy as np

from . import _native
from .errors import CapExceededError, ShapeError

__all__ = [
    "TTVector", "TTOperator",
    "tt_round", "tt_add", "tt_scale", "tt_dot", "tt_norm", "tt_apply",
    "tt_from_separable", "tt_full", "tt_rank_one", "tt_random",
    "compression_ratio", "storage_size",
    "tt_diag_operator", "tt_identity_operator", "tt_op_add", "tt_op_scale",
    "tt_op_compose", "tt_op_round", "tt_op_full",
    "save_tt", "load_tt", "DENSE_CAP", "to_device", "from_device",
]

DENSE_CAP = 10**8


class _Train:
    _order = 3

    def __init__(self, cores):
        cores = [np.asarray(c, dtype=float) for c in cores]
        if not cores:
            raise ShapeError("need at least one core")
        for c in cores:
            if c.ndim != self._order:
                raise ShapeError(f"cores must have {self._order} axes")
        if cores[0].shape[0] != 1 or cores[-1].shape[-1] != 1:
            raise ShapeError("boundary ranks must be 1")
        for a, b in zip(cores[:-1], cores[1:]):
            if a.shape[-1] != b.shape[0]:
                raise ShapeError("adjacent core ranks do not match")
        self.cores = cores

    @property
    def ndim(self):
        return len(self.cores)

    @property
    def ranks(self):
        return tuple([1] + [c.shape[-1] for c in self.cores])


class TTVector(_Train):
    """d-dimensional tensor as order-3 cores (r_prev, n, r_next)."""

    _order = 3

    @property
    def mode_sizes(self):
        return tuple(c.shape[1] for c in self.cores)

    def __repr__(self):
        return f"TTVector(modes={self.mode_sizes}, ranks={self.ranks})"


class TTOperator(_Train):
    """Linear operator as order-4 cores (r_prev, m_row, n_col, r_next)."""

    _order = 4

    @property
    def row_sizes(self):
        return tuple(c.shape[1] for c in self.cores)

    @property
    def col_sizes(self):
        return tuple(c.shape[2] for c in self.cores)

    def __repr__(self):
        return f"TTOperator(rows={self.row_sizes}, cols={self.col_sizes}, ranks={self.ranks})"


# -- host <-> device ------------------------------------------------------------


def to_device(t):
    """Upload a train; returns a ``_native.DeviceTrain`` handle."""
    return _native.DeviceTrain.upload(t.cores, isinstance(t, TTOperator))


def from_device(h):
    cores, is_op = h.download()
    return TTOperator(cores) if is_op else TTVector(cores)


def _unary(t, fn):
    h = to_device(t)
    try:
        return fn(h)
    finally:
        h.free()


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
        o = _native.DeviceTrain(out)
        try:
            return from_device(o)
        finally:
            o.free()

    return _unary(v, run)


def tt_op_round(a, tol, max_rank=None):
    """Operator recompression through the merged-mode view (tensor_train.py:616)."""
    return tt_round(a, tol, max_rank)


def tt_norm(a):
    L = _native.lib()

    def run(h):
        out = _native._D()
        _native.check(L.t2s2_norm(_native.context(), h.handle, out))
        return float(out.value)

    return _unary(a, run)


def tt_dot(a, b):
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
        o = _native.DeviceTrain(out)
        try:
            return from_device(o)
        finally:
            o.free()
    finally:
        ha.free()
        hb.free()


def tt_add(a, b):
    """Exact sum; internal ranks add (tensor_train.py:253)."""
    if isinstance(a, TTVector) and a.mode_sizes != b.mode_sizes:
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


# -- structural constructors (problem setup) ------------------------------------------


def tt_scale(a, s):
    """Scale the first core (tensor_train.py:277)."""
    cores = [c.copy() for c in a.cores]
    cores[0] = cores[0] * float(s)
    return type(a)(cores)


def tt_op_scale(a, s):
    return tt_scale(a, s)


def tt_rank_one(factors, scale=1.0):
    cores = [np.asarray(f, dtype=float).reshape(1, -1, 1) for f in factors]
    cores[0] = cores[0] * scale
    return TTVector(cores)


def tt_random(modes, rank, rng, norm=1.0):
    """Random train with uniform internal rank, scaled to ``norm``."""
    d = len(modes)
    rk = [1] + [rank] * (d - 1) + [1]
    v = TTVector([rng.standard_normal((rk[l], modes[l], rk[l + 1])) for l in range(d)])
    nrm = tt_norm(v)
    return tt_scale(v, norm / nrm) if nrm > 0 else v


def tt_from_separable(terms, modes=None):
    """Exact train of sum_k s_k f_k1 x ... x f_kd; internal ranks = #terms
    (tensor_train.py:215-250)."""
    if not terms:
        raise ShapeError("need at least one term")
    d = len(terms[0][1])
    if any(len(f) != d for _, f in terms):
        raise ShapeError("all terms must supply one factor per mode")
    vecs = [[np.asarray(f, dtype=float) for f in fs] for _, fs in terms]
    if modes is None:
        modes = tuple(len(f) for f in vecs[0])
    if any(tuple(len(f) for f in fs) != tuple(modes) for fs in vecs):
        raise ShapeError("factor lengths disagree across terms")
    scales = np.array([float(s) for s, _ in terms])
    t = len(terms)
    if d == 1:
        col = sum(s * fs[0] for s, fs in zip(scales, vecs))
        return TTVector([col.reshape(1, -1, 1)])
    first = np.stack([s * fs[0] for s, fs in zip(scales, vecs)], axis=-1)[None]
    cores = [first]
    for l in range(1, d - 1):
        mid = np.zeros((t, modes[l], t))
        for k in range(t):
            mid[k, :, k] = vecs[k][l]
        cores.append(mid)
    cores.append(np.stack([fs[-1] for fs in vecs], axis=0)[:, :, None])
    return TTVector(cores)


def tt_diag_operator(v):
    """Diagonal operator with the entries of v (tensor_train.py:543)."""
    cores = []
    for c in v.cores:
        r0, n, r1 = c.shape
        core = np.zeros((r0, n, n, r1))
        idx = np.arange(n)
        core[:, idx, idx, :] = c
        cores.append(core)
    return TTOperator(cores)


def tt_identity_operator(modes):
    return TTOperator([np.eye(n).reshape(1, n, n, 1) for n in modes])


def tt_op_add(a, b):
    """Block sum of two operators; ranks add (tensor_train.py:560)."""
    if a.row_sizes != b.row_sizes or a.col_sizes != b.col_sizes:
        raise ShapeError("operator shapes do not match")
    d = a.ndim
    if d == 1:
        return TTOperator([a.cores[0] + b.cores[0]])
    cores = []
    for l, (ca, cb) in enumerate(zip(a.cores, b.cores)):
        if l == 0:
            cores.append(np.concatenate([ca, cb], axis=3))
        elif l == d - 1:
            cores.append(np.concatenate([ca, cb], axis=0))
        else:
            blk = np.zeros((ca.shape[0] + cb.shape[0],) + ca.shape[1:3]
                           + (ca.shape[3] + cb.shape[3],))
            blk[: ca.shape[0], :, :, : ca.shape[3]] = ca
            blk[ca.shape[0]:, :, :, ca.shape[3]:] = cb
            cores.append(blk)
    return TTOperator(cores)


def tt_op_compose(a, b):
    """a @ b with b acting first; bond ranks multiply (tensor_train.py:589)."""
    if a.col_sizes != b.row_sizes:
        raise ShapeError("inner operator sizes do not match")
    cores = []
    for ca, cb in zip(a.cores, b.cores):
        core = np.einsum("amkb,cknd->acmnbd", ca, cb)
        cores.append(core.reshape(ca.shape[0] * cb.shape[0], ca.shape[1], cb.shape[2],
                                  ca.shape[3] * cb.shape[3]))
    return TTOperator(cores)


def storage_size(v):
    return int(sum(c.size for c in v.cores))


def compression_ratio(v):
    dense = float(np.prod([float(n) for n in v.mode_sizes]))
    return storage_size(v) / dense


# -- "TTS2" container (tensor_train.py:648-712) -----------------------------------------

_MAGIC, _VERSION, _VEC, _OP = b"TTS2", 1, 1, 2


def save_tt(obj, path):
    is_op = isinstance(obj, TTOperator)
    out = io.BytesIO()
    out.write(_MAGIC + struct.pack("<BBI", _VERSION, _OP if is_op else _VEC, obj.ndim))
    if is_op:
        out.write(b"".join(struct.pack("<II", m, n) for m, n in zip(obj.row_sizes, obj.col_sizes)))
    else:
        out.write(b"".join(struct.pack("<I", n) for n in obj.mode_sizes))
    out.write(b"".join(struct.pack("<I", r) for r in obj.ranks))
    for c in obj.cores:
        out.write(np.ascontiguousarray(c, dtype="<f8").tobytes())
    data = out.getvalue()
    if hasattr(path, "write"):
        path.write(data)
    else:
        with open(path, "wb") as fh:
            fh.write(data)


def load_tt(path):
    if hasattr(path, "read"):
        data = path.read()
    else:
        with open(path, "rb") as fh:
            data = fh.read()
    if data[:4] != _MAGIC:
        raise ValueError("not a TTS2 container")
    version, kind = struct.unpack_from("<BB", data, 4)
    if version != _VERSION:
        raise ValueError(f"unsupported container version {version}")
    (d,) = struct.unpack_from("<I", data, 6)
    off = 10
    if kind == _OP:
        sizes = struct.unpack_from(f"<{2 * d}I", data, off)
        off += 8 * d
        rows, cols = sizes[0::2], sizes[1::2]
    else:
        rows, cols = struct.unpack_from(f"<{d}I", data, off), None
        off += 4 * d
    ranks = struct.unpack_from(f"<{d + 1}I", data, off)
    off += 4 * (d + 1)
    cores = []
    for l in range(d):
        shape = ((ranks[l], rows[l], cols[l], ranks[l + 1]) if kind == _OP
                 else (ranks[l], rows[l], ranks[l + 1]))
        count = int(np.prod(shape))
        cores.append(np.frombuffer(data, dtype="<f8", count=count, offset=off)
                     .reshape(shape).astype(float))
        off += 8 * count
    return TTOperator(cores) if kind == _OP else TTVector(cores)
