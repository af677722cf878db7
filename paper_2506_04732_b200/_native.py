"""ctypes binding of ``libt2s2.so`` (include/t2s2.h).

This is the binding a reference maintainer would add to ``pkg/src/ttss``
(see INTEGRATION.md).  There is no fallback: if the library or a CUDA
device is missing, every entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import MarchStepError, ShapeError

__all__ = [
    "NativeUnavailable",
    "lib",
    "context",
    "DeviceTrain",
    "SolverConfigC",
    "SolveReportC",
    "StepReportC",
    "check",
    "LIB_PATH",
]

LIB_PATH = os.environ.get("T2S2_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                     "lib", "libt2s2.so")
MAX_SWEEPS = 1024

T2S2_OK = 0
T2S2_ERR_ARG = 1
T2S2_ERR_CUDA = 2
T2S2_ERR_SHAPE = 3
T2S2_ERR_VALUE = 4
T2S2_ERR_STAGNATION = 5
T2S2_ERR_CAPACITY = 6


class NativeUnavailable(RuntimeError):
    """The CUDA engine (libt2s2.so) could not be loaded or initialised."""


class SolverConfigC(ctypes.Structure):
    _fields_ = [
        ("max_sweeps", ctypes.c_int),
        ("residual_tol", ctypes.c_double),
        ("rounding_tol", ctypes.c_double),
        ("enrichment_rank", ctypes.c_int),
        ("max_rank", ctypes.c_int),
        ("local_solver", ctypes.c_int),
        ("local_direct_size", ctypes.c_int),
        ("inner_tol_factor", ctypes.c_double),
        ("stagnation_window", ctypes.c_int),
        ("stagnation_drop", ctypes.c_double),
    ]


class SolveReportC(ctypes.Structure):
    _fields_ = [
        ("n_sweeps", ctypes.c_int),
        ("residuals", ctypes.c_double * MAX_SWEEPS),
        ("ranks", ctypes.c_int * MAX_SWEEPS),
        ("compression", ctypes.c_double * MAX_SWEEPS),
        ("wall_time", ctypes.c_double),
        ("converged", ctypes.c_int),
        ("stagnated", ctypes.c_int),
    ]


class StepReportC(ctypes.Structure):
    _fields_ = [
        ("step", ctypes.c_int),
        ("max_rank", ctypes.c_int),
        ("compression", ctypes.c_double),
        ("residual", ctypes.c_double),
        ("sweeps", ctypes.c_int),
    ]


class KernelStatC(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_char * 32),
        ("launches", ctypes.c_longlong),
        ("device_ms", ctypes.c_double),
        ("flops", ctypes.c_double),
        ("bytes", ctypes.c_double),
    ]


class LaunchRecordC(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_int),
        ("flops", ctypes.c_double),
        ("bytes", ctypes.c_double),
        ("device_ms", ctypes.c_double),
    ]


_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_IP = ctypes.POINTER(ctypes.c_int)
_DP = ctypes.POINTER(ctypes.c_double)

_SIGNATURES = {
    "t2s2_context_create": (_I, [_I, ctypes.POINTER(_P)]),
    "t2s2_sm_partitions": (_I, [_I, _I, _IP]),
    "t2s2_context_create_on_partition": (_I, [_I, _I, ctypes.POINTER(_P)]),
    "t2s2_device_clock": (_I, [_P, ctypes.POINTER(ctypes.c_ulonglong)]),
    "t2s2_context_destroy": (None, [_P]),
    "t2s2_last_error": (ctypes.c_char_p, [_P]),
    "t2s2_synchronize": (_I, [_P]),
    "t2s2_stream": (_P, [_P]),
    "t2s2_context_set_sm_budget": (_I, [_P, _I]),
    "t2s2_stats_reset": (_I, [_P, _I]),
    "t2s2_stats_read": (_I, [_P, ctypes.POINTER(KernelStatC), _I, _IP]),
    "t2s2_launch_log": (_I, [_P, ctypes.POINTER(LaunchRecordC), _I, _IP]),
    "t2s2_read_trace": (_I, [_P, _I, _IP]),
    "t2s2_train_upload": (_I, [_P, _I, _IP, _IP, _IP, _DP, ctypes.POINTER(_P)]),
    "t2s2_train_upload_device": (_I, [_P, _I, _IP, _IP, _IP, _P, ctypes.POINTER(_P)]),
    "t2s2_train_shape": (_I, [_P, _IP, _IP, _IP, _IP, ctypes.POINTER(ctypes.c_size_t)]),
    "t2s2_train_download": (_I, [_P, _P, _DP, ctypes.c_size_t]),
    "t2s2_train_free": (None, [_P]),
    "t2s2_round": (_I, [_P, _P, _D, _I, ctypes.POINTER(_P)]),
    "t2s2_norm": (_I, [_P, _P, _DP]),
    "t2s2_dot": (_I, [_P, _P, _P, _DP]),
    "t2s2_add": (_I, [_P, _P, _P, _D, _D, ctypes.POINTER(_P)]),
    "t2s2_scale": (_I, [_P, _P, _D, ctypes.POINTER(_P)]),
    "t2s2_apply": (_I, [_P, _P, _P, ctypes.POINTER(_P)]),
    "t2s2_full": (_I, [_P, _P, _DP, ctypes.c_size_t]),
    "t2s2_solve": (_I, [_P, _P, _P, _P, ctypes.POINTER(SolverConfigC), ctypes.POINTER(_P),
                        ctypes.POINTER(SolveReportC)]),
    "t2s2_dense_solve": (_I, [_P, _I, _DP, _DP, _DP]),
    "t2s2_gemm": (_I, [_P, _I, _I, _I, _I, _I, _P, _I, _P, _I, _P, _I]),
    "t2s2_residual": (_I, [_P, _P, _P, _P, _D, _DP]),
    "t2s2_march": (_I, [_P, _P, _P, _P, _I, ctypes.POINTER(_P), ctypes.POINTER(_P), _I, _D,
                        ctypes.POINTER(SolverConfigC), _I, ctypes.POINTER(_P),
                        ctypes.POINTER(StepReportC), _IP]),
}

EXPORTED = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None
_tls = threading.local()  # one engine context (and stream) per host thread


def load_library(path=LIB_PATH):
    """Load libt2s2.so and declare its prototypes (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `make` or __graft_entry__.build()"
            )
        try:
            lib = ctypes.CDLL(path)
        except OSError as exc:
            raise NativeUnavailable(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib():
    return load_library()


def context():
    """This thread's engine context on device ``T2S2_DEVICE`` (default
    ``LOCAL_RANK`` or 0).  Each host thread gets its own context and stream;
    a train belongs to the thread that created it.  (Solves of different
    contexts on one GPU are not safe to overlap with unbounded kernels: see
    sweep.py; set_thread_sm_budget caps a context's cooperative grids.)"""
    ctx = getattr(_tls, "ctx", None)
    if ctx is not None:
        return ctx
    l = lib()
    dev = device_index()
    h = _P()
    part = getattr(_tls, "partition", None)
    if part is None:
        rc = l.t2s2_context_create(dev, ctypes.byref(h))
    else:
        rc = l.t2s2_context_create_on_partition(dev, int(part), ctypes.byref(h))
    if rc != T2S2_OK:
        raise NativeUnavailable(f"t2s2_context_create(device={dev}, partition={part}) failed "
                                f"with code {rc} (no CUDA device?)")
    budget = getattr(_tls, "sm_budget", 0)
    if budget:
        l.t2s2_context_set_sm_budget(h, int(budget))
    _tls.ctx = h
    return h


def device_index():
    return int(os.environ.get("T2S2_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def sm_partitions(count):
    """Split this process's device into `count` disjoint SM partitions
    (green contexts; once per process).  Returns their SM counts."""
    out = (ctypes.c_int * count)()
    rc = lib().t2s2_sm_partitions(device_index(), int(count), out)
    if rc != T2S2_OK:
        raise NativeUnavailable(f"t2s2_sm_partitions({count}) failed with code {rc}")
    return list(out)


def use_partition(part):
    """Bind this host thread's (future) engine context to SM partition
    `part` of sm_partitions(); call before the thread's first engine call."""
    if getattr(_tls, "ctx", None) is not None:
        raise RuntimeError("this thread already has an engine context")
    _tls.partition = int(part)


def device_clock_ns():
    """The device's global nanosecond timer, read on this thread's stream
    after its queued work (blocking)."""
    v = ctypes.c_ulonglong()
    check(lib().t2s2_device_clock(context(), ctypes.byref(v)))
    return int(v.value)


def num_sms():
    """Multiprocessor count of this thread's device (via torch if present)."""
    try:
        import torch

        dev = int(os.environ.get("T2S2_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        return torch.cuda.get_device_properties(dev).multi_processor_count
    except Exception:
        return 148


def set_thread_sm_budget(sms):
    """Cap the cooperative local-solve kernels of this thread's context."""
    _tls.sm_budget = int(sms)
    ctx = getattr(_tls, "ctx", None)
    if ctx is not None:
        lib().t2s2_context_set_sm_budget(ctx, int(sms))


def check(rc, step=None):
    if rc == T2S2_OK:
        return
    msg = lib().t2s2_last_error(context()).decode(errors="replace")
    if rc == T2S2_ERR_SHAPE:
        raise ShapeError(msg)
    if rc == T2S2_ERR_VALUE:
        raise ValueError(msg)
    if rc == T2S2_ERR_STAGNATION:
        raise MarchStepError(step if step is not None else -1, msg)
    raise RuntimeError(f"t2s2 error {rc}: {msg}")


def stats_reset(profile_events=False):
    check(lib().t2s2_stats_reset(context(), 1 if profile_events else 0))


def read_trace(mode):
    """0 off, 1 record, 2 replay the recorded host reads (see t2s2.h); returns
    the number of reads recorded."""
    n = ctypes.c_int()
    check(lib().t2s2_read_trace(context(), int(mode), ctypes.byref(n)))
    return n.value


def stats_read():
    """{family: dict(launches, device_ms, flops, bytes)} since the last reset."""
    n = ctypes.c_int()
    check(lib().t2s2_stats_read(context(), None, 0, ctypes.byref(n)))
    buf = (KernelStatC * max(n.value, 1))()
    check(lib().t2s2_stats_read(context(), buf, n.value, ctypes.byref(n)))
    return {buf[i].family.decode(): dict(launches=int(buf[i].launches),
                                         device_ms=float(buf[i].device_ms),
                                         flops=float(buf[i].flops), bytes=float(buf[i].bytes))
            for i in range(n.value)}


def launch_log():
    """Per-launch records [(family, flops, bytes, device_ms)] since the last
    stats_reset(profile_events=True), in launch order."""
    names = list(stats_read())
    n = ctypes.c_int()
    check(lib().t2s2_launch_log(context(), None, 0, ctypes.byref(n)))
    buf = (LaunchRecordC * max(n.value, 1))()
    check(lib().t2s2_launch_log(context(), buf, n.value, ctypes.byref(n)))
    return [(names[buf[i].family], buf[i].flops, buf[i].bytes, buf[i].device_ms)
            for i in range(n.value)]


def dense_solve(a, b):
    """x = a^{-1} b through the engine's fused LU kernel (testing hook)."""
    a = np.asfortranarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty_like(b)
    n = b.size
    check(lib().t2s2_dense_solve(context(), n, a.ravel(order="F").ctypes.data_as(_DP),
                                 b.ctypes.data_as(_DP), x.ctypes.data_as(_DP)))
    return x


def gemm_device(ta, tb, m, n, k, a_ptr, lda, b_ptr, ldb, c_ptr, ldc):
    """C = op(A) op(B) on device pointers (row-major fp64) through the
    engine's GEMM program kernel (testing / benchmarking hook)."""
    check(lib().t2s2_gemm(context(), int(ta), int(tb), m, n, k, ctypes.c_void_p(a_ptr), lda,
                          ctypes.c_void_p(b_ptr), ldb, ctypes.c_void_p(c_ptr), ldc))


def synchronize():
    check(lib().t2s2_synchronize(context()))


def _iarr(vals):
    a = (ctypes.c_int * len(vals))(*[int(v) for v in vals])
    return a


class DeviceTrain:
    """Owning handle of a device-resident train (vector or operator)."""

    __slots__ = ("handle",)

    def __init__(self, handle):
        self.handle = handle

    @classmethod
    def upload(cls, cores, is_op):
        cores = [np.ascontiguousarray(c, dtype=np.float64) for c in cores]
        d = len(cores)
        rows = _iarr([c.shape[1] for c in cores])
        cols = _iarr([c.shape[2] for c in cores]) if is_op else None
        ranks = _iarr([1] + [c.shape[-1] for c in cores])
        flat = np.concatenate([c.ravel() for c in cores]) if d else np.zeros(0)
        flat = np.ascontiguousarray(flat)
        h = _P()
        check(lib().t2s2_train_upload(context(), d, rows, cols, ranks,
                                      flat.ctypes.data_as(_DP), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def upload_flat(cls, host_ptr, rows, cols, ranks):
        """Upload from a caller-owned flat float64 buffer (e.g. pinned memory)."""
        h = _P()
        check(lib().t2s2_train_upload(context(), len(rows), _iarr(rows),
                                      _iarr(cols) if cols is not None else None,
                                      _iarr(ranks), ctypes.cast(host_ptr, _DP), ctypes.byref(h)))
        return cls(h)

    def download_into(self, host_ptr, capacity):
        check(lib().t2s2_train_download(context(), self.handle, ctypes.cast(host_ptr, _DP),
                                        int(capacity)))

    @classmethod
    def upload_device(cls, ptr, d, rows, cols, ranks):
        h = _P()
        check(lib().t2s2_train_upload_device(context(), d, _iarr(rows),
                                             _iarr(cols) if cols is not None else None,
                                             _iarr(ranks), _P(ptr), ctypes.byref(h)))
        return cls(h)

    def shape(self):
        d = ctypes.c_int()
        check(lib().t2s2_train_shape(self.handle, ctypes.byref(d), None, None, None, None))
        n = d.value
        rows, cols, ranks = (ctypes.c_int * n)(), (ctypes.c_int * n)(), (ctypes.c_int * (n + 1))()
        total = ctypes.c_size_t()
        check(lib().t2s2_train_shape(self.handle, None, rows, cols, ranks, ctypes.byref(total)))
        return list(rows), list(cols), list(ranks), total.value

    @property
    def ranks(self):
        return tuple(self.shape()[2])

    def download(self):
        rows, cols, ranks, total = self.shape()
        buf = np.empty(total, dtype=np.float64)
        check(lib().t2s2_train_download(context(), self.handle, buf.ctypes.data_as(_DP), total))
        is_op = any(c > 0 for c in cols)
        cores, off = [], 0
        for l in range(len(rows)):
            shape = ((ranks[l], rows[l], cols[l], ranks[l + 1]) if is_op
                     else (ranks[l], rows[l], ranks[l + 1]))
            size = int(np.prod(shape))
            cores.append(buf[off: off + size].reshape(shape).copy())
            off += size
        return cores, is_op

    def free(self):
        if self.handle:
            lib().t2s2_train_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
