"""The engine's GEMM program kernel against cuBLAS (torch.matmul, fp64) on
the contraction shapes of a rank-64 config-4 normal-operator application
and a square reference shape (development tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import _native  # noqa: E402

shapes = [  # (name, M, N, K)
    ("stage1 x.a1.a2 x n.w x z", 1024, 2112, 64),
    ("stage2/3 operator core (x.a.w) x m.A x a.n", 16384, 132, 132),
    ("stage4 x.m x y x A1.A2.w", 2112, 64, 1024),
    ("stage2-like 132 x 64 x 132 (one batch entry)", 132, 64, 132),
    ("square 2048", 2048, 2048, 2048),
    ("square 4096", 4096, 4096, 4096),
]
dev = torch.device("cuda")
_native.context()
for name, M, N, K in shapes:
    a = torch.randn(M, K, dtype=torch.float64, device=dev)
    b = torch.randn(K, N, dtype=torch.float64, device=dev)
    c = torch.empty(M, N, dtype=torch.float64, device=dev)
    ref = a @ b
    _native.gemm_device(0, 0, M, N, K, a.data_ptr(), K, b.data_ptr(), N, c.data_ptr(), N)
    _native.synchronize()
    err = ((c - ref).norm() / ref.norm()).item()
    st = torch.cuda.Stream(device=dev)  # noqa: F841
    reps = 20
    _native.stats_reset(profile_events=True)
    for _ in range(reps):
        _native.gemm_device(0, 0, M, N, K, a.data_ptr(), K, b.data_ptr(), N, c.data_ptr(), N)
    s = _native.stats_read()["gemm"]
    ours = s["device_ms"] / reps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    cub = e0.elapsed_time(e1) / reps
    fl = 2.0 * M * N * K
    print(f"{name:48s} ours {ours * 1e3:9.1f} us {fl / ours / 1e9:6.2f} TF | cuBLAS {cub * 1e3:9.1f} us"
          f" {fl / cub / 1e9:6.2f} TF | rel err {err:.1e}", flush=True)
