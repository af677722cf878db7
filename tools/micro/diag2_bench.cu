// Micro-benchmark: the warp-register Gauss-Jordan diagonal block (gj_diag_w)
// against the grouped eight-warp factorisation (gj_diag): cycles per call,
// alone and alternating with the special tile, and both results against a
// host inverse.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DGJ_MICRO \
//        -I paper_2506_04732_b200/csrc tools/micro/diag2_bench.cu -o tools/micro/diag2_bench
#include "../../paper_2506_04732_b200/csrc/gj_solve.cu"

#include <vector>

using namespace t2s2;

// The single-warp register Gauss-Jordan candidate (not in the product: it
// measured 16.4k cycles per block against 10.6k for gj_diag).  Lane i holds
// row i of [D | I], fully unrolled; step st: lane st publishes its row to
// shared memory, every lane forms its multiplier (pivot by one shuffle),
// 32 FMAs.  U^{-1} = D^{-1} L by DMMA on all warps.
struct WarpGj {
  double rowb[2][kP];
  double fm[kP * kP];
};
__device__ WarpGj* g_wgj_unused;

template <int ST>
__device__ __forceinline__ void gjw_step(double (&a)[kP], double (&b)[kP], double& myrinv, bool& ok,
                                         int lane, WarpGj& w) {
  double* rb = w.rowb[ST & 1];
  if (lane == ST) {
#pragma unroll
    for (int j = 0; j < kP; j += 2) {
      double2 v;
      v.x = j > ST ? a[j] : b[j];
      v.y = j + 1 > ST ? a[j + 1] : b[j + 1];
      *reinterpret_cast<double2*>(rb + j) = v;
    }
  }
  const double piv = __shfl_sync(0xffffffffu, a[ST], ST);
  const double rinv = __drcp_rn(piv);
  ok = ok && fabs(piv) > 0.0 && isfinite(piv);
  const double f = lane == ST ? 0.0 : a[ST] * rinv;
  if (lane > ST) ok = ok && fabs(f) <= kPivThresh;
  if (lane == ST) myrinv = rinv;
  w.fm[ST * kP + lane] = f;
  __syncwarp();
#pragma unroll
  for (int j = 0; j < kP; j += 2) {
    const double2 u = *reinterpret_cast<const double2*>(rb + j);
    if (j > ST) a[j] = fma(-f, u.x, a[j]); else b[j] = fma(-f, u.x, b[j]);
    if (j + 1 > ST) a[j + 1] = fma(-f, u.y, a[j + 1]); else b[j + 1] = fma(-f, u.y, b[j + 1]);
  }
}
template <int ST>
struct GjwSteps {
  static __device__ __forceinline__ void run(double (&a)[kP], double (&b)[kP], double& myrinv, bool& ok,
                                             int lane, WarpGj& w) {
    GjwSteps<ST - 1>::run(a, b, myrinv, ok, lane, w);
    gjw_step<ST>(a, b, myrinv, ok, lane, w);
  }
};
template <>
struct GjwSteps<-1> {
  static __device__ __forceinline__ void run(double (&)[kP], double (&)[kP], double&, bool&, int, WarpGj&) {}
};

__device__ void gj_diag_w(const GjArgs& a, int p, int kb, Smem& s) {
  __shared__ __align__(16) WarpGj w;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __syncthreads();
  double* gl = a.inv + (size_t)p * kInv;
  if (warp == 0) {
    double av[kP], bv[kP];
#pragma unroll
    for (int j = 0; j < kP; ++j) {
      av[j] = (lane < kb && j < kb) ? s.dg[j * 33 + lane] : (lane == j ? 1.0 : 0.0);
      bv[j] = lane == j ? 1.0 : 0.0;
    }
    double myrinv = 1.0;
    bool ok = true;
    GjwSteps<kP - 1>::run(av, bv, myrinv, ok, lane, w);
    if (!__all_sync(0xffffffffu, ok) && lane == 0) gj_fail(a);
#pragma unroll
    for (int j = 0; j < kP; ++j) {
      const double v = bv[j] * myrinv;
      s.za[j * kLdP + lane] = v;
      gl[j * kP + lane] = (lane < kb && j < kb) ? v : 0.0;
    }
  }
  __syncthreads();
  {
    const int m0 = (warp >> 1) * 8, n0 = (warp & 1) * 16;
    double acc[2][2] = {};
#pragma unroll
    for (int kk = 0; kk < kP; kk += 4) {
      const int kr = kk + (lane & 3);
      const double af = s.za[kr * kLdP + m0 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = n0 + j * 8 + (lane >> 2);
        const double lf = kr > n ? w.fm[n * kP + kr] : (kr == n ? 1.0 : 0.0);
        dmma(acc[j][0], acc[j][1], af, lf);
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = m0 + (lane >> 2), cc = n0 + j * 8 + (lane & 3) * 2 + h;
        gl[kP * kP + cc * kP + rr] = (rr <= cc && cc < kb) ? acc[j][h] : 0.0;
      }
  }
  __syncthreads();
}

template <int WHICH>
__global__ void diag_loop(GjArgs a, int kb, int reps, long long* cyc) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem& s = *reinterpret_cast<Smem*>(smraw);
  long long t = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < kP * kP; e += kThr) {
      const int c = e >> 5, i = e & 31;
      s.dg[c * 33 + i] = __ldcg(a.A + e);
    }
    __syncthreads();
    long long t0 = clock64();
    if (WHICH == 0) gj_diag(a, 0, kb, s); else gj_diag_w(a, 0, kb, s);
    t += clock64() - t0;
  }
  if (threadIdx.x == 0) *cyc = t / reps;
}

template <int WHICH>
__global__ void special_loop(GjArgs a, int reps, long long* cyc) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem& s = *reinterpret_cast<Smem*>(smraw);
  const Phase ph(a.N, 1);
  long long tt = 0, td = 0;
  for (int r = 0; r < reps; ++r) {
    long long t0 = clock64();
    special_tile(a, ph, s);
    __syncthreads();
    long long t1 = clock64();
    for (int e = threadIdx.x; e < kP * 33; e += kThr) s.dg[e] += (e % 34 == 0) ? 40.0 : 0.0;
    __syncthreads();
    long long t2 = clock64();
    if (WHICH == 0) gj_diag(a, 2, kP, s); else gj_diag_w(a, 2, kP, s);
    long long t3 = clock64();
    tt += t1 - t0;
    td += t3 - t2;
  }
  if (threadIdx.x == 0) {
    cyc[0] = tt / reps;
    cyc[1] = td / reps;
  }
}

static void host_inverse(const std::vector<double>& D, int kb, std::vector<double>& Dinv, std::vector<double>& Uinv) {
  // no-pivot LU, then inverses (long double)
  const int n = kb;
  std::vector<long double> L(n * n, 0), U(n * n, 0), A(n * n);
  for (int c = 0; c < n; ++c) for (int r = 0; r < n; ++r) A[r * n + c] = D[c * kP + r];
  for (int k = 0; k < n; ++k) {
    for (int i = k + 1; i < n; ++i) {
      A[i * n + k] /= A[k * n + k];
      for (int j = k + 1; j < n; ++j) A[i * n + j] -= A[i * n + k] * A[k * n + j];
    }
  }
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) {
    L[i * n + j] = i > j ? A[i * n + j] : (i == j ? 1 : 0);
    U[i * n + j] = i <= j ? A[i * n + j] : 0;
  }
  std::vector<long double> Ui(n * n, 0), Li(n * n, 0);
  for (int c = 0; c < n; ++c) {  // U Ui = I
    for (int i = n - 1; i >= 0; --i) {
      long double v = i == c ? 1 : 0;
      for (int j = i + 1; j < n; ++j) v -= U[i * n + j] * Ui[j * n + c];
      Ui[i * n + c] = v / U[i * n + i];
    }
    for (int i = 0; i < n; ++i) {
      long double v = i == c ? 1 : 0;
      for (int j = 0; j < i; ++j) v -= L[i * n + j] * Li[j * n + c];
      Li[i * n + c] = v;
    }
  }
  Dinv.assign(kP * kP, 0.0);
  Uinv.assign(kP * kP, 0.0);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) {
    long double v = 0;
    for (int k = 0; k < n; ++k) v += Ui[i * n + k] * Li[k * n + j];
    Dinv[j * kP + i] = (double)v;
    Uinv[j * kP + i] = (double)Ui[i * n + j];
  }
}

int main() {
  const int N = 1024;
  double *A, *b, *inv, *wbuf;
  int* info;
  long long* cyc;
  cudaMalloc(&A, sizeof(double) * N * N);
  cudaMalloc(&b, sizeof(double) * N);
  cudaMalloc(&inv, sizeof(double) * 64 * kInv);
  cudaMalloc(&wbuf, sizeof(double) * 3 * kP * (N + 1));
  cudaMalloc(&info, 4);
  cudaMalloc(&cyc, 16);
  cudaMemset(A, 0, sizeof(double) * N * N);
  cudaMemset(inv, 0, sizeof(double) * 64 * kInv);
  cudaMemset(wbuf, 0, sizeof(double) * 3 * kP * (N + 1));
  // a block whose no-pivot multipliers stay below 1: diagonally dominant
  std::vector<double> D(kP * kP);
  unsigned long long st = 12345;
  auto rnd = [&] { st = st * 6364136223846793005ull + 1442695040888963407ull; return (double)(st >> 11) / 9007199254740992.0 - 0.5; };
  for (int c = 0; c < kP; ++c) for (int r = 0; r < kP; ++r) D[c * kP + r] = rnd() + (r == c ? 12.0 : 0.0);
  cudaMemcpy(A, D.data(), sizeof(double) * kP * kP, cudaMemcpyHostToDevice);
  GjArgs a{N, A, b, inv, wbuf, info, nullptr, nullptr};
  const int smem = sizeof(Smem);
  cudaFuncSetAttribute(diag_loop<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(diag_loop<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(special_loop<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(special_loop<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int kb : {32, 19}) {
    std::vector<double> Dinv, Uinv;
    host_inverse(D, kb, Dinv, Uinv);
    for (int which = 0; which < 2; ++which) {
      cudaMemset(inv, 0xff, sizeof(double) * kInv);
      cudaMemset(info, 0, 4);
      long long h;
      for (int it = 0; it < 2; ++it) {
        if (which == 0) diag_loop<0><<<1, kThr, smem>>>(a, kb, 50, cyc); else diag_loop<1><<<1, kThr, smem>>>(a, kb, 50, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      }
      std::vector<double> got(kInv);
      int hinfo;
      cudaMemcpy(got.data(), inv, sizeof(double) * kInv, cudaMemcpyDeviceToHost);
      cudaMemcpy(&hinfo, info, 4, cudaMemcpyDeviceToHost);
      double e1 = 0, e2 = 0, m1 = 0, m2 = 0;
      for (int e = 0; e < kP * kP; ++e) {
        e1 = fmax(e1, fabs(got[e] - Dinv[e]));
        m1 = fmax(m1, fabs(Dinv[e]));
        e2 = fmax(e2, fabs(got[kP * kP + e] - Uinv[e]));
        m2 = fmax(m2, fabs(Uinv[e]));
      }
      printf("kb=%d %s: %lld cycles/call, info %d, max err D^-1 %.2e (scale %.2e), U^-1 %.2e (scale %.2e)\n", kb,
             which ? "gj_diag_w" : "gj_diag  ", h, hinfo, e1, m1, e2, m2);
    }
  }
  // a block that needs an interchange: both must decline
  {
    std::vector<double> D2 = D;
    D2[5 * kP + 5] = 0.01;
    cudaMemcpy(A, D2.data(), sizeof(double) * kP * kP, cudaMemcpyHostToDevice);
    for (int which = 0; which < 2; ++which) {
      cudaMemset(info, 0, 4);
      if (which == 0) diag_loop<0><<<1, kThr, smem>>>(a, 32, 1, cyc); else diag_loop<1><<<1, kThr, smem>>>(a, 32, 1, cyc);
      int hinfo;
      cudaMemcpy(&hinfo, info, 4, cudaMemcpyDeviceToHost);
      printf("small pivot, %s: info %d (expected -1)\n", which ? "gj_diag_w" : "gj_diag  ", hinfo);
    }
    cudaMemcpy(A, D.data(), sizeof(double) * kP * kP, cudaMemcpyHostToDevice);
  }
  for (int which = 0; which < 2; ++which)
    for (int it = 0; it < 2; ++it) {
      if (which == 0) special_loop<0><<<1, kThr, smem>>>(a, 50, cyc); else special_loop<1><<<1, kThr, smem>>>(a, 50, cyc);
      long long hh[2];
      cudaMemcpy(hh, cyc, 16, cudaMemcpyDeviceToHost);
      printf("%s: special tile %lld cycles, then diag %lld cycles (alternating)\n", which ? "gj_diag_w" : "gj_diag  ", hh[0], hh[1]);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
