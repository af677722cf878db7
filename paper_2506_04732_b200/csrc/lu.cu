// LU with partial pivoting for the dense local systems of the alternating
// solver (Galerkin and normal-equation blocks, N = r_{l-1} n_l r_l <= the
// direct-solve threshold).
//
// Blocked right-looking getrf on a column-major matrix resident in L2:
// per panel of NB columns one CTA factors the panel (pivot search by
// warp-shuffle argmax), a column-parallel kernel applies the interchanges
// and the unit-lower TRSM to the block row, and the tiled GEMM updates the
// trailing matrix.  The solve keeps the right-hand side in shared memory and
// walks 32-row diagonal blocks with one warp while the block's GEMV runs on
// the whole CTA.
#include <cmath>

#include "blas.h"
#include "linalg.h"

namespace t2s2 {
namespace {

constexpr int NB = 32;
constexpr int kPanelThreads = 1024;

__device__ __forceinline__ void argmax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

// Factor A[k0:N, k0:k0+nb] in place (column-major, ld = N).
__global__ void __launch_bounds__(kPanelThreads)
    panel_kernel(int N, double* A, int k0, int nb, int* ipiv, int* info) {
  __shared__ double wv[32];
  __shared__ int wi[32];
  __shared__ int sh_piv;
  __shared__ double sh_pval;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int j = 0; j < nb; ++j) {
    const int cj = k0 + j;
    double* col = A + (long long)cj * N;
    double best = -1.0;
    int bi = N;
    for (int i = cj + tid; i < N; i += blockDim.x) argmax_merge(best, bi, fabs(col[i]), i);
    for (int o = 16; o > 0; o >>= 1) {
      double v2 = __shfl_xor_sync(0xffffffffu, best, o);
      int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      argmax_merge(best, bi, v2, i2);
    }
    if (lane == 0) {
      wv[warp] = best;
      wi[warp] = bi;
    }
    __syncthreads();
    if (warp == 0) {
      best = lane < nwarps ? wv[lane] : -1.0;
      bi = lane < nwarps ? wi[lane] : N;
      for (int o = 16; o > 0; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, best, o);
        int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        argmax_merge(best, bi, v2, i2);
      }
      if (lane == 0) {
        sh_piv = bi;
        ipiv[cj] = bi;
        sh_pval = col[bi];
        if (col[bi] == 0.0 && *info == 0) *info = cj + 1;
      }
    }
    __syncthreads();
    const int p = sh_piv;
    const double pv = sh_pval;
    if (p != cj) {
      for (int c = tid; c < nb; c += blockDim.x) {
        double* cc = A + (long long)(k0 + c) * N;
        double t = cc[cj];
        cc[cj] = cc[p];
        cc[p] = t;
      }
    }
    __syncthreads();
    if (pv != 0.0) {
      const double rinv = 1.0 / pv;
      for (int i = cj + 1 + tid; i < N; i += blockDim.x) col[i] *= rinv;
    }
    __syncthreads();
    // rank-1 update of the remaining panel columns, one warp per column
    for (int c = j + 1 + warp; c < nb; c += nwarps) {
      double* cc = A + (long long)(k0 + c) * N;
      const double u = cc[cj];
      if (u != 0.0)
        for (int i = cj + 1 + lane; i < N; i += 32) cc[i] = fma(-col[i], u, cc[i]);
    }
    __syncthreads();
  }
}

// Apply the panel's interchanges to the other columns; then, for columns
// right of the panel, U12 = L11^{-1} A12 (unit lower, nb x nb).
__global__ void swap_trsm_kernel(int N, double* A, int k0, int nb, const int* ipiv) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N || (c >= k0 && c < k0 + nb)) return;
  double* cc = A + (long long)c * N;
  for (int j = 0; j < nb; ++j) {
    int p = ipiv[k0 + j];
    if (p != k0 + j) {
      double t = cc[k0 + j];
      cc[k0 + j] = cc[p];
      cc[p] = t;
    }
  }
  if (c < k0 + nb) return;
  double x[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) x[j] = j < nb ? cc[k0 + j] : 0.0;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    if (j >= nb) break;
    const double* lj = A + (long long)(k0 + j) * N + k0;  // column k0+j of L11
#pragma unroll
    for (int i = j + 1; i < NB; ++i)
      if (i < nb) x[i] = fma(-lj[i], x[j], x[i]);
  }
#pragma unroll
  for (int j = 0; j < NB; ++j)
    if (j < nb) cc[k0 + j] = x[j];
}

constexpr int kSolveThreads = 512;

// Forward/backward substitution with one rhs staged in shared memory.
__global__ void __launch_bounds__(kSolveThreads)
    lu_solve_kernel(int N, const double* __restrict__ LU, const int* __restrict__ ipiv,
                    double* b) {
  extern __shared__ double x[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < N; i += blockDim.x) x[i] = b[i];
  __syncthreads();
  int* sp = reinterpret_cast<int*>(x + N);
  for (int i = tid; i < N; i += blockDim.x) sp[i] = ipiv[i];
  __syncthreads();
  if (tid == 0)
    for (int i = 0; i < N; ++i) {
      int p = sp[i];
      if (p != i) {
        double t = x[i];
        x[i] = x[p];
        x[p] = t;
      }
    }
  __syncthreads();
  // L y = P b (unit lower)
  for (int j0 = 0; j0 < N; j0 += 32) {
    const int jb = min(32, N - j0);
    if (warp == 0) {
      for (int jj = 0; jj < jb; ++jj) {
        const double xj = x[j0 + jj];
        __syncwarp();
        if (lane > jj && lane < jb)
          x[j0 + lane] = fma(-LU[(long long)(j0 + jj) * N + j0 + lane], xj, x[j0 + lane]);
        __syncwarp();
      }
    }
    __syncthreads();
    for (int i = j0 + jb + tid; i < N; i += blockDim.x) {
      double acc = x[i];
      for (int jj = 0; jj < jb; ++jj) acc = fma(-LU[(long long)(j0 + jj) * N + i], x[j0 + jj], acc);
      x[i] = acc;
    }
    __syncthreads();
  }
  // U x = y, bottom-up blocks
  for (int j1 = N; j1 > 0; j1 -= 32) {
    const int j0 = j1 - 32 > 0 ? j1 - 32 : 0;
    const int jb = j1 - j0;
    if (warp == 0) {
      for (int jj = jb - 1; jj >= 0; --jj) {
        __syncwarp();
        if (lane == jj) x[j0 + jj] = x[j0 + jj] / LU[(long long)(j0 + jj) * N + j0 + jj];
        __syncwarp();
        const double xj = x[j0 + jj];
        if (lane < jj)
          x[j0 + lane] = fma(-LU[(long long)(j0 + jj) * N + j0 + lane], xj, x[j0 + lane]);
      }
      __syncwarp();
    }
    __syncthreads();
    for (int i = tid; i < j0; i += blockDim.x) {
      double acc = x[i];
      for (int jj = 0; jj < jb; ++jj) acc = fma(-LU[(long long)(j0 + jj) * N + i], x[j0 + jj], acc);
      x[i] = acc;
    }
    __syncthreads();
  }
  for (int i = tid; i < N; i += blockDim.x) b[i] = x[i];
}

}  // namespace

void lu_factor(int N, double* A, int* ipiv, int* info_dev) {
  T2S2_CUDA(cudaMemsetAsync(info_dev, 0, sizeof(int), stream()));
  for (int k0 = 0; k0 < N; k0 += NB) {
    const int nb = N - k0 < NB ? N - k0 : NB;
    {
      LaunchScope ls("lu_panel", (double)(N-k0)*nb*nb, 16.0*(double)(N-k0)*nb);
      panel_kernel<<<1, kPanelThreads, 0, stream()>>>(N, A, k0, nb, ipiv, info_dev);
    }
    T2S2_CHECK_LAUNCH();
    {
      LaunchScope ls("lu_trsm", (double)(N-k0-nb)*nb*nb, 16.0*(double)N*nb);
      swap_trsm_kernel<<<ceil_div(N, 128), 128, 0, stream()>>>(N, A, k0, nb, ipiv);
    }
    T2S2_CHECK_LAUNCH();
    const int rest = N - k0 - nb;
    if (rest > 0) {
      // column-major A22 -= A21 A12  <=>  row-major A22^T -= A12^T A21^T
      gemm(false, false, rest, rest, nb, -1.0, A + (long long)(k0 + nb) * N + k0, N,
           A + (long long)k0 * N + (k0 + nb), N, 1.0, A + (long long)(k0 + nb) * N + (k0 + nb),
           N);
    }
  }
}

void lu_solve(int N, const double* LU, const int* ipiv, double* b) {
  size_t smem = (size_t)N * (sizeof(double) + sizeof(int));
  T2S2_REQUIRE(smem <= 200 * 1024, kErrCapacity, "lu_solve: system too large for smem rhs");
  if (smem > 48 * 1024)
    T2S2_CUDA(cudaFuncSetAttribute(lu_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
  {
    LaunchScope ls("lu_solve", 2.0*(double)N*N, 8.0*(double)N*N);
    lu_solve_kernel<<<1, kSolveThreads, smem, stream()>>>(N, LU, ipiv, b);
  }
  T2S2_CHECK_LAUNCH();
}

}  // namespace t2s2
