// One-launch dense solve A x = b (partial pivoting) for the local systems of
// the alternating solver: a cooperative kernel over all SMs.
//
// Per panel of w columns:
//   1. CTA 0 loads the panel (N-k0) x w into shared memory and factors it
//      there (warp-shuffle argmax pivot search, in-smem swaps and rank-1
//      updates), then writes it back with the pivot rows.
//   2. grid barrier.
//   3. Every CTA owns 16-column blocks of the trailing matrix [k0+w, N]
//      (column N is the right-hand side, so forward substitution comes for
//      free): it applies the panel's interchanges, the unit-lower TRSM for
//      U12 and the rank-w update A22 -= L21 U12 on its columns only, so no
//      other CTA reads or writes them and one barrier per panel suffices.
//   4. grid barrier.
// After the last panel CTA 0 back-substitutes U x = y with x in shared
// memory (32-row diagonal blocks staged in registers of one warp).
//
// The matrix (<= 2000^2 doubles, 32 MB) stays L2-resident across the whole
// factorisation; the L factor is never applied to the left columns because
// the augmented column already carries L^{-1} P b.
#include <cooperative_groups.h>

#include <cmath>

#include "blas.h"
#include "linalg.h"

namespace cg = cooperative_groups;

namespace t2s2 {
namespace {

constexpr int kThreads = 512;
constexpr int kColBlock = 8;
constexpr int kMaxPanel = 32;
constexpr size_t kPanelSmem = 200 * 1024;

__device__ __forceinline__ void amax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

struct LuArgs {
  int N;
  double* A;     // column-major N x N, ld = N
  double* b;     // rhs (N), overwritten with x
  int* piv;      // N scratch (absolute pivot rows)
  int* info;     // 0 or 1 + first zero pivot
  int w;         // panel width
};

// Factor the panel A[k0:N, k0:k0+w] with partial pivoting inside one CTA,
// one barrier per column: rows never move while factoring (a chosen pivot
// row is flagged done and read in place), so each thread only touches its
// own rows; the LAPACK-order interchanges are replayed on an index map and
// applied when the panel is written back.
__device__ void factor_panel(const LuArgs& a, int k0, int w, double* sm, int* s_piv) {
  const int N = a.N, rows = N - k0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  __shared__ double rv[2][32];
  __shared__ int ri[2][32];
  int* cur = reinterpret_cast<int*>(sm + (size_t)rows * w);  // position -> physical row
  int* pos = cur + rows;                                      // physical row -> position
  unsigned char* done = reinterpret_cast<unsigned char*>(pos + rows);
  for (long long e = tid; e < (long long)rows * w; e += blockDim.x) {
    const int c = (int)(e / rows), r = (int)(e % rows);
    sm[e] = a.A[(long long)(k0 + c) * N + k0 + r];
  }
  for (int r = tid; r < rows; r += blockDim.x) {
    cur[r] = r;
    pos[r] = r;
    done[r] = 0;
  }
  __syncthreads();
  for (int j = 0; j < w; ++j) {
    const double* cj = sm + (long long)j * rows;
    double best = -1.0;
    int bi = rows;
    for (int r = tid; r < rows; r += blockDim.x)
      if (!done[r]) amax_merge(best, bi, fabs(cj[r]), r);
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      amax_merge(best, bi, v2, i2);
    }
    if (lane == 0) {
      rv[j & 1][warp] = best;
      ri[j & 1][warp] = bi;
    }
    __syncthreads();
    best = lane < nw ? rv[j & 1][lane] : -1.0;
    bi = lane < nw ? ri[j & 1][lane] : rows;
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      amax_merge(best, bi, v2, i2);
    }
    const int p = bi;  // physical pivot row (ties -> lowest physical index)
    const double pv = cj[p];
    if (tid == 0) {
      // replay the interchange j <-> position of p (LAPACK order)
      const int pp = pos[p];
      a.piv[k0 + j] = k0 + pp;
      const int rj = cur[j];
      cur[j] = p;
      cur[pp] = rj;
      pos[p] = j;
      pos[rj] = pp;
      if (pv == 0.0 && *a.info == 0) *a.info = k0 + j + 1;
    }
    const double inv = pv != 0.0 ? 1.0 / pv : 0.0;
    for (int r = tid; r < rows; r += blockDim.x) {
      if (r == p) {
        done[r] = 1;
        continue;
      }
      if (done[r]) continue;
      const double l = pv != 0.0 ? cj[r] * inv : cj[r];
      sm[(long long)j * rows + r] = l;
      for (int c = j + 1; c < w; ++c) {
        double* cc = sm + (long long)c * rows;
        cc[r] = fma(-l, cc[p], cc[r]);
      }
    }
  }
  __syncthreads();
  for (long long e = tid; e < (long long)rows * w; e += blockDim.x) {
    const int c = (int)(e / rows), i = (int)(e % rows);
    a.A[(long long)(k0 + c) * N + k0 + i] = sm[(long long)c * rows + cur[i]];
  }
}

// Interchanges, TRSM and rank-w update of the owned columns [c0, c1)
// (at most kMaxPanel of them; column N is the right-hand side).
__device__ void update_cols(const LuArgs& a, int k0, int w, int c0, int c1, double* sm) {
  const int N = a.N;
  const int tid = threadIdx.x;
  const int nc = c1 - c0;
  double* L11 = sm;                        // w x w (col-major)
  double* U = sm + kMaxPanel * kMaxPanel;  // w x nc (row j, column c at j*kMaxPanel + c)
  for (int c = tid; c < nc; c += blockDim.x) {
    const int gc = c0 + c;
    double* col = gc < N ? a.A + (long long)gc * N : a.b;
    for (int j = 0; j < w; ++j) {
      const int p = a.piv[k0 + j];
      if (p != k0 + j) {
        const double t = col[k0 + j];
        col[k0 + j] = col[p];
        col[p] = t;
      }
    }
  }
  for (int e = tid; e < w * w; e += blockDim.x) {
    const int c = e / w, r = e % w;
    L11[c * w + r] = a.A[(long long)(k0 + c) * N + k0 + r];
  }
  __syncthreads();
  for (int c = tid; c < nc; c += blockDim.x) {
    const int gc = c0 + c;
    double* col = gc < N ? a.A + (long long)gc * N : a.b;
    double x[kMaxPanel];
#pragma unroll
    for (int j = 0; j < kMaxPanel; ++j) x[j] = j < w ? col[k0 + j] : 0.0;
#pragma unroll
    for (int j = 0; j < kMaxPanel; ++j) {
      if (j < w) {
#pragma unroll
        for (int i = j + 1; i < kMaxPanel; ++i)
          if (i < w) x[i] = fma(-L11[j * w + i], x[j], x[i]);
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxPanel; ++j)
      if (j < w) {
        col[k0 + j] = x[j];
        U[j * kMaxPanel + c] = x[j];
      }
  }
  __syncthreads();
  // A22[:, c0:c1] -= L21 U12: one thread per row keeps its L21 row in
  // registers and sweeps the owned columns (U12 broadcast from smem).
  for (int r = k0 + w + tid; r < N; r += blockDim.x) {
    double l[kMaxPanel];
#pragma unroll
    for (int j = 0; j < kMaxPanel; ++j) l[j] = j < w ? a.A[(long long)(k0 + j) * N + r] : 0.0;
    for (int c = 0; c < nc; ++c) {
      const int gc = c0 + c;
      double* col = gc < N ? a.A + (long long)gc * N : a.b;
      double acc = col[r];
#pragma unroll
      for (int j = 0; j < kMaxPanel; ++j)
        if (j < w) acc = fma(-l[j], U[j * kMaxPanel + c], acc);
      col[r] = acc;
    }
  }
  __syncthreads();
}

__device__ void back_substitute(const LuArgs& a, double* x) {
  const int N = a.N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < N; i += blockDim.x) x[i] = a.b[i];
  __syncthreads();
  for (int j1 = N; j1 > 0; j1 -= 32) {
    const int j0 = j1 - 32 > 0 ? j1 - 32 : 0;
    const int jb = j1 - j0;
    if (warp == 0) {
      // lane i holds row j0+i of the diagonal block
      double u[32];
#pragma unroll
      for (int c = 0; c < 32; ++c)
        u[c] = (lane < jb && c < jb) ? a.A[(long long)(j0 + c) * N + j0 + lane] : 0.0;
      double xi = lane < jb ? x[j0 + lane] : 0.0;
#pragma unroll
      for (int c = 31; c >= 0; --c) {
        if (c < jb) {
          double v = 0.0;
          if (lane == c) v = xi / u[c];
          v = __shfl_sync(0xffffffffu, v, c);
          if (lane == c) xi = v;
          if (lane < c) xi = fma(-u[c], v, xi);
        }
      }
      if (lane < jb) x[j0 + lane] = xi;
    }
    __syncthreads();
    for (int i = tid; i < j0; i += blockDim.x) {
      double acc = x[i];
      for (int c = 0; c < jb; ++c) acc = fma(-a.A[(long long)(j0 + c) * N + i], x[j0 + c], acc);
      x[i] = acc;
    }
    __syncthreads();
  }
  for (int i = tid; i < N; i += blockDim.x) a.b[i] = x[i];
}

// Lookahead schedule: while the other CTAs apply panel p to the trailing
// columns, CTA 0 updates the columns of panel p+1 and factors it, so the
// panel factorisations form the critical path with one grid barrier each.
__global__ void __launch_bounds__(kThreads, 1) lu_fused_kernel(LuArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  __shared__ int s_piv[kMaxPanel];
  const int N = a.N;
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) *a.info = 0;
    __syncthreads();
    factor_panel(a, 0, N < a.w ? N : a.w, sm, s_piv);
  }
  grid.sync();
  for (int k0 = 0; k0 < N; k0 += a.w) {
    const int w = N - k0 < a.w ? N - k0 : a.w;
    const int k1 = k0 + w;                               // next panel start
    const int w2 = N - k1 < a.w ? N - k1 : a.w;          // next panel width (0 at end)
    const int rest0 = k1 + w2;                           // columns for the other CTAs
    if (blockIdx.x == 0) {
      if (w2 > 0) {
        update_cols(a, k0, w, k1, rest0, sm);
        factor_panel(a, k1, w2, sm, s_piv);
      }
    }
    const int workers = gridDim.x > 1 ? gridDim.x - 1 : 1;
    const int wid = gridDim.x > 1 ? (int)blockIdx.x - 1 : 0;
    if (gridDim.x == 1 || blockIdx.x > 0) {
      const int ncols = N + 1 - rest0;
      const int nblk = (ncols + kColBlock - 1) / kColBlock;
      for (int blk = wid; blk < nblk; blk += workers) {
        const int c0 = rest0 + blk * kColBlock;
        const int c1 = c0 + kColBlock < N + 1 ? c0 + kColBlock : N + 1;
        update_cols(a, k0, w, c0, c1, sm);
      }
    }
    grid.sync();
  }
  if (blockIdx.x == 0) back_substitute(a, sm);
}

int g_num_sms = 0;

}  // namespace

bool lu_solve_fused(int N, double* A, double* b, int* piv, int* info_dev) {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    T2S2_CUDA(cudaFuncSetAttribute(lu_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kPanelSmem));
  }
  // panel doubles plus the row maps (2 ints + 1 byte per row)
  int w = (int)((kPanelSmem - 9 * (size_t)N) / (sizeof(double) * (size_t)N));
  if (w > kMaxPanel) w = kMaxPanel;
  if (w < 1) return false;  // caller falls back to the multi-launch path
  LuArgs a{N, A, b, piv, info_dev, w};
  void* params[] = {&a};
  {
    // algorithmic: 2/3 N^3 (factor) + 2 N^2 (solves); bytes: matrix read+write
    LaunchScope ls("lu_fused", 2.0 / 3.0 * (double)N * N * N + 2.0 * (double)N * N,
                   16.0 * (double)N * N);
    T2S2_CUDA(cudaLaunchCooperativeKernel((void*)lu_fused_kernel, dim3(g_num_sms), dim3(kThreads),
                                          params, kPanelSmem, stream()));
  }
  return true;
}

}  // namespace t2s2
