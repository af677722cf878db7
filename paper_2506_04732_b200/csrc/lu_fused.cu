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
#include <cstdio>
#include <cstdlib>

#include "blas.h"
#include "linalg.h"

namespace cg = cooperative_groups;

namespace t2s2 {
namespace {

constexpr int kThreads = 512;
constexpr int kColBlock = 8;
constexpr int kMaxPanel = 32;
constexpr int kRowsPerThread = 5;  // rows <= 5 * 512 = 2560
constexpr size_t kPanelSmem = 200 * 1024;
constexpr int kMoveStride = 2 * (1 + 2 * 2 * kMaxPanel);

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
  int* moves;    // per panel: count, then (dst, src) row offsets relative to k0
  int* flag;     // next-panel chunk completion counter (zeroed by the host)
  unsigned long long* prof;  // optional phase timers (ns): see lu_solve_fused
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Column loop of the panel factorisation: thread t owns rows t + k*kThreads
// (k < RPT); liveness and multipliers stay in registers, values in smem.
// Column loop of the panel factorisation.  Thread t owns rows t + k*kThreads
// (k < RPT).  The panel is processed in register sub-panels of SUB columns:
// a sub-panel's values of the thread's rows live in registers, so a column
// step touches shared memory only to publish candidate pivot rows; one CTA
// barrier per column.  After a sub-panel, its pivot rows' U entries right of
// it are formed (unit-lower forward substitution) and one rank-SUB update is
// applied to the rest of the panel in shared memory.
constexpr int SUB = 8;

template <int RPT>
__device__ __forceinline__ void factor_columns(int rows, int w, double* sm, int* s_piv) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = kThreads / 32;
  __shared__ unsigned rh[2][nw], rl[2][nw];
  __shared__ int ri[2][nw];
  __shared__ double pub[2][nw][SUB];  // each warp's candidate pivot row (sub-panel part)
  __shared__ double pinv[2][nw];      // and the reciprocal of its pivot entry
  bool live[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) live[k] = tid + k * kThreads < rows;
  for (int j0 = 0; j0 < w; j0 += SUB) {
    const int nsub = w - j0 < SUB ? w - j0 : SUB;
    double a[RPT][SUB];
#pragma unroll
    for (int k = 0; k < RPT; ++k)
#pragma unroll
      for (int t = 0; t < SUB; ++t)
        a[k][t] = (tid + k * kThreads < rows && t < nsub) ? sm[(j0 + t) * rows + tid + k * kThreads]
                                                         : 0.0;
#pragma unroll
    for (int t = 0; t < SUB; ++t) {
      if (t >= nsub) break;
      const int j = j0 + t;
      const int buf = j & 1;
      // local candidate: largest |a| among live own rows (first row on ties)
      unsigned long long kb = 0ull;
      int bi = 0x7fffffff, bk = 0;
#pragma unroll
      for (int k = 0; k < RPT; ++k)
        if (live[k]) {
          const unsigned long long b = __double_as_longlong(fabs(a[k][t]));
          if (b > kb || bi == 0x7fffffff) {
            kb = b;
            bi = tid + k * kThreads;
            bk = k;
          }
        }
      const unsigned hi = bi == 0x7fffffff ? 0u : (unsigned)(kb >> 32);
      const unsigned lo = bi == 0x7fffffff ? 0u : (unsigned)kb;
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      const int mi = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bi : 0x7fffffff);
      if (bi == mi && mi != 0x7fffffff) {
        // the warp winner publishes its row's sub-panel values (cols > t)
        // and the reciprocal of its candidate pivot (slot t)
#pragma unroll
        for (int q = 0; q < SUB; ++q) {
          double v = 0.0;
#pragma unroll
          for (int k = 0; k < RPT; ++k)
            if (k == bk) v = a[k][q];
          if (q > t) pub[buf][warp][q] = v;
          if (q == t) {
            pub[buf][warp][q] = v;
            pinv[buf][warp] = v != 0.0 ? __drcp_rn(v) : 1.0;
          }
        }
      }
      if (lane == 0) {
        rh[buf][warp] = mh;
        rl[buf][warp] = ml;
        ri[buf][warp] = mi;
      }
      __syncthreads();
      const unsigned h2 = lane < nw ? rh[buf][lane] : 0u;
      const unsigned l2 = lane < nw ? rl[buf][lane] : 0u;
      const int i2 = lane < nw ? ri[buf][lane] : 0x7fffffff;
      const unsigned gh = __reduce_max_sync(0xffffffffu, h2);
      const unsigned gl = __reduce_max_sync(0xffffffffu, h2 == gh ? l2 : 0u);
      const int p = __reduce_min_sync(0xffffffffu, (h2 == gh && l2 == gl) ? i2 : 0x7fffffff);
      const int pw = __ffs(__ballot_sync(0xffffffffu, lane < nw && i2 == p)) - 1;  // winner warp
      double prow[SUB];
#pragma unroll
      for (int q = 0; q < SUB; ++q) prow[q] = q >= t ? pub[buf][pw][q] : 0.0;
      if (tid == 0) s_piv[j] = p;
      const double inv = pinv[buf][pw];
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        if (tid + k * kThreads == p) live[k] = false;
        if (live[k]) {
          const double l = a[k][t] * inv;
          a[k][t] = l;
#pragma unroll
          for (int q = 0; q < SUB; ++q)
            if (q > t) a[k][q] = fma(-l, prow[q], a[k][q]);
        }
      }
    }
    // sub-panel back to shared memory (pivot rows keep their U entries,
    // the others their multipliers)
#pragma unroll
    for (int k = 0; k < RPT; ++k)
#pragma unroll
      for (int t = 0; t < SUB; ++t)
        if (tid + k * kThreads < rows && t < nsub) sm[(j0 + t) * rows + tid + k * kThreads] = a[k][t];
    const int je = j0 + nsub;
    if (je < w) {
      __syncthreads();
      // U entries of the sub-panel's pivot rows right of it (one thread per
      // column): u_t = a[p_t][c] - sum_{q<t} l[p_t][q] u_q
      for (int c = je + tid; c < w; c += kThreads) {
        double u[SUB];
#pragma unroll
        for (int t = 0; t < SUB; ++t) {
          u[t] = 0.0;
          if (t < nsub) {
            const int pt = s_piv[j0 + t];
            double x = sm[c * rows + pt];
#pragma unroll
            for (int q = 0; q < SUB; ++q)
              if (q < t) x = fma(-sm[(j0 + q) * rows + pt], u[q], x);
            u[t] = x;
            sm[c * rows + pt] = x;
          }
        }
      }
      __syncthreads();
      // rank-nsub update of the live rows, columns je..w-1
      for (int c = je; c < w; ++c) {
        double ut[SUB];
#pragma unroll
        for (int t = 0; t < SUB; ++t) ut[t] = t < nsub ? sm[c * rows + s_piv[j0 + t]] : 0.0;
#pragma unroll
        for (int k = 0; k < RPT; ++k)
          if (live[k]) {
            double x = sm[c * rows + tid + k * kThreads];
#pragma unroll
            for (int t = 0; t < SUB; ++t) x = fma(-a[k][t], ut[t], x);
            sm[c * rows + tid + k * kThreads] = x;
          }
      }
      __syncthreads();
    }
  }
}

// Factor the panel A[k0:N, k0:k0+w] with partial pivoting inside one CTA,
// one barrier per column: rows never move while factoring (a chosen pivot
// row is flagged done and read in place), so each thread only touches its
// own rows; the LAPACK-order interchanges are replayed on an index map and
// applied when the panel is written back.
__device__ __forceinline__ void factor_panel(const LuArgs& a, int k0, int w, double* sm, int* s_piv,
                                          int* mv) {
  const int N = a.N, rows = N - k0;
  const int tid = threadIdx.x;
  int* cur = reinterpret_cast<int*>(sm + (size_t)rows * w);  // position -> physical row
  int* pos = cur + rows;                                      // physical row -> position
  for (int c = 0; c < w; ++c) {
    const double* src = a.A + (long long)(k0 + c) * N + k0;
    double* dst = sm + (long long)c * rows;
    for (int r = tid; r < rows; r += blockDim.x) dst[r] = __ldcg(src + r);
  }
  for (int r = tid; r < rows; r += blockDim.x) {
    cur[r] = r;
    pos[r] = r;
  }
  __syncthreads();
  if (rows <= kThreads)
    factor_columns<1>(rows, w, sm, s_piv);
  else if (rows <= 2 * kThreads)
    factor_columns<2>(rows, w, sm, s_piv);
  else if (rows <= 3 * kThreads)
    factor_columns<3>(rows, w, sm, s_piv);
  else if (rows <= 4 * kThreads)
    factor_columns<4>(rows, w, sm, s_piv);
  else
    factor_columns<5>(rows, w, sm, s_piv);
  // replay the interchanges in LAPACK order on the index maps
  __syncthreads();
  if (tid == 0) {
    for (int j = 0; j < w; ++j) {
      const int p = s_piv[j];
      const int pp = pos[p];
      a.piv[k0 + j] = k0 + pp;
      const int rj = cur[j];
      cur[j] = p;
      cur[pp] = rj;
      pos[p] = j;
      pos[rj] = pp;
      if (sm[j * rows + p] == 0.0 && *a.info == 0) *a.info = k0 + j + 1;
    }
  }
  __syncthreads();
  for (int c = 0; c < w; ++c) {
    double* dst = a.A + (long long)(k0 + c) * N + k0;
    const double* src = sm + (long long)c * rows;
    for (int i = tid; i < rows; i += blockDim.x) dst[i] = src[cur[i]];
  }
  // rows whose position changed: at most 2w of them (the first w positions
  // and the slots the pivots came from); other CTAs replay them per column
  if (tid == 0) {
    int m = 0;
    for (int i = 0; i < w; ++i)
      if (cur[i] != i) {
        mv[1 + 2 * m] = i;
        mv[2 + 2 * m] = cur[i];
        ++m;
      }
    // displaced rows: physical row q (< w) that ended at position pos[q] >= w
    for (int q = 0; q < w; ++q)
      if (pos[q] >= w) {
        mv[1 + 2 * m] = pos[q];
        mv[2 + 2 * m] = q;
        ++m;
      }
    mv[0] = m;
  }
}

// Interchanges, TRSM and rank-w update of the owned columns [c0, c1),
// at most CB of them (column N is the right-hand side).  Loops over the
// panel width stay rolled: the kernel must fit the instruction cache, since
// every phase runs once per panel.
template <int CB>
__device__ __forceinline__ void update_cols(const LuArgs& a, int k0, int w, int c0, int c1,
                                         double* sm, const int* mv) {
  const int N = a.N;
  const int tid = threadIdx.x;
  const int nc = c1 - c0;
  double* L11 = sm;                        // w x w (col-major)
  double* U = sm + kMaxPanel * kMaxPanel;  // row j, column c at j * CB + c
  {
    // replay the panel's row moves: gather every moved value, then scatter
    const int m = mv[0];
    const int pairs = m * nc;
    double v[4];
    int dst[4], cc[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int e = tid + t * blockDim.x;
      dst[t] = -1;
      if (e < pairs) {
        const int c = e / m, k = e % m;
        const int gc = c0 + c;
        const double* col = gc < N ? a.A + (long long)gc * N : a.b;
        dst[t] = mv[1 + 2 * k];
        cc[t] = c;
        v[t] = col[k0 + mv[2 + 2 * k]];
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (dst[t] >= 0) {
        const int gc = c0 + cc[t];
        double* col = gc < N ? a.A + (long long)gc * N : a.b;
        col[k0 + dst[t]] = v[t];
      }
  }
  __syncthreads();
  for (int e = tid; e < w * w; e += blockDim.x) {
    const int c = e / w, r = e % w;
    L11[c * w + r] = a.A[(long long)(k0 + c) * N + k0 + r];
  }
  for (int e = tid; e < w * nc; e += blockDim.x) {
    const int c = e / w, j = e % w;
    const int gc = c0 + c;
    const double* col = gc < N ? a.A + (long long)gc * N : a.b;
    U[j * CB + c] = col[k0 + j];
  }
  // rows w..31 of U take part in the 16-wide register blocks: keep them zero
  for (int e = tid; e < (kMaxPanel - w) * CB; e += blockDim.x) U[w * CB + e] = 0.0;
  __syncthreads();
  // U12 = L11^{-1} A12: one warp per column, lane i holds row i
  {
    const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    for (int c = warp; c < nc; c += nwarps) {
      double xi = lane < w ? U[lane * CB + c] : 0.0;
      double lcol = 0.0;
#pragma unroll 1
      for (int j = 0; j < w; ++j) {
        lcol = lane < w ? L11[j * w + lane] : 0.0;
        const double xj = __shfl_sync(0xffffffffu, xi, j);
        if (lane > j) xi = fma(-lcol, xj, xi);
      }
      if (lane < w) U[lane * CB + c] = xi;
    }
  }
  __syncthreads();
  for (int e = tid; e < w * nc; e += blockDim.x) {
    const int c = e / w, j = e % w;
    const int gc = c0 + c;
    double* col = gc < N ? a.A + (long long)gc * N : a.b;
    col[k0 + j] = U[j * CB + c];
  }
  // A22[:, c0:c1] -= L21 U12: thread per row; its L21 row is prefetched into
  // registers (independent loads), columns are processed 8 at a time.
  for (int r = k0 + w + tid; r < N; r += blockDim.x) {
#pragma unroll 1
    for (int cb = 0; cb < nc; cb += 8) {
      double acc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int gc = c0 + cb + c;
        acc[c] = cb + c < nc ? (gc < N ? a.A[(long long)gc * N + r] : a.b[r]) : 0.0;
      }
#pragma unroll 1
      for (int j0 = 0; j0 < w; j0 += 16) {
        double l[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          l[j] = j0 + j < w ? a.A[(long long)(k0 + j0 + j) * N + r] : 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[c] = fma(-l[j], U[(j0 + j) * CB + cb + c], acc[c]);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int gc = c0 + cb + c;
        if (cb + c < nc) {
          if (gc < N)
            a.A[(long long)gc * N + r] = acc[c];
          else
            a.b[r] = acc[c];
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void back_substitute(const LuArgs& a, double* x) {
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
__device__ __forceinline__ int panel_width(int rows) {
  // panel values plus the two int row maps must fit the dynamic smem
  int w = (int)((kPanelSmem - 8 * (size_t)rows) / (8 * (size_t)rows));
  return w > kMaxPanel ? kMaxPanel : (w < 1 ? 1 : w);
}

// Schedule per iteration (panel p = [k0, k0+w) already factored):
//   workers (CTAs 1..G-1): first the <= 4 eight-column chunks of the next
//     panel [k1, k1+w2) — each signals a global counter when done — then
//     the trailing blocks [k1+w2, N] (column N = right-hand side);
//   CTA 0: waits for the chunk counter, factors panel p+1 in shared memory.
//   one grid barrier.
// Panel widths adapt to the shrinking row count (wider panels later).
__global__ void __launch_bounds__(kThreads, 1) lu_fused_kernel(LuArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  __shared__ int s_piv[kMaxPanel];
  const int N = a.N;
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.info = 0;
  __syncthreads();
  unsigned long long t0 = 0, acc_upd = 0, acc_fac = 0, acc_sync = 0, acc_work = 0;
  int k0 = 0, w = 0;                                     // panel being applied
  int k1 = 0, w2 = N < panel_width(N) ? N : panel_width(N);  // panel being factored
  int pidx = -1, target = 0;
  const int workers = gridDim.x > 1 ? gridDim.x - 1 : 1;
  const int wid = gridDim.x > 1 ? (int)blockIdx.x - 1 : 0;
  while (w > 0 || w2 > 0) {
    if (a.prof && threadIdx.x == 0) t0 = gtimer();
    const int* mv = a.moves + ((pidx + 2) & 1) * kMoveStride;
    int* mv_next = a.moves + ((pidx + 3) & 1) * kMoveStride;
    const int nchunk = (w > 0 && w2 > 0) ? (w2 + kColBlock - 1) / kColBlock : 0;
    target += nchunk;
    if (blockIdx.x == 0 && w2 > 0) {
      if (nchunk > 0) {
        if (threadIdx.x == 0)
          while (atomicAdd(a.flag, 0) < target) __nanosleep(32);
        __syncthreads();
      }
      if (a.prof && threadIdx.x == 0) {
        const unsigned long long t1 = gtimer();
        acc_upd += t1 - t0;
        t0 = t1;
      }
      factor_panel(a, k1, w2, sm, s_piv, mv_next);
      if (a.prof && threadIdx.x == 0) {
        const unsigned long long t1 = gtimer();
        acc_fac += t1 - t0;
        t0 = t1;
      }
    }
    if (w > 0 && (gridDim.x == 1 || blockIdx.x > 0)) {
      const int rest0 = k1 + w2;
      const int ntrail = (N + 1 - rest0 + kColBlock - 1) / kColBlock;
      for (int blk = wid; blk < nchunk + ntrail; blk += workers) {
        int c0, c1;
        if (blk < nchunk) {
          c0 = k1 + blk * kColBlock;
          c1 = c0 + kColBlock < rest0 ? c0 + kColBlock : rest0;
        } else {
          c0 = rest0 + (blk - nchunk) * kColBlock;
          c1 = c0 + kColBlock < N + 1 ? c0 + kColBlock : N + 1;
        }
        update_cols<kColBlock>(a, k0, w, c0, c1, sm, mv);
        if (blk < nchunk && threadIdx.x == 0) {
          __threadfence();
          atomicAdd(a.flag, 1);
        }
      }
      if (a.prof && threadIdx.x == 0) {
        const unsigned long long t1 = gtimer();
        acc_work += t1 - t0;
        t0 = t1;
      }
    }
    grid.sync();
    if (a.prof && threadIdx.x == 0) acc_sync += gtimer() - t0;
    // advance: the factored panel becomes the applied one
    k0 = k1;
    w = w2;
    k1 = k0 + w;
    w2 = k1 < N ? (N - k1 < panel_width(N - k1) ? N - k1 : panel_width(N - k1)) : 0;
    ++pidx;
    if (w == 0) break;
  }
  if (a.prof && threadIdx.x == 0 && blockIdx.x < 2) {
    a.prof[blockIdx.x * 4 + 0] = acc_upd;
    a.prof[blockIdx.x * 4 + 1] = acc_fac;
    a.prof[blockIdx.x * 4 + 2] = acc_work;
    a.prof[blockIdx.x * 4 + 3] = acc_sync;
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
  int w = (int)((kPanelSmem - 8 * (size_t)N) / (sizeof(double) * (size_t)N));
  if (w > kMaxPanel) w = kMaxPanel;
  if (w < 1 || N > kRowsPerThread * kThreads) return false;  // multi-launch fallback
  int* moves = reinterpret_cast<int*>(allocator().alloc(kMoveStride + 1));
  int* flag = moves + 2 * kMoveStride;
  T2S2_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), stream()));
  static const bool prof = getenv("T2S2_LU_PROFILE") != nullptr;
  unsigned long long* pbuf = nullptr;
  if (prof) {
    pbuf = reinterpret_cast<unsigned long long*>(allocator().alloc(16));
    T2S2_CUDA(cudaMemsetAsync(pbuf, 0, 128, stream()));
  }
  LuArgs a{N, A, b, piv, info_dev, w, moves, flag, pbuf};
  void* params[] = {&a};
  {
    // algorithmic: 2/3 N^3 (factor) + 2 N^2 (solves); bytes: matrix read+write
    LaunchScope ls("lu_fused", 2.0 / 3.0 * (double)N * N * N + 2.0 * (double)N * N,
                   16.0 * (double)N * N);
    const int grid = sm_budget() > 0 && sm_budget() < g_num_sms ? sm_budget() : g_num_sms;
    T2S2_CUDA(cudaLaunchCooperativeKernel((void*)lu_fused_kernel, dim3(grid), dim3(kThreads),
                                          params, kPanelSmem, stream()));
  }
  allocator().release(reinterpret_cast<double*>(moves));
  if (prof) {
    unsigned long long h[16];
    T2S2_CUDA(cudaMemcpyAsync(h, pbuf, 128, cudaMemcpyDeviceToHost, stream()));
    T2S2_CUDA(cudaStreamSynchronize(stream()));
    fprintf(stderr, "lu N=%d w=%d cta0: upd %.1f fac %.1f sync %.1f us | cta1: work %.1f sync %.1f us\n",
            N, w, h[0] / 1e3, h[1] / 1e3, h[3] / 1e3, h[6] / 1e3, h[7] / 1e3);

    allocator().release(reinterpret_cast<double*>(pbuf));
  }
  return true;
}

}  // namespace t2s2
