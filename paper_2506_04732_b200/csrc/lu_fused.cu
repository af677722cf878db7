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
  unsigned long long* prof;  // optional phase timers (ns), null in the product
  int* swapped;  // optional: set to 1 when any row interchange was made
};

__device__ __forceinline__ void dmma_8x8x4_lu(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Column loop of the panel factorisation, run by the first nthr threads of
// the CTA (nthr a power of two, nthr * RPT >= rows: only warps that own rows
// take part, synchronised by named barrier 1).  Thread t owns rows
// t + k*nthr.  The panel is processed in register sub-panels of SUB columns:
// a sub-panel's values of the thread's rows live in registers, so a column
// step touches shared memory only to publish candidate pivot rows; one
// barrier per column.
//
// Pivot search: one 32-bit key per row, (|a| hi word >> 11) << 12 | (4095 -
// row): the magnitude to 2^-9 relative resolution, ties to the lowest row,
// so one REDUX per level finds it.  (Any row within 0.2% of the column
// maximum is an equally stable pivot: |multipliers| <= 1.002.)
//
// After a sub-panel, its pivot rows' U entries right of it are formed
// (unit-lower forward substitution from preloaded values) and one rank-SUB
// update is applied to the rest of the panel in shared memory.
__device__ __forceinline__ void bar_panel(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

struct PanelScratch {
  double pub[2][kThreads / 32][10];  // each warp's candidate row; [8] = 1/pivot
  double Lp[8][8];                   // multipliers of the sub-panel's pivot rows
  double Us[kMaxPanel][8];           // U rows right of the sub-panel
  unsigned rk[2][kThreads / 32];     // each warp's best key
};

__device__ __forceinline__ PanelScratch& panel_scratch() {
  __shared__ __align__(16) PanelScratch ps;
  return ps;
}

template <int RPT, int SUB>
__device__ __forceinline__ void factor_columns(int rows, int w, double* sm, int* s_piv, int nthr,
                                            unsigned long long* prof) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = nthr >> 5;
  const unsigned full = 0xffffffffu;
  PanelScratch& ps = panel_scratch();
  auto& rk = ps.rk;
  auto& pub = ps.pub;
  auto& Lp = ps.Lp;
  auto& Us = ps.Us;
  long long c0 = clock64(), c_steps = 0, c_sub = 0;
  int row[RPT];
  bool live[RPT];
  unsigned tag[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    row[k] = tid + k * nthr;
    live[k] = row[k] < rows;
    tag[k] = 4095u - (unsigned)row[k];
  }
  for (int j0 = 0; j0 < w; j0 += SUB) {
    const int nsub = w - j0 < SUB ? w - j0 : SUB;
    double a[RPT][SUB];
    int pv[SUB];
#pragma unroll
    for (int k = 0; k < RPT; ++k)
#pragma unroll
      for (int t = 0; t < SUB; ++t)
        a[k][t] = (row[k] < rows && t < nsub) ? sm[(j0 + t) * rows + row[k]] : 0.0;
#pragma unroll
    for (int t = 0; t < SUB; ++t) {
      pv[t] = 0;
      if (t >= nsub) break;
      const int buf = (j0 + t) & 1;
      unsigned key = 0u;
      int bk = 0;
#pragma unroll
      for (int k = 0; k < RPT; ++k)
        if (live[k]) {
          const unsigned kk = (((unsigned)__double2hiint(fabs(a[k][t])) >> 11) << 12) | tag[k];
          if (kk > key) {
            key = kk;
            bk = k;
          }
        }
      const unsigned wk = __reduce_max_sync(full, key);
      if (key == wk && key != 0u) {
        // the warp's winner publishes its row (multipliers left of t,
        // values from t on) and the reciprocal of its candidate pivot
        double* dst = pub[buf][warp];
#pragma unroll
        for (int q = 0; q < SUB; ++q) {
          double v = a[0][q];
#pragma unroll
          for (int k = 1; k < RPT; ++k)
            if (k == bk) v = a[k][q];
          dst[q] = v;
          if (q == t) dst[8] = v != 0.0 ? __drcp_rn(v) : 1.0;
        }
      }
      if (lane == 0) rk[buf][warp] = wk;
      bar_panel(nthr);
      const unsigned g = __reduce_max_sync(full, lane < nw ? rk[buf][lane] : 0u);
      const int p = 4095 - (int)(g & 4095u);
      pv[t] = p;
      const double* src = pub[buf][(p & (nthr - 1)) >> 5];
      double prow[SUB];
#pragma unroll
      for (int q = 0; q < SUB; ++q) prow[q] = q > t ? src[q] : 0.0;
      const double inv = src[8];
      if (tid < t) Lp[t][tid] = src[tid];
      if (tid == 0) s_piv[j0 + t] = p;
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        if (row[k] == p) live[k] = false;
        if (live[k]) {
          const double l = a[k][t] * inv;
          a[k][t] = l;
#pragma unroll
          for (int q = 0; q < SUB; ++q)
            if (q > t) a[k][q] = fma(-l, prow[q], a[k][q]);
        }
      }
    }
    if (prof) {
      const long long c1 = clock64();
      c_steps += c1 - c0;
      c0 = c1;
    }
    // sub-panel back to shared memory (pivot rows keep their U entries,
    // the others their multipliers)
#pragma unroll
    for (int k = 0; k < RPT; ++k)
#pragma unroll
      for (int t = 0; t < SUB; ++t)
        if (row[k] < rows && t < nsub) sm[(j0 + t) * rows + row[k]] = a[k][t];
    const int je = j0 + nsub;
    if (je < w) {
      bar_panel(nthr);
      // U entries of the sub-panel's pivot rows right of it (one thread per
      // column): u_t = a[p_t][c] - sum_{q<t} l[p_t][q] u_q
      for (int c = je + tid; c < w; c += nthr) {
        double x[SUB];
#pragma unroll
        for (int t = 0; t < SUB; ++t) x[t] = t < nsub ? sm[c * rows + pv[t]] : 0.0;
#pragma unroll
        for (int t = 1; t < SUB; ++t)
#pragma unroll
          for (int q = 0; q < t; ++q) x[t] = fma(-Lp[t][q], x[q], x[t]);
#pragma unroll
        for (int t = 0; t < SUB; ++t) {
          Us[c][t] = x[t];
          if (t < nsub) sm[c * rows + pv[t]] = x[t];
        }
      }
      bar_panel(nthr);
      // rank-nsub update of the live rows, columns je..w-1, two at a time
      int c = je;
      for (; c + 1 < w; c += 2) {
        double u0[SUB], u1[SUB], x0[RPT], x1[RPT];
#pragma unroll
        for (int t = 0; t < SUB; ++t) {
          u0[t] = Us[c][t];
          u1[t] = Us[c + 1][t];
        }
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          x0[k] = live[k] ? sm[c * rows + row[k]] : 0.0;
          x1[k] = live[k] ? sm[(c + 1) * rows + row[k]] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < RPT; ++k)
#pragma unroll
          for (int t = 0; t < SUB; ++t) {
            x0[k] = fma(-a[k][t], u0[t], x0[k]);
            x1[k] = fma(-a[k][t], u1[t], x1[k]);
          }
#pragma unroll
        for (int k = 0; k < RPT; ++k)
          if (live[k]) {
            sm[c * rows + row[k]] = x0[k];
            sm[(c + 1) * rows + row[k]] = x1[k];
          }
      }
      if (c < w) {
        double ut[SUB];
#pragma unroll
        for (int t = 0; t < SUB; ++t) ut[t] = Us[c][t];
#pragma unroll
        for (int k = 0; k < RPT; ++k)
          if (live[k]) {
            double x = sm[c * rows + row[k]];
#pragma unroll
            for (int t = 0; t < SUB; ++t) x = fma(-a[k][t], ut[t], x);
            sm[c * rows + row[k]] = x;
          }
      }
    }
    if (prof) {
      const long long c1 = clock64();
      c_sub += c1 - c0;
      c0 = c1;
    }
  }
  if (prof && threadIdx.x == 0) {
    prof[12] += c_steps;
    prof[13] += c_sub;
  }
}

// Smallest power-of-two thread count (>= one warp) giving each thread at
// most rpt rows.
__device__ __forceinline__ int panel_threads(int rows, int rpt) {
  int n = 32;
  while (n * rpt < rows) n <<= 1;
  return n;
}

// Panel configurations measured on B200 (tools/micro/fc2_bench.cu): one row
// per thread with as few warps as possible up to 512 rows, then SUB = 4 to
// keep the larger register row blocks spill-free.
__device__ __forceinline__ void factor_columns_any(int rows, int w, double* sm, int* s_piv,
                                                unsigned long long* prof) {
  const int tid = threadIdx.x;
  if (rows <= kThreads) {
    const int n = panel_threads(rows, 1);
    if (tid < n) factor_columns<1, 8>(rows, w, sm, s_piv, n, prof);
  } else if (rows <= 2 * kThreads) {
    factor_columns<2, 4>(rows, w, sm, s_piv, kThreads, prof);
  } else if (rows <= 3 * kThreads) {
    factor_columns<3, 4>(rows, w, sm, s_piv, kThreads, prof);
  } else if (rows <= 4 * kThreads) {
    factor_columns<4, 4>(rows, w, sm, s_piv, kThreads, prof);
  } else {
    factor_columns<5, 4>(rows, w, sm, s_piv, kThreads, prof);
  }
}

// Factor the panel A[k0:N, k0:k0+w] with partial pivoting inside one CTA,
// one barrier per column: rows never move while factoring (a chosen pivot
// row is flagged done and read in place), so each thread only touches its
// own rows.  Afterwards positions 0..w-1 take the pivot rows in order and
// each low row (physical index < w) that was not chosen takes the slot of a
// chosen pivot from below the panel top: any such bijection is a valid row
// permutation (the right-hand side rides along as column N, so no LAPACK
// ipiv sequence is needed) and one warp computes it with ballots.
__device__ __forceinline__ void factor_panel(const LuArgs& a, int k0, int w, double* sm, int* s_piv,
                                          int* mv) {
  const int N = a.N, rows = N - k0;
  const int tid = threadIdx.x, lane = tid & 31;
  unsigned long long tp = a.prof && tid == 0 ? gtimer() : 0;
#define T2S2_PHASE(slot)                                 \
  if (a.prof && tid == 0) {                              \
    const unsigned long long tq = gtimer();              \
    a.prof[8 + (slot)] += tq - tp;                       \
    tp = tq;                                             \
  }
  int* cur = reinterpret_cast<int*>(sm + (size_t)rows * w);  // position -> physical row
  {
    // every element of the panel in flight at once: asynchronous 8-byte
    // copies global -> shared (the panel is L2-resident)
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);
    int c = tid / rows, r = tid - c * rows;
    const int step_c = kThreads / rows, step_r = kThreads - step_c * rows;
    const double* col0 = a.A + (long long)k0 * N + k0;
    for (int e = tid; e < rows * w; e += kThreads) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sbase + 8u * (unsigned)e),
                   "l"(col0 + (long long)c * N + r)
                   : "memory");
      c += step_c;
      r += step_r;
      if (r >= rows) {
        r -= rows;
        ++c;
      }
    }
  }
  for (int r = tid; r < rows; r += kThreads) cur[r] = r;
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  T2S2_PHASE(0)
  factor_columns_any(rows, w, sm, s_piv, a.prof);
  __syncthreads();
  T2S2_PHASE(1)
  if (tid < 32) {
    const unsigned full = 0xffffffffu;
    const bool act = lane < w;
    const int p = act ? s_piv[lane] : 0;
    const unsigned wmask = w >= 32 ? full : ((1u << w) - 1u);
    const unsigned chosen_low = __reduce_or_sync(full, (act && p < w) ? (1u << p) : 0u);
    const unsigned free_low = ~chosen_low & wmask;  // low rows displaced by pivots
    const bool high = act && p >= w;
    const unsigned high_mask = __ballot_sync(full, high);
    const unsigned lt = (1u << lane) - 1u;
    const int k = __popc(high_mask & lt);
    const unsigned moved = __ballot_sync(full, act && p != lane);
    const int n1 = __popc(moved);
    if (act) {
      cur[lane] = p;
      a.piv[k0 + lane] = k0 + p;
    }
    if (act && p != lane) {
      const int m = __popc(moved & lt);
      mv[1 + 2 * m] = lane;
      mv[2 + 2 * m] = p;
    }
    if (high) {
      const int q = __fns(free_low, 0, k + 1);
      cur[p] = q;
      mv[1 + 2 * (n1 + k)] = p;
      mv[2 + 2 * (n1 + k)] = q;
    }
    if (lane == 0) {
      mv[0] = n1 + __popc(high_mask);
      if (mv[0] > 0 && a.swapped) *a.swapped = 1;
    }
    const unsigned zero = __ballot_sync(full, act && sm[lane * rows + p] == 0.0);
    if (lane == 0 && zero && *a.info == 0) *a.info = k0 + __ffs(zero);
  }
  __syncthreads();
  T2S2_PHASE(2)
  {
    int c = tid / rows, r = tid - c * rows;
    const int step_c = kThreads / rows, step_r = kThreads - step_c * rows;
    double* col0 = a.A + (long long)k0 * N + k0;
#pragma unroll 4
    for (int e = tid; e < rows * w; e += kThreads) {
      col0[(long long)c * N + r] = sm[c * rows + cur[r]];
      c += step_c;
      r += step_r;
      if (r >= rows) {
        r -= rows;
        ++c;
      }
    }
  }
  __syncthreads();
  T2S2_PHASE(3)
#undef T2S2_PHASE
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

// One next-panel column c brought up to date with panel [k0, k0+w): the
// critical path between two panel factorisations, so every input is loaded
// in one asynchronous batch into shared memory (the factored panel and the
// column), the row moves are applied there, the unit-lower TRSM runs in one
// warp and the rank-w update reads L21 from shared memory; the column is
// written back once.
__device__ __forceinline__ void update_next_col(const LuArgs& a, int k0, int w, int c, double* sm,
                                             const int* mv) {
  const int N = a.N, rows = N - k0;
  const int tid = threadIdx.x, lane = tid & 31;
  double* L = sm;                     // panel, positions k0.., ld = rows
  double* X = sm + (size_t)rows * w;  // column c, positions k0..
  {
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);
    int cc = tid / rows, r = tid - cc * rows;
    const int step_c = kThreads / rows, step_r = kThreads - step_c * rows;
    const double* col0 = a.A + (long long)k0 * N + k0;
    for (int e = tid; e < rows * w; e += kThreads) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sbase + 8u * (unsigned)e),
                   "l"(col0 + (long long)cc * N + r)
                   : "memory");
      cc += step_c;
      r += step_r;
      if (r >= rows) {
        r -= rows;
        ++cc;
      }
    }
    const double* xc = a.A + (long long)c * N + k0;
    const unsigned xbase = sbase + 8u * (unsigned)(rows * w);
    for (int e = tid; e < rows; e += kThreads)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(xbase + 8u * (unsigned)e),
                   "l"(xc + e)
                   : "memory");
  }
  const int m = __ldcg(mv);
  int dst = -1, src = 0;
  if (tid < m) {
    dst = __ldcg(mv + 1 + 2 * tid);
    src = __ldcg(mv + 2 + 2 * tid);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  double v = 0.0;
  if (dst >= 0) v = X[src];
  __syncthreads();
  if (dst >= 0) X[dst] = v;
  __syncthreads();
  if (tid < 32) {
    // U12 = L11^{-1} x[0:w]: lane i holds row i
    double xi = lane < w ? X[lane] : 0.0;
#pragma unroll 1
    for (int j = 0; j < w; ++j) {
      const double lij = lane < w ? L[j * rows + lane] : 0.0;
      const double xj = __shfl_sync(0xffffffffu, xi, j);
      if (lane > j) xi = fma(-lij, xj, xi);
    }
    if (lane < w) X[lane] = xi;
  }
  __syncthreads();
  double* out = a.A + (long long)c * N + k0;
  for (int i = tid; i < rows; i += kThreads) {
    double x = X[i];
    if (i >= w) {
#pragma unroll 4
      for (int j = 0; j < w; ++j) x = fma(-L[j * rows + i], X[j], x);
    }
    out[i] = x;
  }
  __threadfence();
  __syncthreads();
}

// U x = y by 32-row blocks from the bottom.  Warp 0 solves a diagonal block
// from registers (reciprocal pivots, one shuffle per row) and, while the
// whole CTA applies the solved block to the rows above (32 independent
// loads per row in flight), already loads the next diagonal block.
__device__ __forceinline__ void back_substitute(const LuArgs& a, double* x) {
  const int N = a.N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned full = 0xffffffffu;
  for (int i = tid; i < N; i += blockDim.x) x[i] = __ldcg(a.b + i);
  double u[32];
  auto load_diag = [&](int j0, int jb) {
#pragma unroll
    for (int c = 0; c < 32; ++c)
      u[c] = (lane < jb && c < jb) ? __ldcg(a.A + (long long)(j0 + c) * N + j0 + lane) : 0.0;
  };
  int j1 = N, j0 = N - 32 > 0 ? N - 32 : 0;
  if (warp == 0) load_diag(j0, j1 - j0);
  __syncthreads();
  while (j1 > 0) {
    const int jb = j1 - j0;
    if (warp == 0) {
      double d = 1.0;
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c == lane) d = u[c];
      const double rinv = lane < jb ? 1.0 / d : 0.0;
      double xi = lane < jb ? x[j0 + lane] : 0.0;
#pragma unroll
      for (int c = 31; c >= 0; --c) {
        if (c < jb) {
          const double v = __shfl_sync(full, xi * rinv, c);
          if (lane == c) xi = v;
          if (lane < c) xi = fma(-u[c], v, xi);
        }
      }
      if (lane < jb) x[j0 + lane] = xi;
    }
    __syncthreads();
    const int n1 = j0, n0 = j0 - 32 > 0 ? j0 - 32 : 0;
    if (warp == 0 && n1 > 0) load_diag(n0, n1 - n0);  // in flight during the update
    if (j0 > 0) {
      // jb == 32 here: only the top block can be partial
      for (int i = tid; i < j0; i += blockDim.x) {
        double acc = x[i];
#pragma unroll
        for (int h = 0; h < 32; h += 16) {
          double uu[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) uu[c] = __ldcg(a.A + (long long)(j0 + h + c) * N + i);
#pragma unroll
          for (int c = 0; c < 16; ++c) acc = fma(-uu[c], x[j0 + h + c], acc);
        }
        x[i] = acc;
      }
    }
    __syncthreads();
    j1 = n1;
    j0 = n0;
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
    // next-panel columns are on the critical path: one column per worker
    // when there are enough workers, so each one's update is short
    const int cw = workers >= 2 * w2 ? 1 : kColBlock;
    const int nchunk = (w > 0 && w2 > 0) ? (w2 + cw - 1) / cw : 0;
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
          c0 = k1 + blk * cw;
          c1 = c0 + cw < rest0 ? c0 + cw : rest0;
        } else {
          c0 = rest0 + (blk - nchunk) * kColBlock;
          c1 = c0 + kColBlock < N + 1 ? c0 + kColBlock : N + 1;
        }
        if (blk < nchunk && cw == 1) {
          update_next_col(a, k0, w, c0, sm, mv);
        } else {
          update_cols<kColBlock>(a, k0, w, c0, c1, sm, mv);
          if (blk < nchunk) __threadfence();
        }
        if (blk < nchunk) {
          __syncthreads();
          if (threadIdx.x == 0) atomicAdd(a.flag, 1);
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

}  // namespace

bool lu_solve_fused(int N, double* A, double* b, int* piv, int* info_dev, int* swapped) {
  max_dynamic_smem((const void*)lu_fused_kernel, (int)kPanelSmem);
  int w = (int)((kPanelSmem - 8 * (size_t)N) / (sizeof(double) * (size_t)N));
  if (w > kMaxPanel) w = kMaxPanel;
  if (w < 1 || N > kRowsPerThread * kThreads) return false;  // multi-launch fallback
  int* moves = reinterpret_cast<int*>(allocator().alloc(kMoveStride + 1));
  int* flag = moves + 2 * kMoveStride;
  T2S2_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), stream()));
  LuArgs a{N, A, b, piv, info_dev, w, moves, flag, nullptr, swapped};
  void* params[] = {&a};
  {
    // algorithmic: 2/3 N^3 (factor) + 2 N^2 (solves); bytes: matrix read+write
    LaunchScope ls("lu_fused", 2.0 / 3.0 * (double)N * N * N + 2.0 * (double)N * N,
                   16.0 * (double)N * N);
    const int grid = sm_budget() > 0 && sm_budget() < num_sms() ? sm_budget() : num_sms();
    T2S2_CUDA(cudaLaunchCooperativeKernel((void*)lu_fused_kernel, dim3(grid), dim3(kThreads),
                                          params, kPanelSmem, stream()));
  }
  allocator().release(reinterpret_cast<double*>(moves));
  return true;
}

}  // namespace t2s2
