// Verified no-pivot dense solve of a local system by blocked Gauss-Jordan
// elimination in ONE cooperative launch, one grid barrier per 32-column
// panel and no back-substitution chain.
//
// The local systems of an implicit step (I + dt L projected on orthonormal
// interface bases, tt_solver.py:350-362 solves them with numpy.linalg.solve)
// are well conditioned and their diagonal pivots are large.  Every
// multiplier is checked against kPivThresh (below, threshold partial
// pivoting: no interchange while |l| <= 8); if one exceeds it, or a pivot is
// zero, the kernel declines (*info = -1) and the caller runs the
// partial-pivoting kernel.
//
// Panel p (rows/columns [k0, k1), k1 = k0 + 32), normalised block
// Gauss-Jordan:
//   CTA 0 (previous phase) factored the diagonal block D_p = L U (in
//   groups of four steps: U, L^{-1} and U^{-1} together, multipliers
//   checked, see gj_diag) and published D^{-1} = U^{-1} L^{-1} and U^{-1}
//   (32 x 32 each).
//   Every other row block I (above AND below the panel) is a tile task
//   together with a column block J of [k1, N] (column N = right-hand side):
//       W_J = D^{-1} A[p, J]            (the panel rows, normalised)
//       A[I, J] -= A[I, p] W_J          (FP64 tensor core, DMMA m8n8k4)
//   and, once per row block below the panel, the multipliers
//   A[I, p] U^{-1} are formed and checked (|l| <= kPivThresh).  A CTA walks a
//   contiguous J-major chunk of tasks, so W_J is formed once per CTA and
//   column block, and the next task's global loads are in flight (in
//   registers) while the current one computes; operand staging is double
//   buffered, one CTA barrier per task.  The tile of row block 0
//   stores W_J to a double-buffered 32 x (N+1) row panel, which the next
//   phase reads as those rows' current values.
//   CTA 0 updates the next diagonal block (special_tile: 32 x 32 products
//   on all warps) and factors it while the other CTAs work (lookahead).
//   No grid-wide barrier: the tile CTAs wait for an arrival count (every
//   CTA of the previous phases, CTA 0 after publishing the next D^{-1}),
//   CTA 0 waits only for the three tile tasks that produce its next
//   diagonal block; the row panels are triple buffered so CTA 0 may run
//   one phase ahead.
// After the last panel every diagonal block is the identity: b holds x.
//
// Algorithmic cost N^3 (vs 2/3 N^3 + back substitution for LU): on this
// latency-bound size range (N <= 2000, <= 63 panels) the extra tiles fill
// otherwise idle SMs and the sequential back-substitution disappears.
#include <cooperative_groups.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "linalg.h"

namespace cg = cooperative_groups;

namespace t2s2 {
namespace {

constexpr int kThr = 256;      // 8 warps
constexpr int kP = 32;         // panel width
constexpr int kT = 64;         // tile rows / columns
constexpr int kLdT = kT + 4;   // smem stride of 64-long columns
constexpr int kLdP = kP + 4;   // smem stride of 32-long columns
constexpr int kInv = 2 * kP * kP;  // per panel: D^{-1} then U^{-1}, column-major
// Multiplier bound: threshold partial pivoting.  Elimination proceeds without
// an interchange while every multiplier satisfies |l| <= kPivThresh (the
// bound sparse LU codes use with u = 1 / kPivThresh); kPivThresh = 1 would be
// exactly "GEPP makes no interchange".  Where GEPP does interchange on the
// local systems of configs 2 and 3, the multipliers are <= 4 (measured), so
// 8 accepts those solves here instead of sending ~3% of them to the pivoting
// kernel at 3-4x the cost; a larger multiplier or a zero pivot still
// declines.  Every candidate is scored by the solver afterwards
// (tt_solver.py:383-399: a local solution that does not lower the residual
// functional is discarded), and the full-length parity runs against ttss hold
// with it: config 2 max 2.9e-10 (GEPP-equivalent bound: 3.3e-10), config 3
// 1.4e-10 (2.0e-10), identical ranks at every step, 125 / 202 sweeps against
// the reference's 132 / 200 (profiles/r02i_parity_full_*.json).
constexpr double kPivThresh = 8.0;

struct GjArgs {
  int N;
  double* A;      // column-major N x N (clobbered)
  double* b;      // right-hand side (column N), overwritten with x
  double* inv;    // npan * kInv
  double* wbuf;   // 3 x (kP x (N+1)), column-major ld kP (phase p: buffer p % 3)
  int* info;      // 0, or -1: a multiplier exceeded 1 / zero pivot
  unsigned* sync; // [0] tile-worker arrivals, [1] diagonal blocks published by CTA 0,
                  // [2 + p] finished feeder tasks of phase p (zeroed by the host)
  unsigned long long* prof;
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void gj_fail(const GjArgs& a) { atomicExch(a.info, -1); }

// named CTA barriers (id 0 is __syncthreads)
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Phase hand-off without a grid-wide barrier, two counters: the tile workers
// add one arrival per phase after their tile tasks, CTA 0 counts the diagonal
// blocks it has published.  A tile worker starts phase p once every worker
// has finished phase p - 1 AND D_p^{-1} is published; CTA 0 waits only for
// the tile tasks that produce its next diagonal block.  (One shared counter
// is not enough: CTA 0 runs a phase ahead, and its early arrival would stand
// in for a tile worker that has not finished — the other workers would start
// on rows and columns that are still being updated.)  Release: the
// CTA's stores, a CTA barrier, one thread's fence and atomic; acquire: one
// thread's ld.acquire spin, then a CTA barrier (loads use ld.global.cg).
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void cta_signal(unsigned* p) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p, 1u);
  }
}
// wait until *p >= target (or, abortable, until *info != 0)
__device__ __forceinline__ void cta_wait(const unsigned* p, unsigned target, const int* info,
                                         bool abortable) {
  if (threadIdx.x == 0)
    while (ld_acquire_u32(p) < target)
      if (abortable && *(volatile const int*)info != 0) break;
  __syncthreads();
}
// The same wait for CTA 0, returning *info as thread 0 saw it: the flag is
// loaded next to the counter (before the acquire load in program order, so
// both are in flight together) instead of in a round trip of its own after
// the wait.  A flag raised after that load is seen one phase later — it only
// skips work, the hand-offs do not depend on it.
__device__ __forceinline__ int cta_wait_info(const unsigned* p, unsigned target, const int* info) {
  __shared__ int seen;
  if (threadIdx.x == 0) {
    int f;
    do {
      f = *(volatile const int*)info;
    } while (ld_acquire_u32(p) < target && f == 0);
    seen = f;
  }
  __syncthreads();
  return seen;
}

// Geometry of one phase.
struct Phase {
  int N, p, k0, kb, k1;  // panel rows/cols [k0, k1)
  int kb2;            // width of the next diagonal block (0 on the last panel)
  int nbelow, nabove, nrb;  // row blocks: [next diag (kb2 rows)], 64-row blocks below, 64-row blocks above
  int ncb;            // column blocks of [k1, N]: [next diag (kb2)], 64-wide blocks
  int kprev;          // first row of the previous panel (rows read from wbuf), -1 if p == 0
  __device__ Phase(int N_, int p_) : N(N_), p(p_) {
    k0 = p * kP;
    kb = N - k0 < kP ? N - k0 : kP;
    k1 = k0 + kb;
    kb2 = N - k1 < kP ? N - k1 : kP;
    const int rest = N - k1 - kb2;  // rows below the next diagonal block
    nbelow = (kb2 > 0 ? 1 : 0) + (rest + kT - 1) / kT;
    nabove = (k0 + kT - 1) / kT;
    nrb = nbelow + nabove;
    const int crest = N + 1 - k1 - kb2;  // columns after the next diagonal block (incl. rhs)
    ncb = (kb2 > 0 ? 1 : 0) + (crest + kT - 1) / kT;
    kprev = p > 0 ? k0 - kP : -1;
  }
  __device__ void rows(int I, int& r, int& m) const {
    if (I < nbelow) {
      if (kb2 > 0 && I == 0) {
        r = k1;
        m = kb2;
        return;
      }
      r = k1 + kb2 + (kb2 > 0 ? I - 1 : I) * kT;
      m = N - r < kT ? N - r : kT;
    } else {
      r = (I - nbelow) * kT;
      m = k0 - r < kT ? k0 - r : kT;
    }
  }
  __device__ void cols(int J, int N, int& c, int& n) const {
    if (kb2 > 0 && J == 0) {
      c = k1;
      n = kb2;
      return;
    }
    const int j = kb2 > 0 ? J - 1 : J;
    c = k1 + kb2 + j * kT;
    n = N + 1 - c < kT ? N + 1 - c : kT;
  }
};

// Current value of the augmented matrix entry (r, c), c <= N: rows of the
// previous panel live in the row-panel buffer of the previous phase.
__device__ __forceinline__ const double* src_ptr(const GjArgs& a, const Phase& ph, int r, int c) {
  if (ph.kprev >= 0 && r >= ph.kprev && r < ph.k0)
    return a.wbuf + (size_t)((ph.p - 1) % 3) * kP * (a.N + 1) + (size_t)c * kP + (r - ph.kprev);
  return c < a.N ? a.A + (size_t)c * a.N + r : a.b + r;
}
__device__ __forceinline__ double* dst_ptr(const GjArgs& a, int r, int c) {
  return c < a.N ? a.A + (size_t)c * a.N + r : a.b + r;
}

struct Smem {
  double di[kP * kLdP];   // D^{-1}: A operand, [k*kLdP + m]
  double ui[kP * kLdP];   // U^{-1}: B operand, [n*kLdP + k]
  double ab2[2][kP * kLdT];  // A[I, p] (m x kb): A operand [k*kLdT + m], double buffered
  double pb[kT * kLdP];   // A[p, J] (kb x n): B operand [n*kLdP + k]
  double ws[kT * kLdP];   // W = D^{-1} A[p, J] (32 x n): B operand [n*kLdP + k]
  double dg[kP * 33];     // diagonal block being factored, [c*33 + r]
  double za[kP * kLdP], xb[kP * kLdP];  // U^{-1}, L^{-1} as DMMA operands (gj_diag)
  double gl[kP / 4][4][kP], gy[kP / 4][4][kP];  // gj_diag: each group's l and y columns
};

// Load D^{-1}, U^{-1} of panel p into shared memory.  All global loads are
// issued into registers before the first shared-memory store: a load followed
// by its store is one exposed L2 round trip per element otherwise (the
// compiler does not move the loads across the stores).
struct InvRegs {
  double d[kP * kP / kThr], u[kP * kP / kThr];
};
__device__ __forceinline__ void load_inv_issue(const GjArgs& a, int p, InvRegs& R) {
  const double* g = a.inv + (size_t)p * kInv;
#pragma unroll
  for (int q = 0; q < kP * kP / kThr; ++q) {
    const int e = threadIdx.x + q * kThr;
    R.d[q] = __ldcg(g + e);
    R.u[q] = __ldcg(g + kP * kP + e);
  }
}
__device__ __forceinline__ void load_inv_store(const InvRegs& R, Smem& s) {
#pragma unroll
  for (int q = 0; q < kP * kP / kThr; ++q) {
    const int e = threadIdx.x + q * kThr, c = e >> 5, r = e & 31;
    s.di[c * kLdP + r] = R.d[q];  // Dinv[r][c] -> A op [k=c][m=r]
    s.ui[c * kLdP + r] = R.u[q];  // Uinv[r][c] -> B op [n=c][k=r]
  }
}
__device__ void load_inv(const GjArgs& a, int p, Smem& s) {
  InvRegs R;
  load_inv_issue(a, p, R);
  load_inv_store(R, s);
}

// One tile task of a phase: rows [r, r+m) x columns [c, c+n) of the
// augmented matrix (column N = right-hand side).
struct Task {
  int I, J, r, m, c, n;
};
__device__ __forceinline__ Task task_of(const Phase& ph, int t) {
  Task k;
  k.J = t / ph.nrb;
  k.I = t - k.J * ph.nrb;
  ph.rows(k.I, k.r, k.m);
  ph.cols(k.J, ph.N, k.c, k.n);
  return k;
}

// The global loads of one task, held in registers while the previous task
// computes: A[I, p] (8 per thread), A[p, J] (8 per thread, only for a new
// column block) and this lane's C fragments (warp tile 32 x 16).
struct TileRegs {
  double ab[8], pb[8], cv[4][2][2];
};

// Source of row r of the augmented matrix: element (r, c) at
// base + c * stride, except column N of a matrix row, which is b[r].  The
// previous panel's rows live in its row-panel buffer (stride kP).
struct RowSrc {
  const double* base;
  int stride;
  bool buf;
};
__device__ __forceinline__ RowSrc row_src(const GjArgs& a, const Phase& ph, int r) {
  if (ph.kprev >= 0 && r >= ph.kprev && r < ph.k0)
    return {a.wbuf + (size_t)((ph.p - 1) % 3) * kP * (a.N + 1) + (r - ph.kprev), kP, true};
  return {a.A + r, a.N, false};
}
__device__ __forceinline__ const double* elem(const GjArgs& a, const RowSrc& rs, int r, int c) {
  return (c == a.N && !rs.buf) ? a.b + r : rs.base + (size_t)c * rs.stride;
}

// A full 64 x 64 tile of matrix columns whose rows are not in the previous
// panel's row buffer, under a full panel: every address is tile origin +
// per-thread constant (+ a multiple of N), no predicates — the path of almost
// every task of a large system (the general path spends ~19 instructions of
// address arithmetic, predicates and reconvergence per DMMA,
// profiles/r02i_gj_sizes.ncu-rep).
__device__ __forceinline__ bool task_interior(const GjArgs& a, const Phase& ph, const Task& k) {
  return k.m == kT && k.n == kT && k.c + kT <= a.N && ph.kb == kP &&
         (ph.kprev < 0 || k.r >= ph.k0 || k.r + kT <= ph.kprev);
}

__device__ __forceinline__ void tile_load(const GjArgs& a, const Phase& ph, const Task& k, bool want_p,
                                          TileRegs& R) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp >> 2) * 32, wn0 = (warp & 3) * 16;
  if (!want_p && task_interior(a, ph, k)) {
    const int N = a.N;
    const double* ct = a.A + (size_t)k.c * N + k.r + (wn0 + (lane & 3) * 2) * N + wm0 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double* pc = ct + (j * 8 + h) * N;
#pragma unroll
        for (int i = 0; i < 4; ++i) R.cv[i][j][h] = __ldcg(pc + i * 8);
      }
    const double* ap = a.A + (size_t)ph.k0 * N + k.r + (tid >> 6) * N + (tid & 63);
#pragma unroll
    for (int q = 0; q < 8; ++q) R.ab[q] = __ldcg(ap + q * 4 * N);
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = wm0 + i * 8 + (lane >> 2);
    const RowSrc rs = row_src(a, ph, k.r + rr);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = wn0 + j * 8 + (lane & 3) * 2 + h;
        R.cv[i][j][h] = (rr < k.m && cc < k.n) ? __ldcg(elem(a, rs, k.r + rr, k.c + cc)) : 0.0;
      }
  }
  {
    const int i = tid & 63, kk0 = tid >> 6;  // row i, columns k0 + kk0 + 4q
    const RowSrc rs = row_src(a, ph, k.r + i);
    const bool rowok = i < k.m;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int kk = kk0 + 4 * q;
      R.ab[q] = (rowok && kk < ph.kb) ? __ldcg(rs.base + (size_t)(ph.k0 + kk) * rs.stride) : 0.0;
    }
  }
  if (want_p) {
    const int kk = tid & 31, j0 = tid >> 5;  // panel row k0 + kk, columns c + j0 + 8q
    const bool rowok = kk < ph.kb;
    const double* rowp = a.A + ph.k0 + kk;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = j0 + 8 * q, c = k.c + j;
      R.pb[q] = (rowok && j < k.n) ? __ldcg(c == a.N ? a.b + ph.k0 + kk : rowp + (size_t)c * a.N) : 0.0;
    }
  }
}

__device__ __forceinline__ void tile_stage(const TileRegs& R, bool want_p, Smem& s, int buf) {
  const int tid = threadIdx.x;
  double* ab = s.ab2[buf];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int e = tid + q * kThr;
    ab[(e >> 6) * kLdT + (e & 63)] = R.ab[q];
  }
  if (want_p) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = tid + q * kThr;
      s.pb[(e >> 5) * kLdP + (e & 31)] = R.pb[q];
    }
  }
}

// Compute one staged task (operands in s.ab / s.pb, C fragments in cv):
//   want_w : W = D^{-1} A[p, J] for a new column block (store_w: publish it
//            as the panel rows' new values),
//   check  : the multipliers A[I, p] U^{-1} of rows below the panel,
//   C -= A[I, p] W  -> global memory, or s.dg for the next diagonal block.
__device__ void tile_compute(const GjArgs& a, const Phase& ph, const Task& k, const double (&cv)[4][2][2],
                             bool want_w, bool store_w, bool check, bool to_diag, Smem& s, int buf) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* ab = s.ab2[buf];
  if (want_w) {
    const int wr0 = (warp >> 2) * 16, wc0 = (warp & 3) * 16;
    double acc[2][2][2] = {};
#pragma unroll
    for (int kk = 0; kk < kP; kk += 4) {
      const int kr = kk + (lane & 3);
      double af[2], bf[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = s.di[kr * kLdP + wr0 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = s.pb[(wc0 + j * 8 + (lane >> 2)) * kLdP + kr];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    double* wdst = a.wbuf + (size_t)(ph.p % 3) * kP * (a.N + 1);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kr = wr0 + i * 8 + (lane >> 2), cc = wc0 + j * 8 + (lane & 3) * 2 + h;
          s.ws[cc * kLdP + kr] = acc[i][j][h];
          if (store_w && kr < ph.kb && cc < k.n) wdst[(size_t)(k.c + cc) * kP + kr] = acc[i][j][h];
        }
  }
  if (check) {
    const int mm0 = (warp >> 1) * 16, mn0 = (warp & 1) * 16;
    double acc[2][2][2] = {};
#pragma unroll
    for (int kk = 0; kk < kP; kk += 4) {
      const int kr = kk + (lane & 3);
      double af[2], bf[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = ab[kr * kLdT + mm0 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = s.ui[(mn0 + j * 8 + (lane >> 2)) * kLdP + kr];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (mm0 + i * 8 + (lane >> 2) < k.m && !(fabs(acc[i][j][h]) <= kPivThresh)) bad = true;
    if (bad) gj_fail(a);
  }
  if (want_w || check) __syncthreads();  // W visible, s.pb free
  const int wm0 = (warp >> 2) * 32, wn0 = (warp & 3) * 16;
  if (wm0 < k.m && wn0 < k.n) {
    double acc[4][2][2] = {};
#pragma unroll
    for (int kk = 0; kk < kP; kk += 4) {
      const int kr = kk + (lane & 3);
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = ab[kr * kLdT + wm0 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = s.ws[(wn0 + j * 8 + (lane >> 2)) * kLdP + kr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (!to_diag && task_interior(a, ph, k)) {
      const int N = a.N;
      double* ct = a.A + (size_t)k.c * N + k.r + (wn0 + (lane & 3) * 2) * N + wm0 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double* pc = ct + (j * 8 + h) * N;
#pragma unroll
          for (int i = 0; i < 4; ++i) pc[i * 8] = cv[i][j][h] - acc[i][j][h];
        }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int rr = wm0 + i * 8 + (lane >> 2), cc = wn0 + j * 8 + (lane & 3) * 2 + h;
            if (rr < k.m && cc < k.n) {
              const double v = cv[i][j][h] - acc[i][j][h];
              if (to_diag)
                s.dg[cc * 33 + rr] = v;
              else
                *dst_ptr(a, k.r + rr, k.c + cc) = v;
            }
          }
    }
  }
  // no closing barrier: the next task stages into the other s.ab2 buffer,
  // and s.pb / s.ws are rewritten only after the next staging barrier, which
  // every warp reaches after its C stage here
}

// The next diagonal block (rows and columns [k1, k1 + kb2), kb2 <= 32) on
// CTA 0 — the head of every panel's critical path — as 32 x 32 products on
// all eight warps (warp tile 8 x 16) instead of a 64 x 64 tile task:
//   W = D^{-1} A[p, J0] (published to the row panel) and
//   A[I0, J0] - A[I0, p] W left in s.dg.  One SM's DMMA rate bounds these
//   products (~3.7 cycles per m8n8k4), so nothing else is computed here.
#ifdef GJ_TIMELINE
__device__ unsigned long long g_sp_acc[8];
__device__ long long g_sp_last;
#define GJ_SP(k)                                            \
  if (threadIdx.x == 0) {                                   \
    const long long t_ = clock64();                         \
    if ((k) > 0) g_sp_acc[k] += (unsigned long long)(t_ - g_sp_last); \
    g_sp_last = t_;                                         \
  }
#else
#define GJ_SP(k)
#endif
__device__ void special_tile(const GjArgs& a, const Phase& ph, Smem& s, bool inv_resident) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = ph.k1, m = ph.kb2, k0 = ph.k0, kb = ph.kb, N = a.N;
  const int m0 = (warp >> 1) * 8, n0 = (warp & 1) * 16;
  // The three blocks lie in A itself (rows >= k1 are never in the previous
  // panel's row buffer; columns < N): one base pointer each, 32-bit offsets
  // (N <= 8192).
  const double* Ad = a.A + (size_t)r * N + r;    // A[I0, J0](rr, cc) = Ad[cc N + rr]
  const double* Aip = a.A + (size_t)k0 * N + r;  // A[I0, p](i, kk)   = Aip[kk N + i]
  const double* Apj = a.A + (size_t)r * N + k0;  // A[p, J0](k, j)    = Apj[j N + k]
  double cv[2][2];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rr = m0 + (lane >> 2), cc = n0 + j * 8 + (lane & 3) * 2 + h;
      cv[j][h] = (rr < m && cc < m) ? __ldcg(Ad + cc * N + rr) : 0.0;
    }
  // every global load in flight before the first shared-memory store
  double ra[4], rp[4], rd[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = tid + q * kThr, hi = e >> 5, lo = e & 31;
    ra[q] = (lo < m && hi < kb) ? __ldcg(Aip + hi * N + lo) : 0.0;  // A[I0, p](i = lo, kk = hi)
    rp[q] = (lo < kb && hi < m) ? __ldcg(Apj + hi * N + lo) : 0.0;  // A[p, J0](k = lo, j = hi)
  }
  if (!inv_resident) {  // D^{-1} of this panel (CTA 0 keeps its own copy in s.di: gj_diag)
    const double* g = a.inv + (size_t)ph.p * kInv;
#pragma unroll
    for (int q = 0; q < 4; ++q) rd[q] = __ldcg(g + tid + q * kThr);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = tid + q * kThr, hi = e >> 5, lo = e & 31;
    s.ab2[0][hi * kLdT + lo] = ra[q];
    s.pb[hi * kLdP + lo] = rp[q];
    if (!inv_resident) s.di[hi * kLdP + lo] = rd[q];
  }
  GJ_SP(2)
  __syncthreads();
  GJ_SP(3)
  {
    // (the multipliers A[I0, p] U^{-1} of these rows are checked off the
    // critical path, by the tile task of the same row block and the next
    // column block)
    double aw[2][2] = {};
#pragma unroll
    for (int kk = 0; kk < kP; kk += 4) {
      const int kr = kk + (lane & 3);
      const double fw = s.di[kr * kLdP + m0 + (lane >> 2)];  // D^{-1}[row][kr]
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma(aw[j][0], aw[j][1], fw, s.pb[(n0 + j * 8 + (lane >> 2)) * kLdP + kr]);
    }
    double* wdst = a.wbuf + (size_t)(ph.p % 3) * kP * (a.N + 1);
    GJ_SP(6)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = m0 + (lane >> 2), cc = n0 + j * 8 + (lane & 3) * 2 + h;
        s.ws[cc * kLdP + rr] = aw[j][h];
        if (rr < kb && cc < m) wdst[(size_t)(r + cc) * kP + rr] = aw[j][h];
      }
  }
  __syncthreads();
  GJ_SP(4)
  {
    double acc[2][2] = {};
#pragma unroll
    for (int kk = 0; kk < kP; kk += 4) {
      const int kr = kk + (lane & 3);
      const double f = s.ab2[0][kr * kLdT + m0 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j)
        dmma(acc[j][0], acc[j][1], f, s.ws[(n0 + j * 8 + (lane >> 2)) * kLdP + kr]);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = m0 + (lane >> 2), cc = n0 + j * 8 + (lane & 3) * 2 + h;
        if (rr < m && cc < m) s.dg[cc * 33 + rr] = cv[j][h] - acc[j][h];
      }
  }
}

// Factor the kb x kb block in s.dg (no interchanges, multipliers checked)
// and publish D^{-1} and U^{-1} (zero padded to 32 x 32) for panel p.
//
// Right-looking elimination in groups of four steps.  Thread (row i = lane,
// column group g = warp) keeps four columns of three matrices in registers:
//   D  the block being eliminated (U in the upper triangle at the end),
//   X  L^{-1}: forward elimination of [L | I] rides along (row st of X is
//      final when st becomes the pivot row),
//   Z  U^{-1} column by column: Y[:, st] = Z[:, st] / u_stst as soon as
//      row st of U is final, then Z[:, j>st] -= Y[:, st] U[st, j].
// Group g (steps 4g..4g+3) is warp g's own columns: that warp factors it
// alone — pivot rows and the pivot by shuffles, registers only — and
// publishes the group's four multiplier columns and four Y columns.  The
// next owner (warp g + 1) takes each step through a two-warp named barrier
// as soon as it is published, so it starts its own group right after the
// last one; every other warp waits at one named barrier per group and
// applies the four steps as shuffle mini-steps (the pivot rows are in lane
// st of the same warp).  Measured (tools/micro/gj_bench.cu): one CTA
// barrier per step 24.6k cycles, per group 14.1k, with the pipelined
// next-owner hand-off 10.5k (a shared-memory round trip through a CTA
// barrier costs ~200 cycles on B200).
// Rolled over the groups: this runs once per panel between tile phases and
// must stay small in the instruction cache.  Then D^{-1} = U^{-1} L^{-1} by
// DMMA.
#ifdef GJ_MICRO
__device__ long long g_diag_t[8];
#define GJ_T(k) if (threadIdx.x == 0) g_diag_t[k] = clock64();
#else
#define GJ_T(k)
#endif

__device__ void gj_diag(const GjArgs& a, int p, int kb, Smem& s) {
  const int tid = threadIdx.x, i = tid & 31, g = tid >> 5, j0 = 4 * g;
  __syncthreads();
  GJ_T(0)
  double dv[4], xv[4], zv[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = j0 + q;
    dv[q] = (i < kb && j < kb) ? s.dg[j * 33 + i] : (i == j ? 1.0 : 0.0);
    xv[q] = i == j ? 1.0 : 0.0;
    zv[q] = xv[q];
  }
  bool ok = true;
  // Four steps per group, group g = steps 4g..4g+3 = the columns of warp g.
  // The owner warp factors its group alone (pivot row and column by
  // shuffles, registers only) and publishes the four multiplier columns
  // l and the four U^{-1} columns y; after ONE barrier every other warp
  // applies the group to its own columns as four shuffle mini-steps
  // (pivot rows from lane st of the same warp).
  // Hand-offs by named barriers: the owner of group g hands each step's
  // columns to the owner of group g + 1 through a two-warp barrier (ids
  // 3..10), which applies it at once and starts its own group as soon as
  // group g is complete; every other warp waits at the group barrier (ids
  // 1, 2: all warps but the next owner) and applies the four steps then.
#pragma unroll 1
  for (int grp = 0; grp < kP / 4; ++grp) {
    // one buffer per group: the next owner moves on to produce group g + 2
    // while other warps may still read group g
    const int st0 = 4 * grp, par = grp & 1, buf = grp;
    const bool has_next = grp + 1 < kP / 4;
    const int gbar = 1 + par, gcount = has_next ? kThr - 32 : kThr;
    const int pbar0 = 3 + 4 * par;
    if (g == grp) {
#pragma unroll
      for (int sidx = 0; sidx < 4; ++sidx) {
        const int st = st0 + sidx;
        const double piv = __shfl_sync(0xffffffffu, dv[sidx], st);
        const double rinv = 1.0 / piv;
        ok = ok && fabs(piv) > 0.0 && isfinite(piv);
        const double l = i > st ? dv[sidx] * rinv : 0.0;   // multiplier l_{i,st}
        const double y = i <= st ? zv[sidx] * rinv : 0.0;  // (U^{-1})_{i,st}
        ok = ok && fabs(l) <= kPivThresh;
        s.gl[buf][sidx][i] = l;
        s.gy[buf][sidx][i] = y;
        if (has_next) named_arrive(pbar0 + sidx, 64);
        if (i <= st) zv[sidx] = y;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q > sidx) {  // columns ahead inside the group: D and Z
            const double u = __shfl_sync(0xffffffffu, dv[q], st);
            dv[q] = fma(-l, u, dv[q]);
            zv[q] = fma(-y, u, zv[q]);
          } else {  // columns j <= st: X
            const double xr = __shfl_sync(0xffffffffu, xv[q], st);
            xv[q] = fma(-l, xr, xv[q]);
          }
        }
      }
      named_arrive(gbar, gcount);
    } else if (g == grp + 1) {
      // next owner: each step as soon as it is published
#pragma unroll
      for (int sidx = 0; sidx < 4; ++sidx) {
        const int st = st0 + sidx;
        named_sync(pbar0 + sidx, 64);
        const double l = s.gl[buf][sidx][i], y = s.gy[buf][sidx][i];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double u = __shfl_sync(0xffffffffu, dv[q], st);
          dv[q] = fma(-l, u, dv[q]);
          zv[q] = fma(-y, u, zv[q]);
        }
      }
    } else {
      named_sync(gbar, gcount);
#pragma unroll
      for (int sidx = 0; sidx < 4; ++sidx) {
        const int st = st0 + sidx;
        const double l = s.gl[buf][sidx][i], y = s.gy[buf][sidx][i];
        if (g > grp) {  // columns ahead: D and Z
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double u = __shfl_sync(0xffffffffu, dv[q], st);
            dv[q] = fma(-l, u, dv[q]);
            zv[q] = fma(-y, u, zv[q]);
          }
        } else {  // columns behind: X
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double xr = __shfl_sync(0xffffffffu, xv[q], st);
            xv[q] = fma(-l, xr, xv[q]);
          }
        }
      }
    }
  }
  __syncthreads();
  GJ_T(1)
  if (!ok) gj_fail(a);
  // D^{-1} = U^{-1} L^{-1} (DMMA, 32 x 32 x 32); publish D^{-1} and U^{-1}
  // zero padded outside kb x kb
  double* gl = a.inv + (size_t)p * kInv;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = j0 + q;
    s.za[j * kLdP + i] = zv[q];  // A operand [k][m] = Z[m][k]
    s.xb[j * kLdP + i] = xv[q];  // B operand [n][k] = X[k][n]
    gl[kP * kP + j * kP + i] = (i < kb && j < kb) ? zv[q] : 0.0;
  }
  __syncthreads();
  GJ_T(2)
  {
    const int lane = i, warp = g, m0 = (warp >> 1) * 8, n0 = (warp & 1) * 16;
    double acc[2][2] = {};
#pragma unroll
    for (int kk = 0; kk < kP; kk += 4) {
      const int kr = kk + (lane & 3);
      const double af = s.za[kr * kLdP + m0 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j)
        dmma(acc[j][0], acc[j][1], af, s.xb[(n0 + j * 8 + (lane >> 2)) * kLdP + kr]);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = m0 + (lane >> 2), cc = n0 + j * 8 + (lane & 3) * 2 + h;
        const double v = (rr < kb && cc < kb) ? acc[j][h] : 0.0;
        gl[cc * kP + rr] = v;
        s.di[cc * kLdP + rr] = v;  // CTA 0's own copy for its next special tile
      }
  }
  GJ_T(3)
  __syncthreads();  // (the grid barrier that follows publishes the stores)
}

__global__ void __launch_bounds__(kThr, 1) gj_kernel(GjArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem& s = *reinterpret_cast<Smem*>(smraw);
  const int N = a.N, G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int npan = (N + kP - 1) / kP;
  const bool pr = a.prof && cta < 2 && tid == 0;
  unsigned long long tp = pr ? gtimer() : 0;
#define GJ_PHASE(slot)                         \
  if (pr) {                                    \
    const unsigned long long tq = gtimer();    \
    a.prof[cta * 4 + (slot)] += tq - tp;       \
    tp = tq;                                   \
  }
#ifdef GJ_TIMELINE
  // development timeline (tools/micro/gj_timeline.cu): globaltimer stamps of a few CTAs per phase
  const int tl_slot = cta == 0 ? 0 : cta == 1 ? 1 : cta == 5 ? 2 : cta == G / 2 ? 3 : cta == G - 1 ? 4 : -1;
#define GJ_TL(k) \
  if (a.prof && tid == 0 && tl_slot >= 0) a.prof[((size_t)tl_slot * 128 + p) * 4 + (k)] = gtimer();
#else
#define GJ_TL(k)
#endif
  unsigned* arrivals = a.sync;   // tile workers: G - 1 per phase with a next diagonal block, G in the last
  unsigned* published = a.sync + 1;  // D_0^{-1} .. published by CTA 0
  unsigned* feed = a.sync + 2;   // feed[p]: finished feeder tasks of phase p
  if (cta == 0) {
    // *info = 0 before the first hand-off; every check that can set it runs
    // after that
    if (tid == 0) *a.info = 0;
    __syncthreads();
    const int kb = N < kP ? N : kP;
    for (int e = tid; e < kP * kP; e += kThr) {
      const int c = e >> 5, r = e & 31;
      if (r < kb && c < kb) s.dg[c * 33 + r] = __ldcg(a.A + (size_t)c * N + r);
    }
    gj_diag(a, 0, kb, s);
    cta_signal(published);  // D_0^{-1}
  }
  TileRegs R;
  // The tile tasks of phase p that produce the next diagonal block of phase
  // p + 1 ("feeders": row blocks 0, 1 x column blocks 0, 1 minus the
  // special task itself) — CTA 0 waits for these only.
  auto nfeed = [&](const Phase& ph) {
    const int ni = ph.nbelow < 2 ? ph.nbelow : 2, nj = ph.ncb < 2 ? ph.ncb : 2;
    return ph.kb2 > 0 ? ni * nj - 1 : 0;
  };
  auto is_feeder = [&](const Phase& ph, const Task& k) {
    return ph.kb2 > 0 && k.I < 2 && k.J < 2 && k.I < ph.nbelow;
  };
  for (int p = 0; p < npan; ++p) {
    GJ_PHASE(3)
    const Phase ph(N, p);
    const bool has_diag = ph.kb2 > 0;
    const int ntile = ph.nrb * ph.ncb - (has_diag ? 1 : 0);
    const bool special = has_diag && cta == 0 && G > 1;
    if (special) {
      // wait only for the feeders of phase p - 1, then the next diagonal
      // block: W of its columns, multipliers checked, updated block kept in
      // shared memory, factored
      GJ_TL(0)
      const int declined = p > 0 ? cta_wait_info(feed + (p - 1), (unsigned)nfeed(Phase(N, p - 1)), a.info) : 0;
      GJ_TL(1)
      GJ_SP(0)
      if (declined == 0) {
        GJ_SP(1)
        special_tile(a, ph, s, true);
        GJ_SP(5)
        GJ_TL(2)
        unsigned long long td = pr ? gtimer() : 0;
        gj_diag(a, p + 1, ph.kb2, s);
        if (pr) a.prof[9] += gtimer() - td;
      }
      GJ_TL(3)
      cta_signal(published);  // D_{p+1}^{-1} (also when skipped)
    } else {
      // every tile worker has finished the earlier phases (all of them had a
      // next diagonal block: G - 1 workers each) and D_p^{-1} is published
      GJ_TL(0)
      if (G > 1) {
        cta_wait(arrivals, (unsigned)(G - 1) * (unsigned)p, a.info, false);
        GJ_TL(1)
        cta_wait(published, (unsigned)p + 1u, a.info, false);
      }
      GJ_TL(2)
      const bool live = __ldcg(a.info) == 0;
      if (has_diag && G == 1 && live) {
        special_tile(a, ph, s, false);
        gj_diag(a, p + 1, ph.kb2, s);
      }
      // a contiguous chunk of the J-major task list (consecutive tasks share
      // W); the next task's loads are in flight while one computes.  A
      // one-CTA launch (small N) does all of it after the diagonal block.
      const bool sep = has_diag && G > 1;
      const int G1 = sep ? G - 1 : G, me = sep ? cta - 1 : cta, off = has_diag ? 1 : 0;
      const int t0 = (int)((long long)ntile * me / G1), t1 = (int)((long long)ntile * (me + 1) / G1);
      if (t0 < t1) {
        Task k = task_of(ph, t0 + off);
        if (live) {
          tile_load(a, ph, k, true, R);
          load_inv(a, p, s);
        }
        int lastJ = -1;
        for (int tt = t0; tt < t1; ++tt) {
          Task kn = k;
          if (live) {
            const bool neww = k.J != lastJ;
            const int buf = (tt - t0) & 1;
            tile_stage(R, neww, s, buf);
            double cv[4][2][2];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) cv[i][j][h] = R.cv[i][j][h];
            __syncthreads();
            if (tt + 1 < t1) {
              kn = task_of(ph, tt + 1 + off);
              tile_load(a, ph, kn, kn.J != k.J, R);
            }
            // multipliers of rows below the panel are checked once per row
            // block, in its first column block
            // (the next diagonal block's rows, I = 0, have no tile in column block 0 — that is
            // CTA 0's special tile — and are checked with column block 1)
            tile_compute(a, ph, k, cv, neww, k.I == 0,
                         k.I < ph.nbelow && k.J == (has_diag && k.I == 0 ? 1 : 0), false, s, buf);
            lastJ = k.J;
          } else if (tt + 1 < t1) {
            kn = task_of(ph, tt + 1 + off);
          }
          if (G > 1 && is_feeder(ph, k)) cta_signal(feed + p);  // signalled even when skipped
          k = kn;
        }
      }
      __syncthreads();
      GJ_TL(3)
      if (G > 1) cta_signal(arrivals);
    }
    GJ_PHASE(0)
  }
  // the system is now the identity on every panel: b holds x except the
  // last panel's rows, which are in its row-panel buffer (a single panel
  // never ran a tile phase: x = D^{-1} b)
  if (cta == 0) {
    // the last phase has no next diagonal block: all G CTAs were tile workers
    if (G > 1) cta_wait(arrivals, (unsigned)(G - 1) * (unsigned)(npan - 1) + (unsigned)G, a.info, false);
    if (__ldcg(a.info) == 0) {
      const int p = npan - 1, k0 = p * kP, kb = N - k0;
      if (npan > 1) {
        if (tid < kb) a.b[k0 + tid] = __ldcg(a.wbuf + (size_t)(p % 3) * kP * (N + 1) + (size_t)N * kP + tid);
      } else {
        double* sy = s.dg;
        if (tid < kP) sy[tid] = tid < kb ? __ldcg(a.b + tid) : 0.0;
        __syncthreads();
        if (tid < kb) {
          double v = 0.0;
          for (int k = 0; k < kb; ++k) v = fma(__ldcg(a.inv + k * kP + tid), sy[k], v);
          a.b[tid] = v;
        }
      }
    }
  }
  (void)grid;
  GJ_PHASE(2)
#undef GJ_PHASE
}

}  // namespace

#ifndef GJ_MICRO

bool gj_solve_nopivot(int N, double* A, double* b, int* info_dev) {
  const int sms = num_sms();
  int grid = sm_budget() > 0 && sm_budget() < sms ? sm_budget() : sms;
  if (N < 1 || N > 8192) return false;
  // no more CTAs than the first (largest) phase has tile tasks: a smaller
  // grid makes every grid barrier cheaper; tiny systems run on one CTA
  {
    const int kb2 = N - kP < kP ? N - kP : kP, rest = N - kP - kb2;
    const int nrb = (kb2 > 0 ? 1 : 0) + (rest > 0 ? (rest + kT - 1) / kT : 0);
    const int crest = N + 1 - kP - kb2;
    const int ncb = (kb2 > 0 ? 1 : 0) + (crest + kT - 1) / kT;
    const int tasks = nrb * ncb;  // including the diagonal block's
    const int want = tasks <= 3 ? 1 : tasks;
    if (want < grid) grid = want;
  }
  const size_t smem = sizeof(Smem);
  max_dynamic_smem((const void*)gj_kernel, (int)smem);
  const int npan = (N + kP - 1) / kP;
  double* inv = allocator().alloc((size_t)npan * kInv);
  double* wbuf = allocator().alloc((size_t)3 * kP * (N + 1));
  unsigned* sync = zero_words((size_t)npan + 3);
  GjArgs a{N, A, b, inv, wbuf, info_dev, sync, nullptr};  // *info zeroed by the kernel
  void* params[] = {&a};
  {
    // algorithmic work of the operation (a dense solve: LU 2/3 N^3 + two triangular
    // solves 2 N^2), not the N^3 this Gauss-Jordan variant executes; bytes: one read
    // and one write of the matrix
    LaunchScope ls("gj_nopivot", 2.0 / 3.0 * (double)N * N * N + 2.0 * (double)N * N,
                   16.0 * (double)N * N);
    T2S2_CUDA(cudaLaunchCooperativeKernel((void*)gj_kernel, dim3(grid), dim3(kThr), params, smem,
                                          stream()));
  }
  allocator().release(inv);
  allocator().release(wbuf);
  return true;
}

#endif  // GJ_MICRO

}  // namespace t2s2
