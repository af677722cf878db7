// Device GMRES(restart) and Jacobi-PCG (see iterative.h).
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cmath>

#include "blas.h"
#include "gemm_device.cuh"
#include "iterative.h"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace t2s2 {
namespace {

constexpr int kMaxRestart = 64;
constexpr int kThreads = 1024;

struct GmState {
  double h[kMaxRestart][kMaxRestart + 1];  // h[col][row] as in scipy
  double gc[kMaxRestart], gs[kMaxRestart];
  double S[kMaxRestart + 1];
  double presid, ptol;
  int col_final;
  int active;
  int breakdown;
  int restart;
};

constexpr int kCgMaxCtas = 148;
__device__ double cta_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[32] = v;
  }
  __syncthreads();
  return red[32];
}

__device__ double cta_dot(const double* a, const double* b, int n, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s = fma(a[i], b[i], s);
  return cta_sum(s, red);
}

// LAPACK 3.10+ dlartg: c >= 0, r carries the sign of f, s = g / r.
__device__ void lartg(double f, double g, double& c, double& s, double& r) {
  if (g == 0.0) {
    c = 1.0;
    s = 0.0;
    r = f;
  } else if (f == 0.0) {
    c = 0.0;
    s = g > 0 ? 1.0 : -1.0;
    r = fabs(g);
  } else {
    double d = sqrt(f * f + g * g);
    c = fabs(f) / d;
    r = f > 0 ? d : -d;
    s = g / r;
  }
}

// New cycle: V[0] = r / ||r||, S = (||r||, 0, ...).
__global__ void __launch_bounds__(kThreads)
    gm_cycle_kernel(GmState* st, const double* r, double* V, int n, double ptol) {
  __shared__ double red[33];
  const double nr = sqrt(cta_dot(r, r, n, red));
  const double inv = 1.0 / nr;
  for (int i = threadIdx.x; i < n; i += blockDim.x) V[i] = r[i] * inv;
  for (int e = threadIdx.x; e < kMaxRestart * (kMaxRestart + 1); e += blockDim.x)
    (&st->h[0][0])[e] = 0.0;
  for (int e = threadIdx.x; e <= kMaxRestart; e += blockDim.x) st->S[e] = 0.0;
  if (threadIdx.x == 0) {
    st->S[0] = nr;
    st->ptol = ptol;
    st->active = 1;
    st->breakdown = 0;
    st->col_final = -1;
    st->presid = 0.0;
  }
}

__global__ void gm_set_restart(GmState* st, int restart) { st->restart = restart; }

// CTA 0's copy of the cycle's rotations and right-hand side (GmState gc, gs,
// S) and the Hessenberg column being finished.  The column update is a
// chain of dependent reads of what the previous iteration wrote: run against
// global memory every link was an L2 round trip (~20 us for column 40,
// most of the Arnoldi step); here it runs in shared memory and global memory
// only receives the results.
struct RotSmem {
  double gc[kMaxRestart], gs[kMaxRestart], S[kMaxRestart + 1], hc[kMaxRestart + 2];
};

// thread 0 of CTA 0: load the rotations of the columns before col0
__device__ void rot_load(const GmState* st, RotSmem& r, int col0) {
  for (int k = threadIdx.x; k < col0; k += blockDim.x) {
    r.gc[k] = st->gc[k];
    r.gs[k] = st->gs[k];
  }
  for (int k = threadIdx.x; k <= col0; k += blockDim.x) r.S[k] = st->S[k];
  __syncthreads();
}

// one thread: r.hc[0..col] = the new column's projections, h1 = ||w|| after
// orthogonalisation; previous rotations applied, the new one formed (LAPACK
// dlartg), S advanced, convergence / breakdown / last column recorded
__device__ void finish_column(GmState* st, RotSmem& r, int col, double h1, bool brk, int restart) {
  double* hc = r.hc;
  hc[col + 1] = brk ? 0.0 : h1;
  for (int k = 0; k < col; ++k) {
    const double c = r.gc[k], s = r.gs[k];
    const double n0 = hc[k], n1 = hc[k + 1];
    hc[k] = c * n0 + s * n1;
    hc[k + 1] = -s * n0 + c * n1;
  }
  double c, s, mag;
  lartg(hc[col], hc[col + 1], c, s, mag);
  r.gc[col] = c;
  r.gs[col] = s;
  hc[col] = mag;
  hc[col + 1] = 0.0;
  const double t = -s * r.S[col];
  r.S[col] = c * r.S[col];
  r.S[col + 1] = t;
  // results to global memory (stores only)
  double* gh = st->h[col];
  for (int k = 0; k <= col + 1; ++k) gh[k] = hc[k];
  st->gc[col] = c;
  st->gs[col] = s;
  st->S[col] = r.S[col];
  st->S[col + 1] = t;
  st->presid = fabs(t);
  if (brk) st->breakdown = 1;
  if (fabs(t) <= st->ptol || brk || col == restart - 1) {
    st->active = 0;
    st->col_final = col;
  }
}

// Arnoldi step for column col (w = A v_col already in V[col+1]) on one CTA:
// modified Gram-Schmidt as scipy's loop (small systems).
__device__ void gm_arnoldi_cta(GmState* st, double* V, int n, int col, int restart, double* red,
                               RotSmem& rot) {
  double* w = V + (size_t)(col + 1) * n;
  const double h0 = sqrt(cta_dot(w, w, n, red));
  for (int k = 0; k <= col; ++k) {
    const double* vk = V + (size_t)k * n;
    const double t = cta_dot(vk, w, n, red);
    if (threadIdx.x == 0) rot.hc[k] = t;
    for (int i = threadIdx.x; i < n; i += blockDim.x) w[i] = fma(-t, vk[i], w[i]);
    __syncthreads();
  }
  const double h1 = sqrt(cta_dot(w, w, n, red));
  const bool brk = h1 <= DBL_EPSILON * h0;
  if (!brk) {
    const double inv = 1.0 / h1;
    for (int i = threadIdx.x; i < n; i += blockDim.x) w[i] *= inv;
  }
  if (threadIdx.x == 0) finish_column(st, rot, col, h1, brk, restart);
}

// Arnoldi step over G CTAs (cooperative): classical Gram-Schmidt applied
// twice (CGS2, as orthogonal as scipy's modified Gram-Schmidt to working
// precision) so the column costs three grid barriers instead of one CTA-wide
// reduction per basis vector.  Dots: per-CTA partials (warp per basis
// vector), every CTA sums them in the same order.
// vb(k): this CTA's chunk (len entries) of basis vector k; wl: its chunk of w.
template <class BasisChunk>
__device__ void mc_dots(const BasisChunk& vb, const double* wl, int len, int nk, double* part, int G) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = warp; k < nk; k += nw) {
    const double* v = k < nk - 1 ? vb(k) : wl;  // last: ||w||^2
    double acc = 0.0;
    for (int j = lane; j < len; j += 32) acc = fma(v[j], wl[j], acc);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) part[(size_t)k * G + blockIdx.x] = acc;
  }
}

// out[k] = sum_c part[k * G + c] for k < nk in a fixed order (every CTA the
// same bits): warp w takes rows k = w, w + nw, ...; lane l adds the partials
// c = l, l + 32, ... in that order, then the lanes combine by a butterfly.
// All loads of a warp's rows are issued before the first sum, so a call
// costs one L2 round trip plus five shuffle steps per row (an ordered walk
// over G partials per row made the Arnoldi step of a 40-column cycle spend
// more time summing than orthogonalising).
constexpr int kMaxPartialsPerLane = (kCgMaxCtas + 31) / 32;
constexpr int kMaxRowsPerWarp = (kMaxRestart + 2 + 7) / 8;  // 8 warps per CTA
__device__ __forceinline__ void sum_partials(const double* part, int G, int nk, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double v[kMaxRowsPerWarp];
#pragma unroll
  for (int r = 0; r < kMaxRowsPerWarp; ++r) {
    const int k = warp + r * nw;
    double t = 0.0;
    if (k < nk) {
#pragma unroll
      for (int j = 0; j < kMaxPartialsPerLane; ++j) {
        const int c = lane + 32 * j;
        if (c < G) t += __ldcg(part + (size_t)k * G + c);
      }
    }
    v[r] = t;
  }
#pragma unroll
  for (int r = 0; r < kMaxRowsPerWarp; ++r) {
    const int k = warp + r * nw;
    if (k < nk) {  // uniform over the warp
      double t = v[r];
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) out[k] = t;
    }
  }
}

struct ArnoldiSmem {
  double hs[kMaxRestart + 2], h2[kMaxRestart + 2], red[33], sw1[1];
};
__device__ void gm_arnoldi_grid(GmState* st, double* V, int n, int col, double* part, int G,
                                cg::grid_group& grid, ArnoldiSmem& sm, RotSmem& rot, double* Vs, int stride) {
  // Vs (may be null): this CTA's chunk of every basis vector, resident in
  // shared memory for the whole cycle (slot k at Vs + k * stride, slots
  // 0..col loaded, slot col + 1 receives w): the dots and updates of CGS2
  // then read shared memory instead of col + 1 rows of V from L2, twice.
  double* hs = sm.hs;
  double* h2 = sm.h2;
  const bool vec = (int)blockIdx.x < G;  // CTAs beyond G only join the barriers
  const int chunk = (n + G - 1) / G, i0 = vec ? blockIdx.x * chunk : n;
  const int i1 = i0 + chunk < n ? i0 + chunk : n;
  const int len = i1 > i0 ? i1 - i0 : 0;
  double* w = V + (size_t)(col + 1) * n;
  double* wl = Vs ? Vs + (size_t)(col + 1) * stride : w + i0;  // this CTA's chunk of w
  auto vb = [&](int k) -> const double* { return Vs ? Vs + (size_t)k * stride : V + (size_t)k * n + i0; };
  if (Vs && vec) {
    for (int j = threadIdx.x; j < len; j += blockDim.x) wl[j] = __ldcg(w + i0 + j);
    __syncthreads();
  }
  const int nk = col + 2;  // col+1 dots and ||w||^2
  // two partial buffers: the second pass may write while a slow CTA still sums the first
  double* part2 = part + (size_t)(kMaxRestart + 3) * kCgMaxCtas;
  if (vec) mc_dots(vb, wl, len, nk, part, G);
  grid.sync();
  if (vec) {
    sum_partials(part, G, nk, hs);
    __syncthreads();
    for (int j = threadIdx.x; j < len; j += blockDim.x) {
      double x = wl[j];
      for (int k = 0; k <= col; ++k) x = fma(-hs[k], vb(k)[j], x);
      wl[j] = x;
    }
    __syncthreads();
    mc_dots(vb, wl, len, nk, part2, G);
  }
  grid.sync();
  double ww = 0.0;
  if (vec) {
    sum_partials(part2, G, nk, h2);
    __syncthreads();
    for (int j = threadIdx.x; j < len; j += blockDim.x) {
      double x = wl[j];
      for (int k = 0; k <= col; ++k) x = fma(-h2[k], vb(k)[j], x);
      wl[j] = x;
      ww = fma(x, x, ww);
    }
  }
  for (int o = 16; o > 0; o >>= 1) ww += __shfl_xor_sync(0xffffffffu, ww, o);
  double* red = sm.red;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = ww;
  __syncthreads();
  if (threadIdx.x == 0 && vec) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
    part[(size_t)(kMaxRestart + 2) * G + blockIdx.x] = t;
  }
  grid.sync();
  if (!vec) return;
  sum_partials(part + (size_t)(kMaxRestart + 2) * G, G, 1, sm.sw1);
  __syncthreads();
  const double sww = sm.sw1[0];
  const double h0 = sqrt(hs[nk - 1]);
  const double h1 = sqrt(sww);
  const bool brk = h1 <= DBL_EPSILON * h0;
  if (!brk) {
    const double inv = 1.0 / h1;
    for (int j = threadIdx.x; j < len; j += blockDim.x) wl[j] *= inv;
  }
  if (Vs) {  // the next matvec and the final update read V from global memory
    __syncthreads();
    for (int j = threadIdx.x; j < len; j += blockDim.x) w[i0 + j] = wl[j];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k <= col; ++k) rot.hc[k] = hs[k] + h2[k];
    finish_column(st, rot, col, h1, brk, st->restart);
  }
}

// y = H^{-1} S (upper triangular, scipy's pseudo-solve), x += y V.
__global__ void __launch_bounds__(kThreads)
    gm_update_kernel(GmState* st, const double* V, double* x, int n) {
  __shared__ double y[kMaxRestart];
  const int c = st->col_final;
  if (threadIdx.x == 0) {
    if (st->h[c][c] == 0.0) st->S[c] = 0.0;
    for (int k = 0; k <= c; ++k) y[k] = st->S[k];
    for (int k = c; k > 0; --k) {
      if (y[k] != 0.0) {
        y[k] /= st->h[k][k];
        const double t = y[k];
        for (int j = 0; j < k; ++j) y[j] -= t * st->h[k][j];
      }
    }
    if (y[0] != 0.0) y[0] /= st->h[0][0];
  }
  __syncthreads();
  // every CTA solved for y itself; the update is split over the grid
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = x[i];
    for (int k = 0; k <= c; ++k) acc = fma(y[k], V[(size_t)k * n + i], acc);
    x[i] = acc;
  }
}

// scipy cg (Jacobi-preconditioned) as ONE cooperative kernel for the whole
// iteration loop: the matvec q = A p is a GEMM program run inside the loop
// (gemm_device.cuh, a grid barrier between its stages), the vector updates
// and the three sums of an iteration run on the first a.G CTAs, and every CTA
// decides convergence from the same sums, so the loop ends grid-wide without
// the host.  Reductions are deterministic: per-CTA partials, one grid
// barrier, every CTA sums the G partials in CTA order (sum_partials: the
// loads in flight at once, the adds in order).  With an empty program the
// kernel runs the vector part of ONE iteration after a matvec launched
// before it (operators whose matvec does not fit one program).
struct CgState {
  double rho_cur;
  int active;
  int iters;  // iterations performed so far
};

struct PcgArgs {
  CgState* st;
  const double* q;  // A p
  double* x;
  double* r;
  const double* diag;
  double* p;
  double* part;  // 3 * G partials
  int n, G;
  double atol;
  int top;         // start with the top of iteration 0 (rho, p from the initial residual)
  int it0, count;  // then iterations it0 .. it0 + count - 1
};

constexpr int kPcgThreads = 256;  // the GEMM programs' CTA

__device__ __forceinline__ double block_reduce(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  return t;
}

template <bool WIDE>
__global__ void __launch_bounds__(kPcgThreads, 2)
    pcg_kernel(const __grid_constant__ GemmProgram prog, const PcgArgs a) {
  extern __shared__ __align__(16) double gemm_smem[];
  __shared__ double red[32];
  __shared__ double sums[2];
  cg::grid_group grid = cg::this_grid();
  CgState* st = a.st;
  if (!st->active) return;  // uniform: written only after a grid barrier of this launch
  const int G = a.G, n = a.n;
  const bool vec = (int)blockIdx.x < G;  // this CTA takes part in the vector phases
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = G * blockDim.x;
  const double* q = a.q;
  const double* diag = a.diag;
  double *x = a.x, *r = a.r, *p = a.p, *part = a.part;
  double rho_cur;
  if (a.top) {
    // top of iteration 0: ||r|| < atol -> stop; rho = r.(r/diag); p = r/diag
    if (vec) {
      double rr = 0.0, rz = 0.0;
      for (int i = gt; i < n; i += gs) {
        const double ri = r[i];
        rr = fma(ri, ri, rr);
        rz = fma(ri, ri / diag[i], rz);
      }
      rr = block_reduce(rr, red);
      rz = block_reduce(rz, red);
      if (threadIdx.x == 0) {
        part[blockIdx.x] = rr;
        part[G + blockIdx.x] = rz;
      }
    }
    grid.sync();
    sum_partials(part, G, 2, sums);  // rows: rr partials, rz partials
    __syncthreads();
    const double srr = sums[0];
    rho_cur = sums[1];
    if (sqrt(srr) < a.atol) {
      if (blockIdx.x == 0 && threadIdx.x == 0) st->active = 0;
      return;
    }
    if (vec)
      for (int i = gt; i < n; i += gs) p[i] = r[i] / diag[i];
    if (a.count == 0) {
      // the matvec runs outside: this launch was the top of iteration 0 only
      if (blockIdx.x == 0 && threadIdx.x == 0) st->rho_cur = rho_cur;
      return;
    }
    grid.sync();  // p complete before the first matvec
  } else {
    rho_cur = st->rho_cur;
  }
  int it = a.it0;
  bool done = false;
  for (; it < a.it0 + a.count; ++it) {
    if (prog.nstage > 0) {
      gemm_device::gemm_program_run<WIDE>(prog, gemm_smem, grid);  // q = A p
      grid.sync();
    }
    // alpha = rho / p.q
    if (vec) {
      double pq = 0.0;
      for (int i = gt; i < n; i += gs) pq = fma(p[i], q[i], pq);
      pq = block_reduce(pq, red);
      if (threadIdx.x == 0) part[2 * G + blockIdx.x] = pq;
    }
    grid.sync();
    __syncthreads();  // sums[] of the previous phase read by every thread
    sum_partials(part + 2 * G, G, 1, sums);
    __syncthreads();
    const double alpha = rho_cur / sums[0];
    // x += alpha p, r -= alpha q, and the next iteration's top
    if (vec) {
      double rr = 0.0, rz = 0.0;
      for (int i = gt; i < n; i += gs) {
        x[i] = fma(alpha, p[i], x[i]);
        const double ri = fma(-alpha, q[i], r[i]);
        r[i] = ri;
        rr = fma(ri, ri, rr);
        rz = fma(ri, ri / diag[i], rz);
      }
      rr = block_reduce(rr, red);
      rz = block_reduce(rz, red);
      if (threadIdx.x == 0) {
        part[blockIdx.x] = rr;
        part[G + blockIdx.x] = rz;
      }
    }
    grid.sync();
    __syncthreads();  // sums[0] (p.q) read by every thread above
    sum_partials(part, G, 2, sums);
    __syncthreads();
    const double srr = sums[0], rho = sums[1];
    if (sqrt(srr) < a.atol) {
      done = true;
      ++it;
      break;
    }
    const double beta = rho / rho_cur;
    if (vec)
      for (int i = gt; i < n; i += gs) p[i] = fma(p[i], beta, r[i] / diag[i]);
    rho_cur = rho;
    // p complete before the next matvec of this launch reads it (the launch
    // boundary orders it otherwise)
    if (prog.nstage > 0 && it + 1 < a.it0 + a.count) grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->rho_cur = rho_cur;
    st->iters = it;
    if (done) st->active = 0;
  }
}

// The column loop of one GMRES cycle as ONE cooperative kernel: for each
// column the matvec V[col + 1] = A V[col] (the GEMM program, built for column
// 0 and shifted by col * n in a shared-memory copy), then the Arnoldi step —
// CGS2 over the first a.G CTAs, or scipy's modified Gram-Schmidt on CTA 0 for
// small systems — whose state update (Givens rotation, convergence) ends the
// loop grid-wide through st->active.  With an empty program the kernel runs
// the Arnoldi step of ONE column after a matvec launched before it.
struct GmresArgs {
  GmState* st;
  double* V;
  double* part;
  int n, G, restart;
  int col0, ncol;  // columns col0 .. col0 + ncol - 1
  // resident basis: each vector CTA keeps its chunk of V[0..restart] in
  // shared memory behind the GEMM ring (vs_off doubles in), stride doubles
  // per vector; stride == 0: the basis is read from global memory
  int vs_off, stride;
};

template <bool WIDE>
__global__ void __launch_bounds__(kPcgThreads, 2)
    gmres_cols_kernel(const __grid_constant__ GemmProgram prog, const GmresArgs a) {
  extern __shared__ __align__(16) double gemm_smem[];
  __shared__ GemmProgram sp;
  __shared__ ArnoldiSmem sm;
  __shared__ RotSmem rot;
  cg::grid_group grid = cg::this_grid();
  GmState* st = a.st;
  if (!st->active) return;  // uniform: written only after a grid barrier of this launch
  static_assert(sizeof(GemmProgram) % 8 == 0, "GemmProgram copied in 8-byte words");
  if (prog.nstage > 0) {
    const long long* src = reinterpret_cast<const long long*>(&prog);
    long long* dst = reinterpret_cast<long long*>(&sp);
    for (int i = threadIdx.x; i < (int)(sizeof(GemmProgram) / 8); i += blockDim.x) dst[i] = src[i];
  }
  const double* lo = a.V;                      // the program reads V[0] and writes V[1]:
  const double* hi = a.V + 2 * (size_t)a.n;    // operands in [lo, hi) move with the column
  if (blockIdx.x == 0) rot_load(st, rot, a.col0);
  double* Vs = a.stride > 0 ? gemm_smem + a.vs_off : nullptr;
  if (Vs && (int)blockIdx.x < a.G) {
    // this CTA's chunk of the basis vectors that exist already
    const int chunk = (a.n + a.G - 1) / a.G, i0 = blockIdx.x * chunk;
    const int len = (i0 + chunk < a.n ? i0 + chunk : a.n) - i0;
    for (int k = 0; k <= a.col0; ++k)
      for (int j = threadIdx.x; j < len; j += blockDim.x)
        Vs[(size_t)k * a.stride + j] = __ldcg(a.V + (size_t)k * a.n + i0 + j);
  }
  for (int col = a.col0; col < a.col0 + a.ncol; ++col) {
    if (prog.nstage > 0) {
      __syncthreads();
      if ((int)threadIdx.x < prog.nprob) {
        const GemmProb& g = prog.p[threadIdx.x];
        const size_t off = (size_t)col * a.n;
        GemmProb& t = sp.p[threadIdx.x];
        t.A = (g.A >= lo && g.A < hi) ? g.A + off : g.A;
        t.B = (g.B >= lo && g.B < hi) ? g.B + off : g.B;
        t.C = (g.C >= lo && g.C < hi) ? g.C + off : g.C;
      }
      __syncthreads();
      gemm_device::gemm_program_run<WIDE>(sp, gemm_smem, grid);
      grid.sync();
    }
    if (a.G > 1)
      gm_arnoldi_grid(st, a.V, a.n, col, a.part, a.G, grid, sm, rot, Vs, a.stride);
    else if (blockIdx.x == 0)
      gm_arnoldi_cta(st, a.V, a.n, col, a.restart, sm.red, rot);
    if (col + 1 < a.col0 + a.ncol) {
      grid.sync();  // CTA 0's state update is visible
      if (!__ldcg(&st->active)) break;
    }
  }
}

template <class T>
T read_state(const T* d) {
  T h;
  host_read(&h, d, sizeof(T));
  return h;
}

int read_flag(const int* d) { return read_state<int>(d); }

}  // namespace

int gmres(const ProgramBuilder& A, int n, const double* b, double* x, double rtol, int restart,
          int maxiter) {
  const double bnrm2 = dnrm2(b, n);
  const double atol = rtol * bnrm2;  // scipy: max(atol=0, rtol*||b||)
  if (bnrm2 == 0.0) {
    dcopy(x, b, n);
    return 0;
  }
  if (restart > n) restart = n;
  if (restart > kMaxRestart) restart = kMaxRestart;
  double* V = allocator().alloc((size_t)(restart + 1) * n);
  double* r = allocator().alloc(n);
  GmState* st = reinterpret_cast<GmState*>(allocator().alloc(sizeof(GmState) / sizeof(double) + 1));
  double* part = allocator().alloc((size_t)2 * (kMaxRestart + 3) * kCgMaxCtas);  // two CGS2 passes
  auto release = [&]() {
    allocator().release(V);
    allocator().release(r);
    allocator().release(part);
    allocator().release(reinterpret_cast<double*>(st));
  };
  auto residual = [&]() {  // r = b - A x, returns ||r||
    GemmBatch gb;
    A(gb, x, r);
    gb.run();
    daxpby(1.0, b, -1.0, r, n);
    return dnrm2(r, n);
  };
  double rnorm = residual();
  int inner = 0;
  if (rnorm < atol) {
    release();
    return 0;
  }
  // the matvec V[1] = A V[0] as one program inside the column kernel, which
  // shifts it from column to column; T2S2_KRYLOV_EXTERNAL_MATVEC=1 (tests: same
  // bits either way) launches it separately as operators beyond one program do
  GemmBatch gbq;
  A(gbq, V, V + n);
  GemmProgram prog{};
  bool wide = false;
  int max_tiles = 0;
  double mv_flops = 0.0;
  static const bool external = getenv("T2S2_KRYLOV_EXTERNAL_MATVEC") != nullptr;
  const bool fused = !external && gbq.build_program(prog, wide, max_tiles, mv_flops);
  if (!fused) prog = GemmProgram{};
  const void* kern = wide ? (const void*)gmres_cols_kernel<true> : (const void*)gmres_cols_kernel<false>;
  const int ring = gemm_program_smem(wide);
  // Vector CTAs.  Below 1024 unknowns one CTA runs scipy's modified
  // Gram-Schmidt.  Otherwise CGS2 over G CTAs, each with a chunk of at most
  // kResidentChunk entries of every basis vector resident in shared memory
  // when G such CTAs co-reside on this context's SMs (an SM partition has
  // fewer than the device's 148); larger systems read the basis from global
  // memory in chunks of >= 512.  The chunking is the same whether the matvec
  // runs inside the kernel or not (same bits), residency needs the loop kernel.
  constexpr int kResidentChunk = 320;
  int G = 1, stride = 0, smem = ring;
  if (n >= 1024) {
    const int g_res = (n + kResidentChunk - 1) / kResidentChunk;
    const int st_res = ((n + g_res - 1) / g_res + 1) & ~1;
    const int smem_res = ring + (restart + 1) * st_res * (int)sizeof(double);
    max_dynamic_smem(kern, smem_res);
    int cap_res = num_sms() * occupancy(kern, kPcgThreads, smem_res);
    if (sm_budget() > 0 && cap_res > sm_budget()) cap_res = sm_budget();
    if (g_res <= kCgMaxCtas && g_res <= cap_res) {
      G = g_res;
      // not on an SM partition: a green context refuses the cooperative launch
      // with this much dynamic shared memory ("too many blocks", measured with
      // 12 CTAs of 177 KB on 72 SMs); the basis is read from global memory there
      if (fused && !on_partition()) {
        stride = st_res;
        smem = smem_res;
      }
    } else {
      G = n / 512;
      if (G > kCgMaxCtas) G = kCgMaxCtas;
    }
  }
  max_dynamic_smem(kern, smem);
  // cooperative grid: no more CTAs than co-reside on this context's SMs
  int cap = num_sms() * occupancy(kern, kPcgThreads, smem);
  if (sm_budget() > 0 && cap > sm_budget()) cap = sm_budget();
  if (G > cap) G = cap;
  if (G < 1) G = 1;
  int grid = fused && max_tiles > G ? max_tiles : G;
  if (grid > cap) grid = cap;
  GmresArgs ga{st, V, part, n, G, restart, 0, restart, ring / (int)sizeof(double), stride};
  auto launch = [&](int col0, int ncol) {
    ga.col0 = col0;
    ga.ncol = ncol;
    void* params[] = {&prog, &ga};
    LaunchScope ls("gmres", 0.0, 0.0);
    T2S2_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kPcgThreads), params, smem, stream()));
  };
  constexpr int poll = 16;  // external matvec: host poll interval of the convergence flag
  double ptol_max_factor = 1.0;
  double ptol = bnrm2 * std::fmin(ptol_max_factor, atol / bnrm2);
  for (int it = 0; it < maxiter; ++it) {
    {
      LaunchScope ls("gmres", 3.0*n, 24.0*n);
      gm_cycle_kernel<<<1, kThreads, 0, stream()>>>(st, r, V, n, ptol);
      gm_set_restart<<<1, 1, 0, stream()>>>(st, restart);
    }
    T2S2_CHECK_LAUNCH();
    if (fused) {
      launch(0, restart);
      T2S2_CHECK_LAUNCH();
    } else {
      for (int col = 0; col < restart; ++col) {
        if (col > 0 && col % poll == 0 && !read_flag(&st->active)) break;
        GemmBatch gb;  // skipped on the device once converged
        gb.set_guard(&st->active);
        A(gb, V + (size_t)col * n, V + (size_t)(col + 1) * n);
        gb.run();
        launch(col, 1);
        T2S2_CHECK_LAUNCH();
      }
    }
    {
      LaunchScope ls("gmres", 2.0*n*restart, 8.0*n*restart);
      gm_update_kernel<<<G, kThreads, 0, stream()>>>(st, V, x, n);
    }
    T2S2_CHECK_LAUNCH();
    GmState h = read_state<GmState>(st);
    const int cols = h.col_final + 1;
    inner += cols;
    // the work of the columns performed (known only now): matvecs inside the
    // kernel, and 8 n flops per basis vector and column for CGS2
    amend_work("gmres", (fused ? cols * mv_flops : 0.0) + 4.0 * n * cols * (cols + 3.0),
               16.0 * n * cols * (cols + 3.0));
    const double presid = h.presid;
    rnorm = residual();
    if (rnorm <= atol) break;
    if (h.breakdown) break;
    if (presid <= ptol)
      ptol_max_factor = std::fmax(DBL_EPSILON, 0.25 * ptol_max_factor);
    else
      ptol_max_factor = std::fmin(1.0, 1.5 * ptol_max_factor);
    ptol = presid * std::fmin(ptol_max_factor, atol / rnorm);
  }
  release();
  return inner;
}

int pcg(const ProgramBuilder& A, int n, const double* b, double* x, const double* diag, double rtol,
        int maxiter) {
  const double bnrm2 = dnrm2(b, n);
  const double atol = rtol * bnrm2;
  if (bnrm2 == 0.0) {
    dcopy(x, b, n);
    return 0;
  }
  double* r = allocator().alloc(n);
  double* p = allocator().alloc(n);
  double* q = allocator().alloc(n);
  double* part = allocator().alloc(3 * kCgMaxCtas);
  CgState* st = reinterpret_cast<CgState*>(allocator().alloc(sizeof(CgState) / sizeof(double) + 1));
  auto apply = [&](const double* in, double* out) {
    GemmBatch gb;
    A(gb, in, out);
    gb.run();
  };
  apply(x, r);
  daxpby(1.0, b, -1.0, r, n);
  CgState init{0.0, 1, 0};
  T2S2_CUDA(cudaMemcpyAsync(st, &init, sizeof(CgState), cudaMemcpyHostToDevice, stream()));
  // the matvec q = A p as one program inside the kernel; T2S2_KRYLOV_EXTERNAL_MATVEC=1
  // (tests: same bits either way) launches it separately as operators
  // beyond one program do
  GemmBatch gbq;
  A(gbq, p, q);
  GemmProgram prog{};
  bool wide = false;
  int max_tiles = 0;
  double mv_flops = 0.0;
  static const bool external = getenv("T2S2_KRYLOV_EXTERNAL_MATVEC") != nullptr;
  const bool fused = !external && gbq.build_program(prog, wide, max_tiles, mv_flops);
  if (!fused) prog = GemmProgram{};
  const void* kern = wide ? (const void*)pcg_kernel<true> : (const void*)pcg_kernel<false>;
  const int smem = gemm_program_smem(wide);
  max_dynamic_smem(kern, smem);
  // cooperative grid: no more CTAs than co-reside on this context's SMs (an
  // SM partition has fewer than the device's 148); the vector phases run on
  // the first G CTAs — the same G, and so the same reduction order, with and
  // without the program
  int cap = num_sms() * occupancy(kern, kPcgThreads, smem);
  if (sm_budget() > 0 && cap > sm_budget()) cap = sm_budget();
  int G = (n + 1023) / 1024;
  if (G > kCgMaxCtas) G = kCgMaxCtas;
  if (G > cap) G = cap;
  if (G < 1) G = 1;
  int grid = fused && max_tiles > G ? max_tiles : G;
  if (grid > cap) grid = cap;
  PcgArgs a{st, q, x, r, diag, p, part, n, G, atol, 1, 0, maxiter};
  auto launch = [&](int top, int it0, int count) {
    a.top = top;
    a.it0 = it0;
    a.count = count;
    void* params[] = {&prog, &a};
    LaunchScope ls("cg", 0.0, 0.0);
    T2S2_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kPcgThreads), params, smem, stream()));
  };
  int it = 0;
  if (fused) {
    launch(1, 0, maxiter);
    T2S2_CHECK_LAUNCH();
    const CgState h = read_state<CgState>(st);
    it = h.iters;
    // the work of the iterations performed (known only now)
    amend_work("cg", it * (mv_flops + 12.0 * n) + 6.0 * n, it * 88.0 * n + 40.0 * n);
  } else {
    constexpr int poll = 20;  // iterations between host polls of the convergence flag
    launch(1, 0, 0);          // top of iteration 0
    for (; it < maxiter; ++it) {
      if (it > 0 && it % poll == 0 && !read_flag(&st->active)) break;
      GemmBatch gb;  // skipped on the device once converged
      gb.set_guard(&st->active);
      A(gb, p, q);
      gb.run();
      launch(0, it, 1);
      T2S2_CHECK_LAUNCH();
    }
    it = read_state<CgState>(st).iters;
    amend_work("cg", it * 12.0 * n + 6.0 * n, it * 88.0 * n + 40.0 * n);
  }
  allocator().release(r);
  allocator().release(p);
  allocator().release(q);
  allocator().release(part);
  allocator().release(reinterpret_cast<double*>(st));
  return it;
}

}  // namespace t2s2
