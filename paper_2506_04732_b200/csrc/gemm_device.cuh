// Device side of the GEMM programs (blas.h): the DMMA tile engine and the
// stage walker, shared by the program kernel (blas.cu) and the kernels that
// run a program inside their own loop (the Krylov solvers, iterative.cu).
#pragma once

#include <cooperative_groups.h>

#include "blas.h"

namespace t2s2 {
namespace gemm_device {

// Tile TM x TN x TK, 256 threads, FP64 tensor-core MMA (DMMA, mma.sync
// m8n8k4): D[8x8] += A[8x4] B[4x8].  Fragments: lane holds A[lane/4][lane%4],
// B[lane%4][lane/4], C/D[lane/4][2*(lane%4) + {0,1}].
// Operand K-tiles are staged by cp.async (8-byte elements, zero-filled out
// of bounds) through a kStages-deep shared-memory ring: kStages - 1 K-tiles
// are in flight while one is consumed, so a long-K tile costs about one
// exposed L2 latency in total instead of one per K-tile (the chains of the
// sweep are 1-12 K-tiles of 32 on a handful of CTAs).  The DMMA sequence and
// its operands are the same as with a single register prefetch, so results
// are bit-identical.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int kStages = 4;
// dynamic shared memory of a tile ring: ST stages of a TK x (TM+4) A tile and
// a TK x (TN+4) B tile
constexpr int ring_bytes(int TM, int TN, int TK, int ST) { return ST * 8 * TK * (TM + 4 + TN + 4); }
// the 32x32x32 and 64x64x16 rings (every program), and the 64x136x16 ring
// of programs with a problem whose N is 65..136 (see add_general)
constexpr int kGemmSmem = ring_bytes(32, 32, 32, kStages) > ring_bytes(64, 64, 16, kStages)
                              ? ring_bytes(32, 32, 32, kStages)
                              : ring_bytes(64, 64, 16, kStages);
constexpr int kWideN = 136;  // 17 DMMA columns
constexpr int kGemmSmemWide = ring_bytes(64, kWideN, 16, kStages) > kGemmSmem
                                  ? ring_bytes(64, kWideN, 16, kStages)
                                  : kGemmSmem;

// 8-byte async copy; !pred: the source is ignored and zeros are written
// (the ignore-src predicate form: one LDGSTS.ZFILL, no size arithmetic)
__device__ __forceinline__ void cp_async8(unsigned dst, const double* src, bool pred) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      " setp.eq.u32 p, %2, 0;\n"
      " cp.async.ca.shared.global [%0], [%1], 8, p;\n"
      "}\n" ::"r"(dst),
      "l"(src), "r"((unsigned)pred)
      : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Row offset of a 2-level row index: i -> (i / d) * hi + (i % d) * lo.
__device__ __forceinline__ long long row_off(int i, int d, long long hi, long long lo) {
  const int q = i / d;
  return q * hi + (long long)(i - q * d) * lo;
}

// One TM x TN output tile (tile coordinates bx, by of batch entry bz) of a
// general GEMM: A(i,k) = A[row(i) + k*ak], B(k,j) = B[k*bk + j*bj],
// C(i,j) = C[crow(i) + j*cj] (row() two-level, see GemmProb).  Operand
// tiles are fetched with consecutive threads on the contiguous index.
// WGM x WGN warps tile the output (4 x 2 by default; 8 x 1 for the wide
// tile, one warp per 8 rows across all 136 columns).
template <int TM, int TN, int TK, int ST = kStages, int WGM = 4, int WGN = 2>
__device__ __forceinline__ void gemm_tile(const GemmProb& g, int bx, int by, int bz, double* smem) {
  constexpr int PA = (TM * TK + 255) / 256, PB = (TK * TN + 255) / 256;
  constexpr int LA = TM + 4, LB = TN + 4;  // +4: conflict-free DMMA fragment loads
  constexpr int SA = TK * LA, SS = TK * (LA + LB);  // per stage: A tile then B tile
  const double* A = g.A + bz * g.sA;
  const double* B = g.B + bz * g.sB;
  double* C = g.C + bz * g.sC;
  const int M = g.M, N = g.N, K = g.K;
  const int row0 = by * TM, col0 = bx * TN;
  const int tid = threadIdx.x;
  const bool a_ifast = g.alo == 1;  // rows contiguous: threads walk i
  const bool b_jfast = g.bj == 1;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  // loop-invariant per-thread source offsets and shared-memory slots
  long long aoff[PA];
  int akk[PA];
  unsigned adst[PA];
  bool arow[PA], aval[PA];
#pragma unroll
  for (int t = 0; t < PA; ++t) {
    const int e = tid + t * 256;
    aval[t] = e < TM * TK;  // tiles that are not a multiple of 256 elements
    const int ai = a_ifast ? e % TM : e / TK;
    akk[t] = a_ifast ? e / TM : e % TK;
    const int gi = row0 + ai;
    arow[t] = gi < M;
    aoff[t] = (arow[t] ? row_off(gi, g.ad, g.ahi, g.alo) : 0) + (long long)akk[t] * g.ak;
    adst[t] = sbase + 8u * (unsigned)(akk[t] * LA + ai);
  }
  int bkk[PB];
  bool bcol[PB];
  long long boff[PB];
  unsigned bdst[PB];
  bool bval[PB];
#pragma unroll
  for (int t = 0; t < PB; ++t) {
    const int e = tid + t * 256;
    bval[t] = e < TK * TN;
    const int bj = b_jfast ? e % TN : e / TK;
    bkk[t] = b_jfast ? e / TN : e % TK;
    const int gj = col0 + bj;
    bcol[t] = gj < N;
    boff[t] = (long long)bkk[t] * g.bk + (bcol[t] ? (long long)gj * g.bj : 0);
    bdst[t] = sbase + 8u * (unsigned)(SA + bkk[t] * LB + bj);
  }
  const int nk = (K + TK - 1) / TK;
  // issue() runs for kt = 0, 1, 2, ... in order: each element keeps a running
  // source pointer (advanced by one K-tile per call) and the number of
  // K-tiles' worth of k it may still read, so a copy costs a compare, the
  // copy and a pointer increment instead of a 64-bit multiply-add per call.
  const double* ap[PA];
  int alim[PA];
#pragma unroll
  for (int t = 0; t < PA; ++t) {
    ap[t] = A + aoff[t];
    alim[t] = (aval[t] && arow[t]) ? K - akk[t] : 0;  // copy while k0 < alim
  }
  const double* bp[PB];
  int blim[PB];
#pragma unroll
  for (int t = 0; t < PB; ++t) {
    bp[t] = B + boff[t];
    blim[t] = (bval[t] && bcol[t]) ? K - bkk[t] : 0;
  }
  const long long astep = (long long)TK * g.ak, bstep = (long long)TK * g.bk;
  auto issue = [&](int kt) {  // K-tile kt into ring slot kt % ST (always commits a group)
    if (kt < nk) {
      const int k0 = kt * TK;
      const unsigned so = 8u * (unsigned)((kt % ST) * SS);
#pragma unroll
      for (int t = 0; t < PA; ++t) {
        if (!aval[t]) continue;
        const bool ok = k0 < alim[t];
        cp_async8(adst[t] + so, ok ? ap[t] : A, ok);
        ap[t] += astep;
      }
#pragma unroll
      for (int t = 0; t < PB; ++t) {
        if (!bval[t]) continue;
        const bool ok = k0 < blim[t];
        cp_async8(bdst[t] + so, ok ? bp[t] : B, ok);
        bp[t] += bstep;
      }
    }
    cp_async_commit();
  };
  // 8 warps on a 4 x 2 grid of (TM/4) x (TN/2) warp tiles of 8x8 DMMA blocks
  constexpr int WM = TM / WGM, WN = TN / WGN, MB = WM / 8, NB = WN / 8;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / WGN) * WM, wn0 = (warp % WGN) * WN;
  double tc[MB][NB][2] = {};
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) issue(s);
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<ST - 2>();  // this thread's copies of K-tile kt landed
    __syncthreads();          // everyone's did, and slot (kt - 1) % ST is free
    issue(kt + ST - 1);
    const double* As = smem + (kt % ST) * SS;
    const double* Bs = As + SA;
#pragma unroll
    for (int kk = 0; kk < TK; kk += 4) {
      const int kr = kk + (lane & 3);
      double af[MB], bf[NB];
#pragma unroll
      for (int i = 0; i < MB; ++i) af[i] = As[kr * LA + wm0 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < NB; ++j) bf[j] = Bs[kr * LB + wn0 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < MB; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) dmma_8x8x4(tc[i][j][0], tc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();  // drain the (empty) trailing groups
  __syncthreads();     // the ring is reused by the next tile
  const double alpha = g.alpha, beta = g.beta;
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int gi = row0 + wm0 + i * 8 + (lane >> 2);
    if (gi >= M) continue;
    const long long co = row_off(gi, g.cd, g.chi, g.clo);
#pragma unroll
    for (int j = 0; j < NB; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gj = col0 + wn0 + j * 8 + (lane & 3) * 2 + h;
        if (gj >= N) continue;
        double* c = C + co + (long long)gj * g.cj;
        if (g.rs || g.cs) {
          double v = alpha * tc[i][j][h];
          if (g.rs) v *= g.rs[gi];
          if (g.cs) v *= g.cs[gj];
          *c = v;
        } else {
          *c = beta == 0.0 ? alpha * tc[i][j][h] : alpha * tc[i][j][h] + beta * (*c);
        }
      }
  }
}

// elements per tile of a split-K reduction problem
constexpr int kReduceTile = 256;

// The stages of a program on the calling (cooperative) grid: every CTA
// walks the stage's tiles grid-strided, a grid barrier separates the stages
// (none after the last one).  WIDE: the instantiation that also has the
// 64x136 tile (a larger shared-memory ring), used only for programs
// containing such a problem; the other stages of a program with a wide
// problem run in the same instantiation.
template <bool WIDE>
__device__ __forceinline__ void gemm_program_run(const GemmProgram& prog, double* gemm_smem,
                                                 cooperative_groups::grid_group& grid) {
  for (int s = 0; s < prog.nstage; ++s) {
    const int q0 = prog.stage_first[s], q1 = prog.stage_first[s + 1];
    int total = 0;
    for (int q = q0; q < q1; ++q) total += prog.p[q].tiles;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int q = q0, tt = t;
      while (tt >= prog.p[q].tiles) {
        tt -= prog.p[q].tiles;
        ++q;
      }
      const GemmProb& g = prog.p[q];
      if (g.kind == 1) {
        // split-K reduction: C = alpha sum_j P[j] + beta C, partials added in
        // the order j = 0, 1, ... (32-bit index math: a local tensor has
        // fewer than 2^31 entries; four partial loads in flight per thread)
        const unsigned mn = (unsigned)g.M * (unsigned)g.N, N = (unsigned)g.N;
        const unsigned e0 = (unsigned)tt * kReduceTile;
        const unsigned e1 = e0 + kReduceTile < mn ? e0 + kReduceTile : mn;
        const double* P = g.A;
        for (unsigned e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
          double acc = 0.0;
          int j = 0;
          for (; j + 4 <= g.batch; j += 4) {
            const double v0 = P[(size_t)j * mn + e], v1 = P[(size_t)(j + 1) * mn + e];
            const double v2 = P[(size_t)(j + 2) * mn + e], v3 = P[(size_t)(j + 3) * mn + e];
            acc += v0;
            acc += v1;
            acc += v2;
            acc += v3;
          }
          for (; j < g.batch; ++j) acc += P[(size_t)j * mn + e];
          const unsigned i = e / N, c = e - i * N;
          double* cp = g.C + row_off((int)i, g.cd, g.chi, g.clo) + (long long)c * g.cj;
          if (g.rs || g.cs) {
            double v = g.alpha * acc;
            if (g.rs) v *= g.rs[i];
            if (g.cs) v *= g.cs[c];
            *cp = v;
          } else {
            *cp = g.beta == 0.0 ? g.alpha * acc : g.alpha * acc + g.beta * *cp;
          }
        }
        __syncthreads();
      } else if (WIDE && g.big == 2) {
        const int tm = (g.M + 63) / 64;
        gemm_tile<64, kWideN, 16, kStages, 8, 1>(g, 0, tt % tm, tt / tm, gemm_smem);
      } else if (g.big) {
        const int tn = (g.N + 63) / 64, tm = (g.M + 63) / 64;
        const int bz = tt / (tm * tn), rem = tt - bz * tm * tn;
        gemm_tile<64, 64, 16>(g, rem % tn, rem / tn, bz, gemm_smem);
      } else {
        const int tn = (g.N + 31) / 32, tm = (g.M + 31) / 32;
        const int bz = tt / (tm * tn), rem = tt - bz * tm * tn;
        gemm_tile<32, 32, 32>(g, rem % tn, rem / tn, bz, gemm_smem);
      }
    }
    if (s + 1 < prog.nstage) grid.sync();
  }
}

}  // namespace gemm_device
}  // namespace t2s2
