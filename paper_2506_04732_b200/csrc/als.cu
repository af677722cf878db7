// Rank-adaptive alternating TT solver on the device
// (reference: pkg/src/ttss/tt_solver.py).
//
// Sweep structure, candidate logic and truncation follow the reference
// exactly; every contraction, local matrix, factorisation and SVD runs on
// the GPU.  The host reads back only the scalars that steer control flow:
// candidate scores, singular values for the rank decisions, the residual.
#include <chrono>
#include <cmath>

#include "als.h"
#include "blas.h"
#include "iterative.h"
#include "linalg.h"
#include "tt.h"

namespace t2s2 {
namespace {

int grid_of(long long n) {
  long long g = (n + 255) / 256;
  if (g < 1) g = 1;
  if (g > 2368) g = 2368;
  return (int)g;
}

// Column-major Galerkin block B[(x,m,y),(X,n,Y)] = sum_ab pal[x,a,X] ac[a,m,n,b] par[y,b,Y]
// (tt_solver.py:213-216).
__global__ void galerkin_matrix_kernel(int rx, int n, int ry, int ra, int rb,
                                       const double* __restrict__ pal,
                                       const double* __restrict__ ac,
                                       const double* __restrict__ par, double* __restrict__ B) {
  const int N = rx * n * ry;
  // one column per block-row of threads: (col, row) from 2-D indexing
  for (int col = blockIdx.y; col < N; col += gridDim.y) {
    const int Y = col % ry, nn = (col / ry) % n, X = col / (ry * n);
    for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < N; row += gridDim.x * blockDim.x) {
    const int y = row % ry, m = (row / ry) % n, x = row / (ry * n);
    const long long e = (long long)col * N + row;
    double s = 0.0;
    for (int a = 0; a < ra; ++a) {
      const double pl = pal[((long long)x * ra + a) * rx + X];
      if (pl == 0.0) continue;
      const double* acp = ac + (((long long)a * n + m) * n + nn) * rb;
      const double* prp = par + (long long)y * rb * ry + Y;
      double t = 0.0;
      for (int b = 0; b < rb; ++b) t = fma(acp[b], prp[(long long)b * ry], t);
      s = fma(pl, t, s);
    }
    B[e] = s;
    }
  }
}

// The same block, factored: T_a[(m,y),(nn,Y)] = sum_b ac[a,m,nn,b] par[y,b,Y]
// does not depend on (x, X), so CTA c = (nn, Y) forms its slice of T for
// every a in shared memory once and then writes the rx columns (X, nn, Y)
// as B[(x,m,y), col] = sum_a pal[x,a,X] T_a[(m,y)] — per element ra fused
// multiply-adds from shared memory instead of ra (rb + 1) plus the operand
// loads and index divisions.  Every t and every s is formed by the same fma
// sequence as galerkin_matrix_kernel above, so B is bit-identical.
__global__ void __launch_bounds__(256)
    galerkin_factored_kernel(int rx, int n, int ry, int ra, int rb, const double* __restrict__ pal,
                             const double* __restrict__ ac, const double* __restrict__ par,
                             double* __restrict__ B) {
  extern __shared__ double gsm[];
  const int nry = n * ry, N = rx * nry, tid = threadIdx.x;
  double* T = gsm;             // ra x nry
  double* P = T + ra * nry;    // pal, rx x ra x rx
  for (int e = tid; e < rx * ra * rx; e += blockDim.x) P[e] = pal[e];
  for (int c = blockIdx.x; c < nry; c += gridDim.x) {
    const int nn = c / ry, Y = c - nn * ry;
    __syncthreads();  // P loaded; the previous slice's readers are done
    for (int e = tid; e < ra * nry; e += blockDim.x) {
      const int a = e / nry, my = e - a * nry, m = my / ry, y = my - m * ry;
      const double* acp = ac + (((long long)a * n + m) * n + nn) * rb;
      const double* prp = par + (long long)y * rb * ry + Y;
      double t = 0.0;
      for (int b = 0; b < rb; ++b) t = fma(acp[b], prp[(long long)b * ry], t);
      T[e] = t;
    }
    __syncthreads();
    for (int X = 0; X < rx; ++X) {
      double* Bc = B + ((long long)X * nry + c) * N;
      int x = 0, my = tid;
      while (my >= nry && x < rx) {
        my -= nry;
        ++x;
      }
      for (int row = tid; row < N; row += blockDim.x) {
        const double* pl = P + (x * ra) * rx + X;
        double s = 0.0;
        for (int a = 0; a < ra; ++a) {
          const double p = pl[a * rx];
          if (p == 0.0) continue;
          s = fma(p, T[a * nry + my], s);
        }
        Bc[row] = s;
        my += blockDim.x;
        while (my >= nry) {
          my -= nry;
          ++x;
        }
      }
    }
  }
}

// G[a,b,m,P,Q] = sum_k ac[a,k,m,P] ac[b,k,m,Q] (diagonal of A^T A per core).
__global__ void gram_diag_kernel(int ra, int n, int rb, const double* __restrict__ ac,
                                 double* __restrict__ G) {
  const long long total = (long long)ra * ra * n * rb * rb;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (int)total;
       e += gridDim.x * blockDim.x) {
    const int Q = (int)(e % rb);
    int t = e / rb;
    const int P = (int)(t % rb);
    t /= rb;
    const int m = (int)(t % n);
    t /= n;
    const int b = (int)(t % ra), a = (int)(t / ra);
    double s = 0.0;
    for (int k = 0; k < n; ++k)
      s = fma(ac[(((long long)a * n + k) * n + m) * rb + P], ac[(((long long)b * n + k) * n + m) * rb + Q], s);
    G[e] = s;
  }
}

// Jacobi diagonal of the normal block (tt_solver.py:234-236), zeros -> 1.
__global__ void normal_diag_kernel(int rx, int ra, int n, int ry, int rb,
                                   const double* __restrict__ pnl, const double* __restrict__ G,
                                   const double* __restrict__ pnr, double* __restrict__ out) {
  const long long total = (long long)rx * n * ry;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (int)total;
       e += gridDim.x * blockDim.x) {
    const int y = (int)(e % ry), m = (int)((e / ry) % n), x = (int)(e / ((long long)ry * n));
    double s = 0.0;
    for (int a = 0; a < ra; ++a)
      for (int b = 0; b < ra; ++b) {
        const double l = pnl[(((long long)x * ra + a) * ra + b) * rx + x];
        if (l == 0.0) continue;
        const double* g = G + ((((long long)a * ra + b) * n + m) * rb) * rb;
        double t = 0.0;
        for (int P = 0; P < rb; ++P)
          for (int Q = 0; Q < rb; ++Q)
            t = fma(g[P * rb + Q], pnr[(((long long)y * rb + P) * rb + Q) * ry + y], t);
        s = fma(l, t, s);
      }
    out[e] = fabs(s) > 1e-300 ? s : 1.0;
  }
}

// probe[0] += u.nu, probe[1] += c.u, probe[2] += #non-finite(u): one
// deterministic two-level reduction per candidate (tt_solver.py:332-334 and
// the isfinite check at :370/:398), read back together with the LU info.
// One launch: the last CTA to arrive (ticket) sums the per-CTA partials in
// CTA order and re-arms the ticket; when the host reads the probe buffer
// next (rt open) that CTA also publishes the buffer.
__global__ void probe_kernel(const double* __restrict__ u, const double* __restrict__ nu,
                             const double* __restrict__ c, int n, double* part,
                             unsigned* ticket, double* out, const double* buf, ReadTicket rt,
                             int* zero_info, double* gout) {
  // (zero_info: the solver flags behind the probe slots are cleared for the
  // solve that follows this probe — no memset on the stream)
  if (zero_info && blockIdx.x == 0 && threadIdx.x < 2) zero_info[threadIdx.x] = 0;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = u[i], v = nu[i], ci = c[i];
    s0 = fma(x, v, s0);
    s1 = fma(ci, x, s1);
    s2 += isfinite(x) ? 0.0 : 1.0;
    if (gout) gout[i] = v - ci;  // the candidate's residual gradient N u - c (update())
  }
  __shared__ double red[3][32];
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][warp] = s0;
    red[1][warp] = s1;
    red[2][warp] = s2;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[threadIdx.x][w];
    part[blockIdx.x * 3 + threadIdx.x] = t;
  }
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) t += __ldcg(part + b * 3 + threadIdx.x);
    out[threadIdx.x] = t;
  }
  if (threadIdx.x == 0) *ticket = 0u;
  if (rt.dst) {
    // the host reads the whole probe buffer next: publish it from here
    __syncthreads();
    publish_words(rt, reinterpret_cast<const unsigned*>(buf), 32);
  }
}

__global__ void nonfinite_kernel(const double* x, long long n, int* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) *flag = 1;
}

bool all_finite(const DTensor& t) {
  int* flag = reinterpret_cast<int*>(allocator().alloc(1));
  T2S2_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), stream()));
  {
    LaunchScope ls("check", 0, (double)t.size()*8);
    nonfinite_kernel<<<grid_of((long long)t.size()), 256, 0, stream()>>>(t.p, (long long)t.size(),
                                                                           flag);
  }
  T2S2_CHECK_LAUNCH();
  int h = 0;
  host_read(&h, flag, sizeof(int));
  allocator().release(reinterpret_cast<double*>(flag));
  return h == 0;
}

// -- contractions as permute-free batched GEMM chains ---------------------------
//
// The reference contracts with numpy.tensordot, which transposes operands
// into GEMM shape on every call.  Here each recurrence and local operator is
// a chain of 2-4 strided-batched GEMMs whose intermediates are laid out so
// that the next contraction reads them directly (op flags and batch strides
// replace every transposition).  The only extra layout is, per operator core
// ac[a, m, n, A] (row mode m, column mode n), the permuted copy
// acg[m, A, a, n] built once per solve: as a matrix [(m A), (a n)] it applies
// the core to a column-mode index, its transpose [(a n), (m A)] applies it to
// a row-mode index.  ac itself, read as [(a m), (n A)], covers the other two
// cases.  Interfaces keep the reference's layouts (tt_solver.py:94-96):
// pa (test, op, trial), pn (test, op, op, trial), pg (test, op, rhs),
// pb (test, rhs).

// C = op(A) op(B) over a strided batch (alpha 1, beta 0).
void bmm(bool ta, bool tb, int M, int N, int K, const double* A, int lda, long long sA,
         const double* B, int ldb, long long sB, double* C, int ldc, long long sC, int batch) {
  gemm_batched(ta, tb, M, N, K, 1.0, A, lda, sA, B, ldb, sB, 0.0, C, ldc, sC, batch);
}

DTensor op_layout(const DTensor& ac) { return permute(ac, {1, 3, 0, 2}); }  // (m, A, a, n)

// Dimensions of an operator core (ra, nm, nn, rA).
struct OpDims {
  int ra, nm, nn, rA;
  explicit OpDims(const DTensor& ac) : ra(ac.dim(0)), nm(ac.dim(1)), nn(ac.dim(2)), rA(ac.dim(3)) {}
};

// -- interface recurrences (tt_solver.py:98-151) -----------------------------
//
// Each recurrence adds its GEMMs to a GemmBatch at stages s0, s0+1, ...:
// the four families of a move (and the chains of successive cores) run as
// one program.  Outputs are allocated here; intermediates belong to the batch.

// pa[x,a,z] -> [X,A,Z] = sum pa[x,a,z] xc[x,m,X] ac[a,m,n,A] xc[z,n,Z]  (_left_a)
DTensor step_a_left(GemmBatch& gb, int s0, const DTensor& phi, const DTensor& xc, const DTensor& ac,
                    const DTensor& acg) {
  const OpDims o(ac);
  const int r0 = xc.dim(0), r1 = xc.dim(2);
  double* t1 = gb.temp({r0, o.ra, o.nn, r1});  // [x, a, n, Z]
  gb.add(s0, false, false, r0 * o.ra, o.nn * r1, r0, phi.p, r0, 0, xc.p, o.nn * r1, 0, t1, o.nn * r1, 0);
  double* t2 = gb.temp({r0, o.nm, o.rA, r1});  // [x, m, A, Z]
  gb.add(s0 + 1, false, false, o.nm * o.rA, r1, o.ra * o.nn, acg.p, o.ra * o.nn, 0, t1, r1,
         (long long)o.ra * o.nn * r1, t2, r1, (long long)o.nm * o.rA * r1, r0);
  DTensor out({r1, o.rA, r1});
  gb.add(s0 + 2, true, false, r1, o.rA * r1, r0 * o.nm, xc.p, r1, 0, t2, o.rA * r1, 0, out.p, o.rA * r1, 0);
  return out;
}

// pa[X,A,Z] -> [x,a,z]  (_right_a)
DTensor step_a_right(GemmBatch& gb, int s0, const DTensor& phi, const DTensor& xc, const DTensor& ac,
                     const DTensor& acg) {
  const OpDims o(ac);
  const int r0 = xc.dim(0), r1 = xc.dim(2);
  double* t1 = gb.temp({r0, o.nm, o.rA, r1});  // [x, m, A, Z]
  gb.add(s0, false, false, r0 * o.nm, o.rA * r1, r1, xc.p, r1, 0, phi.p, o.rA * r1, 0, t1, o.rA * r1, 0);
  double* t2 = gb.temp({r0, o.ra, o.nn, r1});  // [x, a, n, Z]
  gb.add(s0 + 1, true, false, o.ra * o.nn, r1, o.nm * o.rA, acg.p, o.ra * o.nn, 0, t1, r1,
         (long long)o.nm * o.rA * r1, t2, r1, (long long)o.ra * o.nn * r1, r0);
  DTensor out({r0, o.ra, r0});
  gb.add(s0 + 2, false, true, r0 * o.ra, r0, o.nn * r1, t2, o.nn * r1, 0, xc.p, o.nn * r1, 0, out.p, r0, 0);
  return out;
}

// pn[x,a1,a2,z] -> [X,A1,A2,Z]: both copies act on column modes, contracted
// over the shared row mode k (A^T A)  (_left_n)
DTensor step_n_left(GemmBatch& gb, int s0, const DTensor& phi, const DTensor& xc, const DTensor& ac,
                    const DTensor& acg) {
  const OpDims o(ac);
  const int r0 = xc.dim(0), r1 = xc.dim(2);
  double* t1 = gb.temp({r0, o.ra, o.ra, o.nn, r1});  // [x, a1, a2, n2, Z]
  gb.add(s0, false, false, r0 * o.ra * o.ra, o.nn * r1, r0, phi.p, r0, 0, xc.p, o.nn * r1, 0, t1,
         o.nn * r1, 0);
  double* t2 = gb.temp({r0, o.ra, o.nm, o.rA, r1});  // [x, a1, k, A2, Z]
  gb.add(s0 + 1, false, false, o.nm * o.rA, r1, o.ra * o.nn, acg.p, o.ra * o.nn, 0, t1, r1,
         (long long)o.ra * o.nn * r1, t2, r1, (long long)o.nm * o.rA * r1, r0 * o.ra);
  double* t3 = gb.temp({r0, o.nn, o.rA, o.rA, r1});  // [x, n1, A1, A2, Z]
  gb.add(s0 + 2, true, false, o.nn * o.rA, o.rA * r1, o.ra * o.nm, ac.p, o.nn * o.rA, 0, t2, o.rA * r1,
         (long long)o.ra * o.nm * o.rA * r1, t3, o.rA * r1, (long long)o.nn * o.rA * o.rA * r1, r0);
  DTensor out({r1, o.rA, o.rA, r1});
  gb.add(s0 + 3, true, false, r1, o.rA * o.rA * r1, r0 * o.nn, xc.p, r1, 0, t3, o.rA * o.rA * r1, 0,
         out.p, o.rA * o.rA * r1, 0);
  return out;
}

// pn[X,A1,A2,Z] -> [x,a1,a2,z]  (_right_n)
DTensor step_n_right(GemmBatch& gb, int s0, const DTensor& phi, const DTensor& xc, const DTensor& ac,
                     const DTensor& acg) {
  const OpDims o(ac);
  const int r0 = xc.dim(0), r1 = xc.dim(2);
  const int q = o.rA * o.rA * r1;
  double* t1 = gb.temp({r0, o.nn, o.rA, o.rA, r1});  // [x, n1, A1, A2, Z]
  gb.add(s0, false, false, r0 * o.nn, q, r1, xc.p, r1, 0, phi.p, q, 0, t1, q, 0);
  double* t2 = gb.temp({r0, o.ra, o.nm, o.rA, r1});  // [x, a1, k, A2, Z]
  gb.add(s0 + 1, false, false, o.ra * o.nm, o.rA * r1, o.nn * o.rA, ac.p, o.nn * o.rA, 0, t1, o.rA * r1,
         (long long)o.nn * q, t2, o.rA * r1, (long long)o.ra * o.nm * o.rA * r1, r0);
  double* t3 = gb.temp({r0, o.ra, o.ra, o.nn, r1});  // [x, a1, a2, n2, Z]
  gb.add(s0 + 2, true, false, o.ra * o.nn, r1, o.nm * o.rA, acg.p, o.ra * o.nn, 0, t2, r1,
         (long long)o.nm * o.rA * r1, t3, r1, (long long)o.ra * o.nn * r1, r0 * o.ra);
  DTensor out({r0, o.ra, o.ra, r0});
  gb.add(s0 + 3, false, true, r0 * o.ra * o.ra, r0, o.nn * r1, t3, o.nn * r1, 0, xc.p, o.nn * r1, 0,
         out.p, r0, 0);
  return out;
}

// pg[x,a,b] -> [X,A,B] = sum pg xc[x,n,X] ac[a,k,n,A] bc[b,k,B]  (_left_g)
DTensor step_g_left(GemmBatch& gb, int s0, const DTensor& phi, const DTensor& xc, const DTensor& ac,
                    const DTensor& bc) {
  const OpDims o(ac);
  const int r0 = xc.dim(0), r1 = xc.dim(2), b0 = bc.dim(0), b1 = bc.dim(2);
  double* t1 = gb.temp({r0, o.ra, o.nm, b1});  // [x, a, k, B]
  gb.add(s0, false, false, r0 * o.ra, o.nm * b1, b0, phi.p, b0, 0, bc.p, o.nm * b1, 0, t1, o.nm * b1, 0);
  double* t2 = gb.temp({r0, o.nn, o.rA, b1});  // [x, n, A, B]
  gb.add(s0 + 1, true, false, o.nn * o.rA, b1, o.ra * o.nm, ac.p, o.nn * o.rA, 0, t1, b1,
         (long long)o.ra * o.nm * b1, t2, b1, (long long)o.nn * o.rA * b1, r0);
  DTensor out({r1, o.rA, b1});
  gb.add(s0 + 2, true, false, r1, o.rA * b1, r0 * o.nn, xc.p, r1, 0, t2, o.rA * b1, 0, out.p, o.rA * b1, 0);
  return out;
}

// pg[X,A,B] -> [x,a,b]  (_right_g)
DTensor step_g_right(GemmBatch& gb, int s0, const DTensor& phi, const DTensor& xc, const DTensor& ac,
                     const DTensor& bc) {
  const OpDims o(ac);
  const int r0 = xc.dim(0), r1 = xc.dim(2), b0 = bc.dim(0), b1 = bc.dim(2);
  double* t1 = gb.temp({r0, o.nn, o.rA, b1});  // [x, n, A, B]
  gb.add(s0, false, false, r0 * o.nn, o.rA * b1, r1, xc.p, r1, 0, phi.p, o.rA * b1, 0, t1, o.rA * b1, 0);
  double* t2 = gb.temp({r0, o.ra, o.nm, b1});  // [x, a, k, B]
  gb.add(s0 + 1, false, false, o.ra * o.nm, b1, o.nn * o.rA, ac.p, o.nn * o.rA, 0, t1, b1,
         (long long)o.nn * o.rA * b1, t2, b1, (long long)o.ra * o.nm * b1, r0);
  DTensor out({r0, o.ra, b0});
  gb.add(s0 + 2, false, true, r0 * o.ra, b0, o.nm * b1, t2, o.nm * b1, 0, bc.p, o.nm * b1, 0, out.p, b0, 0);
  return out;
}

// pb[x,b] -> [X,B]  (_left_b)
DTensor step_b_left(GemmBatch& gb, int s0, const DTensor& phi, const DTensor& xc, const DTensor& bc) {
  const int r0 = xc.dim(0), n = xc.dim(1), r1 = xc.dim(2), b0 = bc.dim(0), b1 = bc.dim(2);
  double* t1 = gb.temp({r0, n, b1});
  gb.add(s0, false, false, r0, n * b1, b0, phi.p, b0, 0, bc.p, n * b1, 0, t1, n * b1, 0);
  DTensor out({r1, b1});
  gb.add(s0 + 1, true, false, r1, b1, r0 * n, xc.p, r1, 0, t1, b1, 0, out.p, b1, 0);
  return out;
}

// pb[X,B] -> [x,b]  (_right_b)
DTensor step_b_right(GemmBatch& gb, int s0, const DTensor& phi, const DTensor& xc, const DTensor& bc) {
  const int r0 = xc.dim(0), n = xc.dim(1), r1 = xc.dim(2), b0 = bc.dim(0), b1 = bc.dim(2);
  double* t1 = gb.temp({r0, n, b1});
  gb.add(s0, false, false, r0 * n, b1, r1, xc.p, r1, 0, phi.p, b1, 0, t1, b1, 0);
  DTensor out({r0, b0});
  gb.add(s0 + 1, false, true, r0, b0, n * b1, t1, n * b1, 0, bc.p, n * b1, 0, out.p, b0, 0);
  return out;
}

// -- local systems (tt_solver.py:155-246) -------------------------------------

// (x, m, y) = sum pbl[x,B] bc[B,m,C] pbr[y,C]  (_gal_rhs)
DTensor galerkin_rhs(GemmBatch& gb, int s0, const DTensor& pbl, const DTensor& bc, const DTensor& pbr) {
  const int rx = pbl.dim(0), b0 = bc.dim(0), n = bc.dim(1), b1 = bc.dim(2), ry = pbr.dim(0);
  double* t1 = gb.temp({rx, n, b1});
  gb.add(s0, false, false, rx, n * b1, b0, pbl.p, b0, 0, bc.p, n * b1, 0, t1, n * b1, 0);
  DTensor out({rx, n, ry});
  gb.add(s0 + 1, false, true, rx * n, ry, b1, t1, b1, 0, pbr.p, b1, 0, out.p, ry, 0);
  return out;
}

// projected A^T b (_ls_rhs)
DTensor normal_rhs(GemmBatch& gb, int s0, const DTensor& pgl, const DTensor& ac, const DTensor& bc,
                   const DTensor& pgr) {
  const OpDims o(ac);
  const int rx = pgl.dim(0), b0 = bc.dim(0), b1 = bc.dim(2), ry = pgr.dim(0);
  double* t1 = gb.temp({rx, o.ra, o.nm, b1});  // [x, a, k, C]
  gb.add(s0, false, false, rx * o.ra, o.nm * b1, b0, pgl.p, b0, 0, bc.p, o.nm * b1, 0, t1, o.nm * b1, 0);
  double* t2 = gb.temp({rx, o.nn, o.rA, b1});  // [x, m, A, C]
  gb.add(s0 + 1, true, false, o.nn * o.rA, b1, o.ra * o.nm, ac.p, o.nn * o.rA, 0, t1, b1,
         (long long)o.ra * o.nm * b1, t2, b1, (long long)o.nn * o.rA * b1, rx);
  DTensor out({rx, o.nn, ry});
  gb.add(s0 + 2, false, true, rx * o.nn, ry, o.rA * b1, t2, o.rA * b1, 0, pgr.p, o.rA * b1, 0, out.p, ry, 0);
  return out;
}

// Local operators applied to raw device vectors (the Krylov matvecs and the
// candidate scores); scratch is sized once per local system.
struct NormalOp {  // (A^T A)-projected block (_ls_matvec / _LsApply)
  const DTensor &pnl, &ac, &acg, &pnr;
  OpDims o;
  int rx, rz, ry, rw;
  DTensor t1, t2, t3;
  NormalOp(const DTensor& l, const DTensor& a, const DTensor& ag, const DTensor& r)
      : pnl(l), ac(a), acg(ag), pnr(r), o(a), rx(l.dim(0)), rz(l.dim(3)), ry(r.dim(0)),
        rw(r.dim(3)),
        t1({rx, o.ra, o.ra, o.nn, rw}), t2({rx, o.ra, o.nm, o.rA, rw}),
        t3({rx, o.nn, o.rA, o.rA, rw}) {}
  // 4 stages from s0; the scratch is shared, so one application per batch
  void add(GemmBatch& gb, int s0, const double* u, double* out) {
    gb.add(s0, false, false, rx * o.ra * o.ra, o.nn * rw, rz, pnl.p, rz, 0, u, o.nn * rw, 0, t1.p,
           o.nn * rw, 0);
    gb.add(s0 + 1, false, false, o.nm * o.rA, rw, o.ra * o.nn, acg.p, o.ra * o.nn, 0, t1.p, rw,
           (long long)o.ra * o.nn * rw, t2.p, rw, (long long)o.nm * o.rA * rw, rx * o.ra);
    gb.add(s0 + 2, true, false, o.nn * o.rA, o.rA * rw, o.ra * o.nm, ac.p, o.nn * o.rA, 0, t2.p,
           o.rA * rw, (long long)o.ra * o.nm * o.rA * rw, t3.p, o.rA * rw,
           (long long)o.nn * o.rA * o.rA * rw, rx);
    const int q = o.rA * o.rA * rw;
    gb.add(s0 + 3, false, true, rx * o.nn, ry, q, t3.p, q, 0, pnr.p, q, 0, out, ry, 0);
  }
  void operator()(const double* u, double* out) {
    GemmBatch gb;
    add(gb, 0, u, out);
    gb.run();
  }
  DTensor apply(const DTensor& u) {
    DTensor out({rx, o.nn, ry});
    (*this)(u.p, out.p);
    return out;
  }
};

struct GalerkinOp {  // Galerkin block (_gal_matvec)
  const DTensor &pal, &acg, &par;
  OpDims o;
  int rx, rX, ry, rY;
  DTensor t1, t2;
  GalerkinOp(const DTensor& l, const DTensor& a, const DTensor& ag, const DTensor& r)
      : pal(l), acg(ag), par(r), o(a), rx(l.dim(0)), rX(l.dim(2)), ry(r.dim(0)), rY(r.dim(2)),
        t1({rx, o.ra, o.nn, rY}), t2({rx, o.nm, o.rA, rY}) {}
  // 3 stages from 0; the scratch is shared, so one application per batch
  void add(GemmBatch& gb, const double* u, double* out) {
    gb.add(0, false, false, rx * o.ra, o.nn * rY, rX, pal.p, rX, 0, u, o.nn * rY, 0, t1.p, o.nn * rY, 0);
    gb.add(1, false, false, o.nm * o.rA, rY, o.ra * o.nn, acg.p, o.ra * o.nn, 0, t1.p, rY,
           (long long)o.ra * o.nn * rY, t2.p, rY, (long long)o.nm * o.rA * rY, rx);
    gb.add(2, false, true, rx * o.nm, ry, o.rA * rY, t2.p, o.rA * rY, 0, par.p, o.rA * rY, 0, out, ry, 0);
  }
};

// Column-major normal-equation block N[(x,m,y),(z,n,w)] (tt_solver.py:239-246).
DTensor normal_matrix(const DTensor& pnl, const DTensor& ac, const DTensor& pnr) {
  DTensor g = tensordot(ac, {1}, ac, {1});     // (a, m, P, b, n, Q)
  DTensor t = tensordot(pnl, {1, 2}, g, {0, 3});  // (x, z, m, P, n, Q)
  t = tensordot(t, {3, 5}, pnr, {1, 2});       // (x, z, m, n, y, w)
  return permute(t, {1, 3, 5, 0, 2, 4});       // (z, n, w | x, m, y): column-major
}

DTensor normal_diagonal(const DTensor& pnl, const DTensor& ac, const DTensor& pnr) {
  const int rx = pnl.dim(0), ra = ac.dim(0), n = ac.dim(1), rb = ac.dim(3), ry = pnr.dim(0);
  DTensor G({ra, ra, n, rb, rb});
  {
    LaunchScope ls("normal_diag", 2.0*G.size()*n, 0);
    gram_diag_kernel<<<grid_of((long long)G.size()), 256, 0, stream()>>>(ra, n, rb, ac.p, G.p);
  }
  DTensor out({rx, n, ry});
  {
    LaunchScope ls("normal_diag", 2.0*out.size()*ra*ra*rb*rb, 0);
    normal_diag_kernel<<<grid_of((long long)out.size()), 256, 0, stream()>>>(rx, ra, n, ry, rb, pnl.p,
                                                                            G.p, pnr.p, out.p);
  }
  T2S2_CHECK_LAUNCH();
  return out;
}

DTensor galerkin_matrix(const DTensor& pal, const DTensor& ac, const DTensor& par) {
  const int rx = pal.dim(0), ra = pal.dim(1), n = ac.dim(1), rb = ac.dim(3), ry = par.dim(0);
  const long long N = (long long)rx * n * ry;
  DTensor B({(int)N, (int)N});
  {
    LaunchScope ls("galerkin_build", 2.0*(double)N*N*ra*(rb+1), 8.0*(double)N*N);
    const size_t smem = sizeof(double) * ((size_t)ra * n * ry + (size_t)rx * ra * rx);
    if (smem <= 96 * 1024) {
      max_dynamic_smem((const void*)galerkin_factored_kernel, 96 * 1024);
      galerkin_factored_kernel<<<n * ry, 256, smem, stream()>>>(rx, n, ry, ra, rb, pal.p, ac.p, par.p,
                                                               B.p);
    } else {
      galerkin_matrix_kernel<<<dim3(ceil_div(N, 256), N < 4096 ? (int)N : 4096), 256, 0, stream()>>>(
          rx, n, ry, ra, rb, pal.p, ac.p, par.p, B.p);
    }
  }
  T2S2_CHECK_LAUNCH();
  return B;
}

// Dense direct solve of a column-major N x N system; the LU info (0, or
// 1 + first zero pivot) lands in *info_dev and is read back by the caller.
// Partial-pivoting dense solve (the reference's numpy.linalg.solve).
// info_dev[1] (set to 1, never cleared here) records a row interchange.
// consume: the right-hand side is not needed afterwards — it becomes the
// solution buffer instead of being copied (the caller recomputes it in the
// rare case it solves the same system again).
void dense_solve_pivoted(DTensor& M, DTensor& rhs, DTensor& out, int* info_dev, bool consume = false) {
  const int N = M.dim(0);
  int* ipiv = reinterpret_cast<int*>(allocator().alloc((N + 1) / 2 + 1));
  if (consume)
    out = std::move(rhs);
  else
    out = rhs.clone();
  if (!lu_solve_fused(N, M.p, out.p, ipiv, info_dev, info_dev + 1)) {
    lu_factor(N, M.p, ipiv, info_dev);
    lu_solve(N, M.p, ipiv, out.p);
  }
  allocator().release(reinterpret_cast<double*>(ipiv));
}

// Local dense solve: the verified no-pivot LU first (identical factors when
// partial pivoting would not interchange rows); *info_dev == -1 afterwards
// means it declined and the caller must rebuild M and call
// dense_solve_pivoted.
void dense_solve(DTensor& M, DTensor& rhs, DTensor& out, int* info_dev, bool consume = false) {
  if (consume)
    out = std::move(rhs);
  else
    out = rhs.clone();
  if (gj_solve_nopivot(M.dim(0), M.p, out.p, info_dev)) return;
  // not applicable (nothing launched, the buffer is untouched): the pivoting kernel
  DTensor again = std::move(out);
  dense_solve_pivoted(M, again, out, info_dev, true);
}

// Which dense kernel a kind of local system tries first.  The no-pivot
// Gauss-Jordan kernel declines (in its first panels) when partial pivoting
// would interchange rows; after four declines in a row the pivoting kernel
// runs directly, and as soon as one of its solves makes no interchange
// (info[1] == 0: the no-pivot kernel would have accepted) the no-pivot
// kernel is tried first again.  Results are those of the kernel that
// accepts, so the policy only removes declined launches.
struct PivotPolicy {
  int declines = 0;
  bool pivot_first = false;
  void solve(DTensor& M, DTensor& rhs, DTensor& out, int* info_dev, bool consume = false) const {
    if (pivot_first)
      dense_solve_pivoted(M, rhs, out, info_dev, consume);
    else
      dense_solve(M, rhs, out, info_dev, consume);
  }
  void observe(int info, int swapped) {  // after the first attempt of a system
    if (pivot_first) {
      if (info == 0 && swapped == 0) pivot_first = false, declines = 0;
    } else if (info == -1) {
      if (++declines >= 4) pivot_first = true;
    } else if (info == 0) {
      declines = 0;
    }
  }
};

// Minimum-norm least squares of a singular column-major N x N system, the
// reference's fallback when numpy.linalg.solve raises (tt_solver.py:362,
// :395 call numpy.linalg.lstsq with rcond=None: cutoff eps*N*s_max).
void lstsq_dense(const DTensor& Mcm, const DTensor& rhs, DTensor& out) {
  const int N = Mcm.dim(0);
  DTensor U, sv, Vt;
  svd_thin(N, N, Mcm.p, U, sv, Vt);  // column-major M read as row-major M^T = U S Vt
  const int k = sv.dim(0);
  std::vector<double> hs(k);
  to_host(hs.data(), sv.p, k);
  const double cutoff = 2.220446049250313e-16 * N * (k ? hs[0] : 0.0);
  std::vector<double> inv(k);
  for (int i = 0; i < k; ++i) inv[i] = hs[i] > cutoff ? 1.0 / hs[i] : 0.0;
  DTensor dinv({k}), y({k, 1});
  to_device(dinv.p, inv.data(), k);
  // M = Vt^T S U^T  =>  x = U diag(1/s) Vt b
  gemm(false, false, k, 1, N, 1.0, Vt.p, N, rhs.p, 1, 0.0, y.p, 1);
  scale_rows(y.p, k, 1, 1, dinv.p);
  out = DTensor(rhs.shape);
  gemm(false, false, N, 1, k, 1.0, U.p, k, y.p, 1, 0.0, out.p, 1);
}

// Device scratch for candidate scores: 3 doubles per probe slot + LU info.
struct Probe {
  DTensor buf{std::vector<int>{16}};  // 4 slots x 3, LU info at [12], ticket at [14]
  Probe() { T2S2_CUDA(cudaMemsetAsync(buf.p, 0, 16 * sizeof(double), stream())); }
  int* info() { return reinterpret_cast<int*>(buf.p + 12); }
  unsigned* ticket() { return reinterpret_cast<unsigned*>(buf.p + 14); }
  // info()[0]: LU info; info()[1]: a pivoted solve interchanged rows
  void clear_info() { T2S2_CUDA(cudaMemsetAsync(info(), 0, 2 * sizeof(int), stream())); }
  ReadTicket open;  // the last probe launch publishes the buffer itself
  bool is_open = false;
  // then_read: read() follows this launch with nothing that reads in between
  // grad: also write N u - c (the projected residual gradient of this candidate)
  void run(int slot, const DTensor& u, const DTensor& nu, const DTensor& c, bool then_read,
           bool zero_info = false, DTensor* grad = nullptr) {
    const int n = (int)u.size();
    if (grad) *grad = DTensor(u.shape);
    if (then_read) {
      open = read_open(16 * sizeof(double));
      is_open = true;
    }
    int nb = (n + 255) / 256;
    if (nb > 148) nb = 148;
    double* part = allocator().alloc((size_t)nb * 3);
    {
      LaunchScope ls("reduce", 4.0 * n, 24.0 * n);
      probe_kernel<<<nb, 256, 0, stream()>>>(u.p, nu.p, c.p, n, part, ticket(), buf.p + 3 * slot, buf.p,
                                             then_read ? open : ReadTicket{}, zero_info ? info() : nullptr,
                                             grad ? grad->p : nullptr);
    }
    T2S2_CHECK_LAUNCH();
    allocator().release(part);
  }
  // one read-back: h[3*slot + {0,1,2}], info at h_info, interchange flag
  void read(double* h, int* h_info, int* h_swapped = nullptr) {
    double tmp[16];
    if (is_open) {
      read_close(tmp, sizeof tmp, open);
      is_open = false;
    } else {
      host_read(tmp, buf.p, sizeof tmp);
    }
    for (int i = 0; i < 12; ++i) h[i] = tmp[i];
    *h_info = reinterpret_cast<int*>(tmp + 12)[0];
    if (h_swapped) *h_swapped = reinterpret_cast<int*>(tmp + 12)[1];
  }
};

// -- splits with enrichment (tt_solver.py:261-302) ------------------------------

struct Split {
  DTensor core, carry;
  DTensor next;  // the neighbour core's new buffer (its enrichment part zeroed), if asked for
  int extra = 0;
};

std::vector<double> host_vec(const DTensor& s) {
  std::vector<double> h(s.size());
  to_host(h.data(), s.p, s.size());
  return h;
}

double vec_norm(const std::vector<double>& s) {
  double a = 0.0;
  for (double v : s) a += v * v;
  return std::sqrt(a);
}

int count_significant(const std::vector<double>& zs) {
  const double lead = zs.empty() ? 0.0 : zs[0];
  const double thr = 1e-14 * (lead > 1e-300 ? lead : 1e-300);
  int nz = 0;
  for (double v : zs) nz += v > thr;
  return nz;
}

// Split of a solved core with enrichment from the residual gradient
// (tt_solver.py:261-302).  The truncation rank is decided on the device and
// the projection of the gradient is masked with it, so the core's singular
// values, the gradient's singular values and the rank travel to the host in
// ONE read-back (was two synchronising reads).
struct SplitSync {
  DTensor keep_mask;  // [0] = keep, [1..kk] = mask
  int kk;
  KeepArgs args;
  // kk = min(m, n) of the core's unfolding; the SVD kernel fills keep_mask (svd_thin's keep argument)
  SplitSync(int kk_, const SolverConfig& cfg, int d) : keep_mask({1 + kk_}), kk(kk_) {
    args = KeepArgs{cfg.rounding_tol, std::sqrt((double)(d - 1 > 1 ? d - 1 : 1)), cfg.max_rank, keep_mask.p,
                    keep_mask.p + 1};
  }
  const double* mask() const { return keep_mask.p + 1; }
  // read keep, s and (optionally) zs together
  int read(const DTensor& s, const DTensor* zs, std::vector<double>& hz) {
    const int zk = zs ? zs->dim(0) : 0;
    std::vector<double> h(1 + kk + zk);
    host_read_gather(h.data(), {{keep_mask.p, 1}, {s.p, (size_t)kk}, {zk ? zs->p : nullptr, (size_t)zk}});
    hz.assign(h.begin() + 1 + kk, h.end());
    return (int)h[0];
  }
};

// neighbour: the core the carry goes to; out.next is its new buffer
// (keep + extra, n', r'), rows of the enrichment part zeroed.  Carry, core and
// that zero fill are ONE launch (split_finish).
Split split_forward(const DTensor& u, DTensor* grad, const SolverConfig& cfg, int d,
                    const DTensor* neighbour = nullptr) {
  const int r0 = u.dim(0), n = u.dim(1), r1 = u.dim(2), m = r0 * n;
  DTensor U, s, Vt;
  const int kk = m < r1 ? m : r1;
  SplitSync sync(kk, cfg, d);
  svd_thin(m, r1, u.p, U, s, Vt, nullptr, &sync.args);  // and the truncation rank
  trace_buffer("split_forward s", s.p, s.size());
  const bool enrich = cfg.enrichment_rank > 0 && grad;
  DTensor zu, zs, zvt;
  int zk = 0;
  if (enrich) {
    // z = g - U_keep U_keep^T g, with U_keep = U diag(mask)
    const int gc = (int)(grad->size() / m);
    DTensor z = std::move(*grad);  // the gradient is consumed here
    DTensor tmp({kk, gc});
    {
      GemmBatch gb;  // tmp = diag(mask) U^T z, then z -= U tmp: one launch
      gb.add(0, true, false, kk, gc, m, U.p, kk, 0, z.p, gc, 0, tmp.p, gc, 0);
      gb.scale_last(sync.mask(), nullptr);
      gb.add(1, false, false, m, gc, kk, U.p, kk, 0, tmp.p, gc, 0, z.p, gc, 0, 1, -1.0, 1.0);
      gb.run();
    }
    svd_thin(m, gc, z.p, zu, zs, zvt);
    zk = zs.dim(0);
  }
  std::vector<double> hz;
  const int keep = sync.read(s, enrich ? &zs : nullptr, hz);
  Split out;
  out.carry = DTensor({keep, r1});
  if (enrich && keep < cfg.max_rank) {
    int nz = count_significant(hz);
    int extra = cfg.enrichment_rank;
    if (cfg.max_rank - keep < extra) extra = cfg.max_rank - keep;
    if (nz < extra) extra = nz;
    out.extra = extra > 0 ? extra : 0;
  }
  out.core = DTensor({r0, n, keep + out.extra});
  SplitFinish f{};
  f.d0 = out.carry.p, f.s0 = Vt.p, f.ldd0 = r1, f.lds0 = r1, f.rows0 = keep, f.cols0 = r1, f.rs = s.p;
  f.d1 = out.core.p, f.a1 = U.p, f.b1 = zu.p, f.ldd1 = keep + out.extra, f.lda1 = kk, f.ldb1 = zk;
  f.c1 = keep, f.c2 = out.extra, f.rows1 = m;
  if (neighbour) {
    const int rest = (int)(neighbour->size() / r1);
    out.next = DTensor({keep + out.extra, neighbour->dim(1), neighbour->dim(2)});
    f.d2 = out.next.p + (size_t)keep * rest;
    f.n2 = (long long)out.extra * rest;
  }
  split_finish(f);
  return out;
}

Split split_backward(const DTensor& u, DTensor* grad, const SolverConfig& cfg, int d,
                     const DTensor* neighbour = nullptr) {
  const int r0 = u.dim(0), n = u.dim(1), r1 = u.dim(2), cols = n * r1;
  DTensor U, s, Vt;
  const int kk = r0 < cols ? r0 : cols;
  SplitSync sync(kk, cfg, d);
  svd_thin(r0, cols, u.p, U, s, Vt, nullptr, &sync.args);  // U r0 x kk, Vt kk x cols; and the rank
  trace_buffer("split_backward s", s.p, s.size());
  const bool enrich = cfg.enrichment_rank > 0 && grad;
  DTensor zu, zs, zvt;
  if (enrich) {
    // z = g - g Vt_keep^T Vt_keep, with Vt_keep = diag(mask) Vt
    const int gr = (int)(grad->size() / cols);
    DTensor z = std::move(*grad);  // the gradient is consumed here
    DTensor tmp({gr, kk});
    {
      GemmBatch gb;  // tmp = z Vt^T diag(mask), then z -= tmp Vt: one launch
      gb.add(0, false, true, gr, kk, cols, z.p, cols, 0, Vt.p, cols, 0, tmp.p, kk, 0);
      gb.scale_last(nullptr, sync.mask());
      gb.add(1, false, false, gr, cols, kk, tmp.p, kk, 0, Vt.p, cols, 0, z.p, cols, 0, 1, -1.0, 1.0);
      gb.run();
    }
    svd_thin(gr, cols, z.p, zu, zs, zvt);
  }
  std::vector<double> hz;
  const int keep = sync.read(s, enrich ? &zs : nullptr, hz);
  Split out;
  out.carry = DTensor({r0, keep});
  if (enrich && keep < cfg.max_rank) {
    int nz = count_significant(hz);
    int extra = cfg.enrichment_rank;
    if (cfg.max_rank - keep < extra) extra = cfg.max_rank - keep;
    if (nz < extra) extra = nz;
    out.extra = extra > 0 ? extra : 0;
  }
  out.core = DTensor({keep + out.extra, n, r1});
  SplitFinish f{};
  f.d0 = out.carry.p, f.s0 = U.p, f.ldd0 = keep, f.lds0 = kk, f.rows0 = r0, f.cols0 = keep, f.cs = s.p;
  // the core: keep rows of Vt, then extra rows of the gradient's Vt — two contiguous pieces
  f.d1 = out.core.p, f.a1 = Vt.p, f.b1 = zvt.p, f.rows1 = 1;
  f.c1 = keep * cols, f.c2 = out.extra * cols;
  if (neighbour) {
    out.next = DTensor({neighbour->dim(0), neighbour->dim(1), keep + out.extra});
    if (out.extra > 0) {
      f.d2 = out.next.p;
      f.n2 = (long long)out.next.size();
    }
  }
  split_finish(f);
  return out;
}

// -- residual (tt_solver.py:305-329) ----------------------------------------------

double measure_residual(const Train& A, const std::vector<DTensor>& acg, std::vector<DTensor>& x,
                        const Train& rhs, double bnorm) {
  const int d = A.d();
  // both Gram chains in one program (4 stages per core for <Ax,Ax>, 3 for <Ax,b>)
  GemmBatch gb;
  DTensor phi({1, 1, 1, 1}), psi({1, 1, 1});
  fill_many({{phi.p, 1}, {psi.p, 1}}, 1.0);
  std::vector<DTensor> keep;
  for (int l = 0; l < d; ++l) {
    DTensor nphi = step_n_left(gb, 4 * l, phi, x[l], A.cores[l], acg[l]);
    DTensor npsi = step_g_left(gb, 4 * l, psi, x[l], A.cores[l], rhs.cores[l]);
    keep.push_back(std::move(phi));
    keep.push_back(std::move(psi));
    phi = std::move(nphi);
    psi = std::move(npsi);
  }
  gb.run();
  keep.clear();
  double hv[2];
  host_read_gather(hv, {{phi.p, 1}, {psi.p, 1}});
  const double axax = hv[0], axb = hv[1];
  const double est_sq = axax - 2.0 * axb + bnorm * bnorm;
  const double est = std::sqrt(est_sq > 0.0 ? est_sq : 0.0) / bnorm;
  if (est_sq <= 0.0 || est < 1e-6) {
    Train xt;  // the cores are lent to a train for the apply and taken back
    xt.rows = rhs.rows;
    xt.cores = std::move(x);
    Train diff;
    try {
      diff = tt_add(tt_apply(A, xt), rhs, 1.0, -1.0);
    } catch (...) {
      x = std::move(xt.cores);
      throw;
    }
    x = std::move(xt.cores);
    return tt_norm(diff) / bnorm;
  }
  return est;
}

// -- sweep state -------------------------------------------------------------------

struct Sweep {
  const Train& A;
  const Train& rhs;
  const SolverConfig& cfg;
  int d;
  int gal_rejects = 0;
  int gal_cap;
  std::vector<DTensor> la, ln, lg, lb, ra, rn, rg, rb;
  const std::vector<DTensor>& acg;  // per-core operator layout (m, A, a, n), cached in the train
  static const std::vector<DTensor>& layout_of(const Train& a) {
    bool valid = a.layout_of.size() == a.cores.size() && !a.cores.empty();
    for (size_t l = 0; valid && l < a.cores.size(); ++l) valid = a.layout_of[l] == a.cores[l].p;
    if (!valid) {
      a.solver_layout.clear();
      a.layout_of.clear();
      for (const DTensor& ac : a.cores) {
        a.solver_layout.push_back(op_layout(ac));
        a.layout_of.push_back(ac.p);
      }
    }
    return a.solver_layout;
  }
  Sweep(const Train& a, const Train& b, const SolverConfig& c)
      : A(a), rhs(b), cfg(c), d(a.d()), gal_cap(2 * a.d()),
        la(d + 1), ln(d + 1), lg(d + 1), lb(d + 1), ra(d + 1), rn(d + 1), rg(d + 1), rb(d + 1),
        acg(layout_of(a)) {}

  Probe probe;
  PivotPolicy pol_gal, pol_ls;  // Galerkin / normal-equation systems
  bool gal_direct = false;  // the last update's Galerkin candidate came from a dense solve

  // Guarded update of core l (tt_solver.py:337-422).  Candidate scores
  // q = u^T N u - 2 c^T u, the finiteness checks and the LU info travel to
  // the host together: one read-back per candidate pair.
  void update(int l, std::vector<DTensor>& cores, double current_res, DTensor& best,
              DTensor& grad, int& choice) {
    const DTensor& ac = A.cores[l];
    const DTensor& bc = rhs.cores[l];
    const DTensor& u_old = cores[l];
    const long long size = (long long)u_old.size();
    NormalOp nop(ln[l], ac, acg[l], rn[l + 1]);
    DTensor nu_old({nop.rx, nop.o.nn, nop.ry});
    DTensor c_gal, c_ls;
    {
      GemmBatch gb;
      c_gal = galerkin_rhs(gb, 0, lb[l], bc, rb[l + 1]);
      c_ls = normal_rhs(gb, 0, lg[l], ac, bc, rg[l + 1]);
      nop.add(gb, 0, u_old.p, nu_old.p);
      gb.run();
    }
    // the Galerkin right-hand side again (the direct solve consumes it): same program, same bits
    auto regal = [&]() {
      GemmBatch gb;
      DTensor c = galerkin_rhs(gb, 0, lb[l], bc, rb[l + 1]);
      gb.run();
      return c;
    };
    probe.run(0, u_old, nu_old, c_ls, false, true);  // and clears the solver flags
    const bool direct = cfg.local_solver == 1 || (cfg.local_solver == 0 && size <= cfg.local_direct_size);
    const double inner_rtol = std::fmax(cfg.inner_tol_factor * current_res, 1e-12);
    const bool try_gal = gal_rejects < gal_cap;
    gal_direct = try_gal && direct;
    DTensor u_gal, nu_gal;
    DTensor g_gal;  // N u_gal - c_ls, written by the Galerkin candidate's probe
    if (try_gal) {
      if (direct) {
        DTensor B = galerkin_matrix(la[l], ac, ra[l + 1]);
        pol_gal.solve(B, c_gal, u_gal, probe.info(), true);  // c_gal becomes u_gal
      } else {
        // scipy gmres(x0=u_old, rtol, atol=0, restart=40, maxiter=10)
        u_gal = u_old.clone();
        GalerkinOp gop(la[l], ac, acg[l], ra[l + 1]);
        gmres([&](GemmBatch& gb, const double* in, double* out) { gop.add(gb, in, out); }, (int)size, c_gal.p,
              u_gal.p, inner_rtol, 40, 10);
      }
      u_gal.view(u_old.shape);
      trace_buffer("update u_gal", u_gal.p, u_gal.size());
      nu_gal = nop.apply(u_gal);
      probe.run(1, u_gal, nu_gal, c_ls, true, false, &g_gal);
    }
    double h[12];
    int info = 0, swapped = 0;
    probe.read(h, &info, &swapped);
    if (try_gal && direct) pol_gal.observe(info, swapped);
    if (try_gal && direct && info == -1) {
      // the block needs row interchanges: rebuild it, partial pivoting
      DTensor B = galerkin_matrix(la[l], ac, ra[l + 1]);
      c_gal = regal();
      probe.clear_info();
      dense_solve_pivoted(B, c_gal, u_gal, probe.info(), true);
      u_gal.view(u_old.shape);
      nu_gal = nop.apply(u_gal);
      probe.run(1, u_gal, nu_gal, c_ls, true, false, &g_gal);
      probe.read(h, &info);
    }
    if (try_gal && direct && info != 0) {
      // singular Galerkin block: numpy.linalg.lstsq fallback (tt_solver.py:362)
      DTensor B = galerkin_matrix(la[l], ac, ra[l + 1]);
      c_gal = regal();
      lstsq_dense(B, c_gal, u_gal);
      u_gal.view(u_old.shape);
      nu_gal = nop.apply(u_gal);
      probe.clear_info();
      probe.run(1, u_gal, nu_gal, c_ls, true, false, &g_gal);
      probe.read(h, &info);
    }
    const double q_old = h[0] - 2.0 * h[1];
    double best_q = q_old;
    choice = 0;
    DTensor nu_best;
    // a singular local matrix (numpy LinAlgError) or a non-finite candidate
    // is no candidate (tt_solver.py:359-372)
    if (try_gal && info == 0 && h[5] == 0.0) {
      const double q_gal = h[3] - 2.0 * h[4];
      if (q_gal <= best_q) {
        best_q = q_gal;
        choice = 1;
        best = std::move(u_gal);
        nu_best = std::move(nu_gal);
        gal_rejects = 0;
      } else {
        gal_rejects += 1;
      }
    }
    if (choice == 0) {
      DTensor u_ls;
      probe.clear_info();
      if (direct) {
        DTensor Nm = normal_matrix(ln[l], ac, rn[l + 1]);
        Nm.view({(int)size, (int)size});
        pol_ls.solve(Nm, c_ls, u_ls, probe.info());
      } else {
        // scipy cg(x0=u_old, rtol, atol=0, maxiter=250, M=diag^{-1})
        u_ls = u_old.clone();
        DTensor dg = normal_diagonal(ln[l], ac, rn[l + 1]);
        pcg([&](GemmBatch& gb, const double* in, double* out) { nop.add(gb, 0, in, out); }, (int)size, c_ls.p,
            u_ls.p, dg.p, inner_rtol, 250);
      }
      u_ls.view(u_old.shape);
      trace_buffer("update u_ls", u_ls.p, u_ls.size());
      DTensor nu_ls = nop.apply(u_ls);
      probe.run(2, u_ls, nu_ls, c_ls, true);
      probe.read(h, &info, &swapped);
      if (direct) pol_ls.observe(info, swapped);
      if (direct && info == -1) {
        DTensor Nm = normal_matrix(ln[l], ac, rn[l + 1]);
        Nm.view({(int)size, (int)size});
        probe.clear_info();
        dense_solve_pivoted(Nm, c_ls, u_ls, probe.info());
        u_ls.view(u_old.shape);
        nu_ls = nop.apply(u_ls);
        probe.run(2, u_ls, nu_ls, c_ls, true);
        probe.read(h, &info);
      }
      if (direct && info != 0) {
        // singular normal block: numpy.linalg.lstsq fallback (tt_solver.py:395)
        DTensor Nm = normal_matrix(ln[l], ac, rn[l + 1]);
        Nm.view({(int)size, (int)size});
        lstsq_dense(Nm, c_ls, u_ls);
        u_ls.view(u_old.shape);
        nu_ls = nop.apply(u_ls);
        probe.clear_info();
        probe.run(2, u_ls, nu_ls, c_ls, true);
        probe.read(h, &info);
      }
      if (info == 0 && h[8] == 0.0) {
        const double q_ls = h[6] - 2.0 * h[7];
        if (q_ls <= best_q) {
          best_q = q_ls;
          choice = 2;
          best = std::move(u_ls);
          nu_best = std::move(nu_ls);
        }
      }
    }
    if (choice == 0) {
      best = u_old.clone();
      nu_best = std::move(nu_old);
    }
    // projected residual gradient N u - c steers the enrichment (for the
    // Galerkin candidate its probe has written it already)
    if (choice == 1) {
      grad = std::move(g_gal);
    } else {
      grad = std::move(nu_best);
      daxpy(-1.0, c_ls.p, grad.p, grad.size());
    }
  }
};

}  // namespace

Train als_solve(const Train& A, const Train& rhs, const Train& x0, const SolverConfig& cfg,
                SolveReport& rep) {
  T2S2_REQUIRE(A.is_op() && !rhs.is_op() && A.cols == rhs.rows && A.rows == rhs.rows, kErrShape,
               "operator and right-hand side shapes do not match");
  T2S2_REQUIRE(x0.rows == rhs.rows, kErrShape, "initial guess has wrong mode sizes");
  auto t0 = std::chrono::steady_clock::now();
  const double bnorm = tt_norm(rhs);
  T2S2_REQUIRE(bnorm != 0.0, kErrValue, "rhs must be nonzero");
  Train x = tt_round(x0, cfg.rounding_tol, cfg.max_rank);
  const int d = x.d();
  std::vector<DTensor> cores = std::move(x.cores);
  double best_res = INFINITY;
  std::vector<DTensor> best_cores = clone_all(cores);
  double current_res = 1.0;
  Sweep sw(A, rhs, cfg);

  for (int sweep = 0; sweep < cfg.max_sweeps; ++sweep) {
    right_orthonormalize(cores);
    // the boundary interfaces of both ends, one launch
    sw.ra[d] = DTensor({1, 1, 1});
    sw.rn[d] = DTensor({1, 1, 1, 1});
    sw.rg[d] = DTensor({1, 1, 1});
    sw.rb[d] = DTensor({1, 1});
    sw.la[0] = DTensor({1, 1, 1});
    sw.ln[0] = DTensor({1, 1, 1, 1});
    sw.lg[0] = DTensor({1, 1, 1});
    sw.lb[0] = DTensor({1, 1});
    fill_many({{sw.ra[d].p, 1}, {sw.rn[d].p, 1}, {sw.rg[d].p, 1}, {sw.rb[d].p, 1},
               {sw.la[0].p, 1}, {sw.ln[0].p, 1}, {sw.lg[0].p, 1}, {sw.lb[0].p, 1}},
              1.0);
    {
      GemmBatch gb;  // all four chains over the cores: 4 stages per core
      for (int l = d - 1, s0 = 0; l > 0; --l, s0 += 4) {
        sw.ra[l] = step_a_right(gb, s0, sw.ra[l + 1], cores[l], A.cores[l], sw.acg[l]);
        sw.rn[l] = step_n_right(gb, s0, sw.rn[l + 1], cores[l], A.cores[l], sw.acg[l]);
        sw.rg[l] = step_g_right(gb, s0, sw.rg[l + 1], cores[l], A.cores[l], rhs.cores[l]);
        sw.rb[l] = step_b_right(gb, s0, sw.rb[l + 1], cores[l], rhs.cores[l]);
      }
      gb.run();
    }

    DTensor end_grad;  // residual gradient of the last forward visit
    int end_choice = 0;
    bool end_direct = false;
    for (int l = 0; l < d; ++l) {
      DTensor u, grad;
      int choice;
      sw.update(l, cores, current_res, u, grad, choice);
      rep.choices.push_back(choice);
      if (l == d - 1) {
        cores[l] = std::move(u);
        end_grad = std::move(grad);
        end_choice = choice;
        end_direct = sw.gal_direct;
        break;
      }
      Split sp = split_forward(u, &grad, cfg, d, &cores[l + 1]);
      cores[l] = std::move(sp.core);
      const DTensor& nx = cores[l + 1];
      const int keep = sp.carry.dim(0), r1 = sp.carry.dim(1);
      const int rest = (int)(nx.size() / r1);
      DTensor nn = std::move(sp.next);  // rows of the enrichment part already zero
      {
        // the carry product (next core) and the four interface recurrences
        // of the moved bond are independent: one program
        GemmBatch gb;
        gb.add(0, false, false, keep, rest, r1, sp.carry.p, r1, 0, nx.p, rest, 0, nn.p, rest, 0);
        sw.la[l + 1] = step_a_left(gb, 0, sw.la[l], cores[l], A.cores[l], sw.acg[l]);
        sw.ln[l + 1] = step_n_left(gb, 0, sw.ln[l], cores[l], A.cores[l], sw.acg[l]);
        sw.lg[l + 1] = step_g_left(gb, 0, sw.lg[l], cores[l], A.cores[l], rhs.cores[l]);
        sw.lb[l + 1] = step_b_left(gb, 0, sw.lb[l], cores[l], rhs.cores[l]);
        gb.run();
      }
      cores[l + 1] = std::move(nn);
    }
    for (int l = d - 1; l >= 0; --l) {
      DTensor u, grad;
      int choice;
      if (l == d - 1 && d > 1 && end_choice == 1 && end_direct) {
        // The backward pass re-visits core d-1 with unchanged interfaces:
        // its Galerkin system is the one just solved, so the (deterministic)
        // dense solve would return the current core bit for bit, q_gal ==
        // q_old and the candidate is accepted (tt_solver.py:383-387).  Reuse
        // it.  Not for a GMRES candidate: the reference restarts GMRES from
        // the new core (x0 = u_old), which iterates on unless the forward run
        // reached its tolerance (tt_solver.py:367-377), so that case re-solves.
        u = std::move(cores[l]);  // cores[l] is replaced by the split below
        grad = std::move(end_grad);
        choice = 1;
      } else {
        sw.update(l, cores, current_res, u, grad, choice);
      }
      rep.choices.push_back(choice);
      if (l == 0) {
        cores[l] = std::move(u);
        break;
      }
      Split sp = split_backward(u, &grad, cfg, d, &cores[l - 1]);
      cores[l] = std::move(sp.core);
      const DTensor& pv = cores[l - 1];
      const int r0 = sp.carry.dim(0), keep = sp.carry.dim(1);
      const int rows = (int)(pv.size() / r0);
      const int nk = keep + sp.extra;
      DTensor np = std::move(sp.next);  // zeroed when it has enrichment columns
      {
        // the carry product (previous core) and the four interface
        // recurrences of the moved bond are independent: one program
        GemmBatch gb;
        gb.add(0, false, false, rows, keep, r0, pv.p, r0, 0, sp.carry.p, keep, 0, np.p, nk, 0);
        sw.ra[l] = step_a_right(gb, 0, sw.ra[l + 1], cores[l], A.cores[l], sw.acg[l]);
        sw.rn[l] = step_n_right(gb, 0, sw.rn[l + 1], cores[l], A.cores[l], sw.acg[l]);
        sw.rg[l] = step_g_right(gb, 0, sw.rg[l + 1], cores[l], A.cores[l], rhs.cores[l]);
        sw.rb[l] = step_b_right(gb, 0, sw.rb[l + 1], cores[l], rhs.cores[l]);
        gb.run();
      }
      cores[l - 1] = std::move(np);
    }
    current_res = measure_residual(A, sw.acg, cores, rhs, bnorm);
    rep.residuals.push_back(current_res);
    int mr = 1;
    double stored = 0.0, dense = 1.0;
    for (int l = 0; l < d; ++l) {
      mr = cores[l].dim(-1) > mr ? cores[l].dim(-1) : mr;
      stored += (double)cores[l].size();
      dense *= (double)cores[l].dim(1);
    }
    rep.ranks.push_back(mr);
    rep.compression.push_back(stored / dense);
    const bool done = current_res <= cfg.residual_tol;
    if (current_res < best_res) {
      best_res = current_res;
      if (done) {
        best_cores = std::move(cores);  // the sweep loop ends here: no copy
      } else {
        best_cores = clone_all(cores);
      }
    }
    if (done) {
      rep.converged = true;
      break;
    }
    const int w = cfg.stagnation_window;
    const int nh = (int)rep.residuals.size();
    if (nh > w) {
      double past = INFINITY, now = INFINITY;
      for (int i = 0; i < nh; ++i) {
        if (i < nh - w) past = rep.residuals[i] < past ? rep.residuals[i] : past;
        now = rep.residuals[i] < now ? rep.residuals[i] : now;
      }
      const double denom = past > 1e-300 ? past : 1e-300;
      if (past <= 0.0 || (past - now) / denom < cfg.stagnation_drop) {
        rep.stagnated = true;
        break;
      }
    }
  }
  if (!replaying_reads()) T2S2_CUDA(cudaStreamSynchronize(stream()));
  rep.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  Train out;
  out.rows = rhs.rows;
  out.cores = std::move(best_cores);
  return out;
}

double tt_residual(const Train& A, const Train& x, const Train& rhs, double tol) {
  const double bnorm = tt_norm(rhs);
  T2S2_REQUIRE(bnorm != 0.0, kErrValue, "rhs must be nonzero");
  Train diff = tt_round(tt_add(tt_apply(A, x), rhs, 1.0, -1.0), 0.01 * tol, 0);
  return tt_norm(diff) / bnorm;
}

}  // namespace t2s2
