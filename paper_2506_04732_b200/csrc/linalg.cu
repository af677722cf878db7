// Householder QR and one-sided Jacobi SVD for the small, tall matrices of
// TT orthogonalisation and rounding (core unfoldings of size r*n x r).
//
// One CTA per factorisation: columns live contiguously (column-major
// scratch, L1/L2 resident), one warp owns one column at a time, so a
// Householder step needs two CTA barriers and a Jacobi round one.
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "blas.h"
#include "linalg.h"

namespace t2s2 {
namespace {

constexpr int kQrThreads = 512;
#ifdef SVD_MICRO
__device__ long long g_svd_t[8];
__device__ int g_svd_sweeps;
#define SVD_T(k) if (threadIdx.x == 0) g_svd_t[k] = clock64();
#else
#define SVD_T(k)
#endif

// Threads for a one-CTA factorisation whose column step keeps at most
// `busy` warps working: fewer warps make each CTA barrier cheaper.
inline int threads_for(int busy) {
  int w = busy < 2 ? 2 : (busy > kQrThreads / 32 ? kQrThreads / 32 : busy);
  return 32 * w;
}
constexpr size_t kSmemCap = 200 * 1024;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sum_{i in [lo, hi)} x[i]*y[i]*s over the lanes of a warp, four
// independent accumulators so the loads pipeline (result in every lane)
__device__ __forceinline__ double warp_dot(const double* x, const double* y, int lo, int hi,
                                           int lane, double s = 1.0) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int i = lo + lane;
  for (; i + 96 < hi; i += 128) {
    a0 = fma(x[i] * s, y[i], a0);
    a1 = fma(x[i + 32] * s, y[i + 32], a1);
    a2 = fma(x[i + 64] * s, y[i + 64], a2);
    a3 = fma(x[i + 96] * s, y[i + 96], a3);
  }
  for (; i < hi; i += 32) a0 = fma(x[i] * s, y[i], a0);
  return warp_sum((a0 + a1) + (a2 + a3));
}

// Householder QR of the column-major m x n matrix W in place (LAPACK
// dgeqrf conventions: R on and above the diagonal, reflectors below, tau).
// One warp per column update, three CTA barriers per column.
__device__ void qr_factor(int m, int n, double* W, double* tau) {
  const int k = m < n ? m : n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  __shared__ double sh_tau, sh_scal, sh_beta;
  for (int j = 0; j < k; ++j) {
    double* v = W + (long long)j * m;
    if (warp == 0) {
      const double s = warp_dot(v, v, j + 1, m, lane);
      if (lane == 0) {
        double alpha = v[j];
        if (s == 0.0) {
          sh_tau = 0.0;
          sh_scal = 1.0;
          sh_beta = alpha;
        } else {
          double nrm = sqrt(alpha * alpha + s);
          double beta = alpha >= 0.0 ? -nrm : nrm;
          sh_tau = (beta - alpha) / beta;
          sh_scal = 1.0 / (alpha - beta);
          sh_beta = beta;
        }
        tau[j] = sh_tau;
      }
    }
    __syncthreads();
    const double t = sh_tau, sc = sh_scal;
    if (t != 0.0) {
      for (int c = j + 1 + warp; c < n; c += nwarps) {
        double* col = W + (long long)c * m;
        const double w = warp_dot(v, col, j + 1, m, lane, sc) + col[j];
        double tw = t * w;
        if (lane == 0) col[j] -= tw;
        for (int i = j + 1 + lane; i < m; i += 32) col[i] = fma(-tw, v[i] * sc, col[i]);
      }
    }
    __syncthreads();
    if (t != 0.0) {
      for (int i = j + 1 + tid; i < m; i += blockDim.x) v[i] *= sc;
      if (tid == 0) v[j] = sh_beta;
    }
    __syncthreads();
  }
}

// Q = H_0 ... H_{k-1} [I_k; 0] formed in place over the reflectors in the
// first k columns of W (LAPACK dorg2r order).  R must be read before.
__device__ void qr_form_q(int m, int k, double* W, const double* tau) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  __syncthreads();
  for (int j = k - 1; j >= 0; --j) {
    const double t = tau[j];
    double* v = W + (long long)j * m;  // v_j = 1 implicit, v_i (i>j) stored
    if (t != 0.0)
      for (int c = j + 1 + warp; c < k; c += nwarps) {
        double* col = W + (long long)c * m;
        const double w = warp_dot(v, col, j + 1, m, lane) + col[j];
        const double tw = t * w;
        if (lane == 0) col[j] -= tw;
        for (int i = j + 1 + lane; i < m; i += 32) col[i] = fma(-tw, v[i], col[i]);
      }
    __syncthreads();
    for (int i = tid; i < m; i += blockDim.x) v[i] = i < j ? 0.0 : (i == j ? 1.0 - t : -t * v[i]);
    __syncthreads();
  }
}

// A row-major (m x n) -> Q row-major (m x k), R row-major (k x n).
// W: column-major m x n scratch, tau: k.  SM = true: the working copies live
// in dynamic shared memory (the caller checked the size), so every column
// step is LDS/STS instead of L2 trips.
// cm != 0: A and Q are column-major (A m x n, Q m x k) — the unfolding of a
// core read transposed, as the right-orthogonalisation needs it.
template <bool SM>
__global__ void __launch_bounds__(kQrThreads)
    qr_kernel(int m, int n, const double* __restrict__ A, double* Wg, double* Qg, double* tg,
              double* Q, double* R, int cm) {
  extern __shared__ double qsm[];
  const int k = m < n ? m : n;
  double* W = SM ? qsm : Wg;
  double* tau = SM ? qsm + (size_t)m * n : tg;
  (void)Qg;
  const int tid = threadIdx.x;
  for (int e = tid; e < (int)m * n; e += blockDim.x) {
    if (cm) {
      W[e] = A[e];
    } else {
      int i = (int)(e / n), j = (int)(e % n);
      W[(long long)j * m + i] = A[e];
    }
  }
  __syncthreads();
  qr_factor(m, n, W, tau);
  for (int e = tid; e < (int)k * n; e += blockDim.x) {
    int r = (int)(e / n), c = (int)(e % n);
    R[e] = c >= r ? W[(long long)c * m + r] : 0.0;
  }
  qr_form_q(m, k, W, tau);
  for (int e = tid; e < (int)m * k; e += blockDim.x) {
    if (cm) {
      Q[e] = W[e];
    } else {
      int i = (int)(e / k), c = (int)(e % k);
      Q[e] = W[(long long)c * m + i];
    }
  }
}

// R factor only, one CTA per block of rows (TSQR leaf): CTA c takes rows
// [c*chunk, min((c+1)*chunk, m)) of the row-major m x n matrix A, runs
// Householder in shared memory and writes its upper-trapezoidal R (zero
// padded to n rows) at rows [c*n, (c+1)*n) of Rout.
__global__ void __launch_bounds__(kQrThreads)
    qr_r_kernel(int m, int n, int chunk, const double* __restrict__ A, double* Rout, int cm) {
  extern __shared__ double W[];
  const int r0 = blockIdx.x * chunk;
  const int mr = m - r0 < chunk ? m - r0 : chunk;
  const int k = mr < n ? mr : n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  __shared__ double sh_tau, sh_scal, sh_beta;
  for (int e = tid; e < mr * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    W[j * mr + i] = cm ? A[(long long)j * m + r0 + i] : A[(long long)(r0 + i) * n + j];
  }
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    double* v = W + j * mr;
    if (warp == 0) {
      const double s = warp_dot(v, v, j + 1, mr, lane);
      if (lane == 0) {
        const double alpha = v[j];
        if (s == 0.0) {
          sh_tau = 0.0;
          sh_scal = 1.0;
          sh_beta = alpha;
        } else {
          const double nrm = sqrt(alpha * alpha + s);
          const double beta = alpha >= 0.0 ? -nrm : nrm;
          sh_tau = (beta - alpha) / beta;
          sh_scal = 1.0 / (alpha - beta);
          sh_beta = beta;
        }
      }
    }
    __syncthreads();
    const double t = sh_tau, sc = sh_scal;
    if (t != 0.0)
      for (int c = j + 1 + warp; c < n; c += nwarps) {
        double* col = W + c * mr;
        const double w = warp_dot(v, col, j + 1, mr, lane, sc) + col[j];
        const double tw = t * w;
        if (lane == 0) col[j] -= tw;
        for (int i = j + 1 + lane; i < mr; i += 32) col[i] = fma(-tw, v[i] * sc, col[i]);
      }
    __syncthreads();
    if (t != 0.0 && tid == 0) v[j] = sh_beta;
    __syncthreads();
  }
  double* R = Rout + (long long)blockIdx.x * n * n;
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int r = e / n, c = e % n;
    R[e] = (r < k && c >= r) ? W[c * mr + r] : 0.0;
  }
}

// One-sided (Hestenes) Jacobi on the columns of G (column-major p x q,
// p >= q), V (q x q) accumulating the rotations.  Circle-method ordering:
// each round rotates q/2 disjoint column pairs, one warp per pair.
__device__ void jacobi_sweeps(int p, int q, double* G, double* V) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  __shared__ int sh_rot;
  for (int e = tid; e < (int)q * q; e += blockDim.x) {
    int c = (int)(e / q), i = (int)(e % q);
    V[e] = i == c ? 1.0 : 0.0;
  }
  const double tol = DBL_EPSILON * sqrt((double)p);
  const int qe = q + (q & 1);
  __syncthreads();
  for (int sweep = 0; sweep < 60 && q > 1; ++sweep) {
    if (tid == 0) sh_rot = 0;
    __syncthreads();
    for (int rnd = 0; rnd < qe - 1; ++rnd) {
      for (int pi = warp; pi < qe / 2; pi += nwarps) {
        int a, b;
        if (pi == 0) {
          a = qe - 1;
          b = rnd;
        } else {
          a = (rnd + pi) % (qe - 1);
          b = (rnd - pi + qe - 1) % (qe - 1);
        }
        if (a >= q || b >= q) continue;
        if (a > b) {
          int t = a;
          a = b;
          b = t;
        }
        double* ga = G + (long long)a * p;
        double* gb = G + (long long)b * p;
        double al = 0.0, be = 0.0, ga_b = 0.0, al2 = 0.0, be2 = 0.0, gab2 = 0.0;
        int i = lane;
        for (; i + 32 < p; i += 64) {
          const double x = ga[i], y = gb[i], x2 = ga[i + 32], y2 = gb[i + 32];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga_b = fma(x, y, ga_b);
          al2 = fma(x2, x2, al2);
          be2 = fma(y2, y2, be2);
          gab2 = fma(x2, y2, gab2);
        }
        for (; i < p; i += 32) {
          const double x = ga[i], y = gb[i];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga_b = fma(x, y, ga_b);
        }
        al = warp_sum(al + al2);
        be = warp_sum(be + be2);
        ga_b = warp_sum(ga_b + gab2);
        if (ga_b == 0.0 || al == 0.0 || be == 0.0) continue;
        if (fabs(ga_b) <= tol * sqrt(al) * sqrt(be)) continue;
        double zeta = (be - al) / (2.0 * ga_b);
        double t;
        if (fabs(zeta) > 1e150)
          t = 0.5 / zeta;
        else
          t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        for (int i = lane; i < p; i += 32) {
          double x = ga[i], y = gb[i];
          ga[i] = c * x - sn * y;
          gb[i] = sn * x + c * y;
        }
        double* va = V + (long long)a * q;
        double* vb = V + (long long)b * q;
        for (int i = lane; i < q; i += 32) {
          double x = va[i], y = vb[i];
          va[i] = c * x - sn * y;
          vb[i] = sn * x + c * y;
        }
        if (lane == 0) sh_rot = 1;
      }
      __syncthreads();
    }
    __syncthreads();
#ifdef SVD_MICRO
    if (threadIdx.x == 0) g_svd_sweeps = sweep + 1;
#endif
    if (!sh_rot) break;
    __syncthreads();
  }
}

// Column norms of the rotated G -> s sorted descending (stable), perm[j] =
// source column of the j-th singular value.  sv: q doubles of scratch.
__device__ void jacobi_sort(int p, int q, const double* G, int* perm, double* s, double* sv) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int c = warp; c < q; c += nwarps) {
    const double* g = G + (long long)c * p;
    double acc = 0.0;
    for (int i = lane; i < p; i += 32) acc = fma(g[i], g[i], acc);
    acc = warp_sum(acc);
    if (lane == 0) s[c] = sqrt(acc);
  }
  __syncthreads();
  for (int c = tid; c < q; c += blockDim.x) {
    double sc = s[c];
    int rank = 0;
    for (int o = 0; o < q; ++o) {
      double so = s[o];
      rank += (so > sc) || (so == sc && o < c);
    }
    perm[rank] = c;
  }
  __syncthreads();
  for (int j = tid; j < q; j += blockDim.x) sv[j] = s[perm[j]];
  __syncthreads();
  for (int j = tid; j < q; j += blockDim.x) s[j] = sv[j];
  __syncthreads();
}

// Outputs U (row-major p x q), s (q), Vt (row-major q x q), singular values
// sorted descending.
template <bool SM>
__global__ void __launch_bounds__(kQrThreads)
    jacobi_kernel(int p, int q, double* Gg, double* Vg, int* perm, double* U, double* s,
                  double* Vt) {
  extern __shared__ double jsm[];
  double* G = Gg;
  double* V = SM ? jsm + (size_t)p * q : Vg;
  if (SM) {
    for (int e = threadIdx.x; e < p * q; e += blockDim.x) jsm[e] = Gg[e];
    G = jsm;
    __syncthreads();
  }
  const int tid = threadIdx.x;
  jacobi_sweeps(p, q, G, V);
  double* sv = V + (long long)q * q;  // q extra doubles of scratch after V
  jacobi_sort(p, q, G, perm, s, sv);
  for (int e = tid; e < (int)p * q; e += blockDim.x) {
    int i = (int)(e / q), j = (int)(e % q);
    double sj = s[j];
    U[e] = sj > 0.0 ? G[(long long)perm[j] * p + i] / sj : 0.0;
  }
  for (int e = tid; e < (int)q * q; e += blockDim.x) {
    int j = (int)(e / q), i = (int)(e % q);
    Vt[e] = V[(long long)perm[j] * q + i];
  }
}

// Whole thin SVD of a small row-major m x n matrix in one CTA, everything in
// shared memory: A' = A (m >= n) or A^T (m < n) is factored QR (Householder),
// R by one-sided Jacobi, U' = Q Ur; for the transposed case the roles of the
// factors swap on output.  Replaces QR, transpose, Jacobi and GEMM launches.
__global__ void __launch_bounds__(kQrThreads)
    svd_small_kernel(int m, int n, const double* __restrict__ A, double* U, double* s, double* Vt) {
  extern __shared__ double ssm[];
  const bool tr = m < n;
  const int mp = tr ? n : m, np = tr ? m : n;  // A' is mp x np, mp >= np
  double* W = ssm;                       // mp x np column-major
  double* tau = W + (size_t)mp * np;     // np
  double* G = tau + np;                  // np x np column-major (R, then rotated)
  double* V = G + (size_t)np * np;       // np x np
  double* sv = V + (size_t)np * np;      // np
  double* ss = sv + np;                  // np
  double* Ur = ss + np;                  // np x np: Ur[k*np + j]
  int* perm = reinterpret_cast<int*>(Ur + (size_t)np * np);
  const int tid = threadIdx.x;
  for (int e = tid; e < m * n; e += blockDim.x) {
    const int i = e / n, j = e - (e / n) * n;  // A(i, j)
    if (tr)
      W[(size_t)i * mp + j] = A[e];  // A'(j, i) = A(i, j), column i of A'
    else
      W[(size_t)j * mp + i] = A[e];
  }
  __syncthreads();
  SVD_T(0)
  qr_factor(mp, np, W, tau);
  for (int e = tid; e < np * np; e += blockDim.x) {
    const int c = e / np, i = e - c * np;
    G[e] = i <= c ? W[(size_t)c * mp + i] : 0.0;
  }
  __syncthreads();
  SVD_T(1)
  jacobi_sweeps(np, np, G, V);
  SVD_T(2)
  jacobi_sort(np, np, G, perm, ss, sv);
  for (int e = tid; e < np * np; e += blockDim.x) {
    const int k = e / np, j = e - k * np;
    const double sj = ss[j];
    Ur[e] = sj > 0.0 ? G[(size_t)perm[j] * np + k] / sj : 0.0;
  }
  for (int j = tid; j < np; j += blockDim.x) s[j] = ss[j];
  SVD_T(3)
  qr_form_q(mp, np, W, tau);  // begins with a barrier
  SVD_T(4)
  // U' = Q Ur (mp x np), V' = V[:, perm]
  if (!tr) {
    for (int e = tid; e < m * n; e += blockDim.x) {
      const int i = e / n, j = e - (e / n) * n;
      double acc = 0.0;
      for (int k = 0; k < np; ++k) acc = fma(W[(size_t)k * mp + i], Ur[k * np + j], acc);
      U[e] = acc;
    }
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int j = e / n, i = e - j * n;
      Vt[e] = V[(size_t)perm[j] * n + i];
    }
  } else {
    // A = V' S U'^T: U (m x m) = V'[:, perm] rows, Vt (m x n) = U'^T
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = e / m, j = e - i * m;
      U[e] = V[(size_t)perm[j] * m + i];
    }
    for (int e = tid; e < m * n; e += blockDim.x) {
      const int j = e / n, c = e - j * n;
      double acc = 0.0;
      for (int k = 0; k < np; ++k) acc = fma(W[(size_t)k * mp + c], Ur[k * np + j], acc);
      Vt[e] = acc;
    }
  }
}

// Thin SVD of a small row-major m x n matrix, np = min(m, n) <= 16 columns of
// A' (A, or A^T when m < n) and mp = max(m, n) <= 32 * RPL rows: the same
// algorithm as svd_small_kernel (Householder QR A' = Q R, one-sided Jacobi
// on R with circle ordering, U' = Q G/s, V' = accumulated rotations), with
// warp-level parallelism instead of CTA barriers per step:
//   QR     warp c holds column c of A' in registers (RPL rows per lane); the
//          owner of column j forms its reflector (LAPACK dgeqrf
//          conventions) and publishes it in shared memory, ONE CTA barrier,
//          every later column's warp applies it (warp reduction + axpy);
//   Jacobi in ONE warp, lane c holding column c of R and of V: a round's
//          disjoint pairs (partner lane (2 rnd - c) mod (qe - 1)) exchange
//          columns by shuffles and both lanes of a pair form the same
//          rotation locally — no reductions, no barriers; a sweep ends with
//          a warp vote;
//   Q      each warp applies H_c ... H_0 to its own unit column (no
//          barriers); U' = Q Ur through shared memory.
template <int RPL, int NPX>
__global__ void __launch_bounds__(512)
    svd_warp_kernel(int m, int n, const double* __restrict__ A, double* U, double* s, double* Vt,
                    ReadTicket pub, KeepArgs keep) {
  extern __shared__ double wsm[];
  const bool tr = m < n;
  const int mp = tr ? n : m, np = tr ? m : n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* vb = wsm;                      // reflectors, column j at vb[j*mp], v_j = 1 implicit
  double* Rs = vb + (size_t)mp * np;     // R column-major np x np
  double* tau = Rs + np * np;            // np
  double* Ur = tau + np;                 // np x np: Ur[k*np + j] = G[k][perm j] / s_j
  double* Vs = Ur + np * np;             // V' sorted: Vs[j*np + i] = V[i][perm j]
  double* ssv = Vs + np * np;            // np singular values (sorted)
  double* Qs = ssv + np;                 // Q column-major mp x np
  SVD_T(0)
  double a[RPL];
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = lane + 32 * r;
    a[r] = 0.0;
    if (warp < np && i < mp) a[r] = tr ? A[(size_t)warp * n + i] : A[(size_t)i * n + warp];
  }
  // --- Householder QR, one barrier per column
  for (int j = 0; j < np; ++j) {
    if (warp == j) {
      double ss = 0.0, alpha = 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        if (i > j && i < mp) ss = fma(a[r], a[r], ss);
        if (i == j) alpha = a[r];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      alpha = __shfl_sync(0xffffffffu, alpha, j & 31);
      double t, sc, beta;
      if (ss == 0.0) {
        t = 0.0;
        sc = 1.0;
        beta = alpha;
      } else {
        const double nrm = sqrt(alpha * alpha + ss);
        beta = alpha >= 0.0 ? -nrm : nrm;
        t = (beta - alpha) / beta;
        sc = 1.0 / (alpha - beta);
      }
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        if (i < mp) {
          if (i < j) Rs[j * np + i] = a[r];
          if (i == j) Rs[j * np + i] = beta;
          vb[(size_t)j * mp + i] = i > j ? a[r] * sc : (i == j ? 1.0 : 0.0);
        }
      }
      if (lane == 0) tau[j] = t;
    }
    __syncthreads();
    if (warp > j && warp < np) {
      const double t = tau[j];
      if (t != 0.0) {
        const double* v = vb + (size_t)j * mp;
        double w = 0.0, vv[RPL];
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = lane + 32 * r;
          vv[r] = (i >= j && i < mp) ? v[i] : 0.0;
          w = fma(vv[r], a[r], w);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        const double tw = t * w;
#pragma unroll
        for (int r = 0; r < RPL; ++r) a[r] = fma(-tw, vv[r], a[r]);
      }
    }
  }
  SVD_T(1)
  // --- one-sided Jacobi on R in warp 0: lane c = column c of R and of V
  if (warp == 0) {
    const int c = lane;
    double g[NPX], v[NPX];
#pragma unroll
    for (int i = 0; i < NPX; ++i) {
      g[i] = (c < np && i < np && i <= c) ? Rs[c * np + i] : 0.0;
      v[i] = (i == c && c < np) ? 1.0 : 0.0;
    }
    const double tol = DBL_EPSILON * sqrt((double)np), tol2 = tol * tol;
    const int qe = np + (np & 1);
    for (int sweep = 0; sweep < 60 && np > 1; ++sweep) {
      bool rot = false;
      for (int rnd = 0; rnd < qe - 1; ++rnd) {
        int pt;
        if (c == qe - 1)
          pt = rnd;
        else if (c == rnd)
          pt = qe - 1;
        else {
          pt = 2 * rnd - c;
          if (pt < 0) pt += qe - 1;
          if (pt >= qe - 1) pt -= qe - 1;
        }
        if (c >= qe) pt = c;
        double pg[NPX];
#pragma unroll
        for (int i = 0; i < NPX; ++i) pg[i] = __shfl_sync(0xffffffffu, g[i], pt);
        const bool isa = c < pt;
        bool doit = false;
        double cs = 1.0, ssn = 0.0;  // own' = cs own + ssn partner
        if (c < np && pt < np && pt != c) {
          double o2 = 0.0, p2 = 0.0, op = 0.0;
#pragma unroll
          for (int i = 0; i < NPX; ++i) {
            o2 = fma(g[i], g[i], o2);
            p2 = fma(pg[i], pg[i], p2);
            op = fma(g[i], pg[i], op);
          }
          const double al = isa ? o2 : p2, be = isa ? p2 : o2, gab = op;
          if (!(gab == 0.0 || al == 0.0 || be == 0.0) && !(gab * gab <= tol2 * al * be)) {
            // the rotation of svd_small_kernel (column a: c x - s y, column b:
            // s x + c y) with t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)),
            // zeta = (be - al) / (2 gab), rewritten without forming zeta:
            // t = sign(e) d / (|e| + sqrt(e^2 + d^2)), e = be - al, d = 2 gab
            const double e = be - al, d = 2.0 * gab;
            const double t = (e >= 0.0 ? d : -d) / (fabs(e) + sqrt(fma(e, e, d * d)));
            cs = rsqrt(fma(t, t, 1.0));
            const double sn = cs * t;
            ssn = isa ? -sn : sn;
            doit = true;
            rot = true;
          }
        }
#pragma unroll
        for (int i = 0; i < NPX; ++i) {
          const double pvi = __shfl_sync(0xffffffffu, v[i], pt);
          g[i] = doit ? fma(ssn, pg[i], cs * g[i]) : g[i];
          v[i] = doit ? fma(ssn, pvi, cs * v[i]) : v[i];
        }
      }
#ifdef SVD_MICRO
      if (lane == 0) g_svd_sweeps = sweep + 1;
#endif
      if (!__any_sync(0xffffffffu, rot)) break;
    }
    // singular values sorted descending (stable), Ur = G[:, perm] / s, V' = V[:, perm]
    double nrm = 0.0;
#pragma unroll
    for (int i = 0; i < NPX; ++i) nrm = fma(g[i], g[i], nrm);
    nrm = sqrt(nrm);
    int rank = 0;
    for (int o = 0; o < np; ++o) {
      const double so = __shfl_sync(0xffffffffu, nrm, o);
      rank += (so > nrm) || (so == nrm && o < c);
    }
    if (c < np) {
      ssv[rank] = nrm;
#pragma unroll
      for (int i = 0; i < NPX; ++i)
        if (i < np) {
          Ur[i * np + rank] = nrm > 0.0 ? g[i] / nrm : 0.0;
          Vs[rank * np + i] = v[i];
        }
    }
  }
  SVD_T(2)
  // --- Q = H_0 ... H_{k-1} [I; 0], warp c forms column c on its own
  if (warp < np) {
    double q[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) q[r] = (lane + 32 * r == warp) ? 1.0 : 0.0;
    for (int j = warp; j >= 0; --j) {  // H_j leaves e_c unchanged for j > c
      const double t = tau[j];
      if (t == 0.0) continue;
      const double* v = vb + (size_t)j * mp;
      double w = 0.0, vv[RPL];
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        vv[r] = (i >= j && i < mp) ? v[i] : 0.0;
        w = fma(vv[r], q[r], w);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
      const double tw = t * w;
#pragma unroll
      for (int r = 0; r < RPL; ++r) q[r] = fma(-tw, vv[r], q[r]);
    }
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i < mp) Qs[(size_t)warp * mp + i] = q[r];
    }
  }
  __syncthreads();
  SVD_T(3)
  for (int j = tid; j < np; j += blockDim.x) s[j] = ssv[j];
  if (keep.keep_out && tid == 32) split_keep_device(ssv, np, keep);  // the split's rank (one thread)
  if (pub.dst) {
    // the host decides the rank from s: publish it now, U and Vt follow
    if (tid < 2 * np) pub.dst[tid] = reinterpret_cast<const unsigned*>(ssv)[tid];
    __threadfence_system();
    __syncthreads();
    if (tid == 0) *(volatile unsigned*)pub.flag = pub.value;
  }
  // U' = Q Ur (mp x np); V' = V[:, perm]
  if (!tr) {
    for (int e = tid; e < m * n; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      double acc = 0.0;
      for (int k = 0; k < np; ++k) acc = fma(Qs[(size_t)k * mp + i], Ur[k * np + j], acc);
      U[e] = acc;
    }
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int j = e / n, i = e - j * n;
      Vt[e] = Vs[j * np + i];
    }
  } else {
    // A = V' S U'^T: U (m x m) = V'[:, perm], Vt (m x n) = U'^T
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = e / m, j = e - i * m;
      U[e] = Vs[j * np + i];
    }
    for (int e = tid; e < m * n; e += blockDim.x) {
      const int j = e / n, cc = e - j * n;
      double acc = 0.0;
      for (int k = 0; k < np; ++k) acc = fma(Qs[(size_t)k * mp + cc], Ur[k * np + j], acc);
      Vt[e] = acc;
    }
  }
}

template <int RPL, int NPX>
void launch_svd_warp(int m, int n, const double* A, double* U, double* s, double* Vt, size_t smem,
                     int thr, const ReadTicket& pub, const KeepArgs& keep) {
  max_dynamic_smem((const void*)svd_warp_kernel<RPL, NPX>, (int)kSmemCap);
  svd_warp_kernel<RPL, NPX><<<1, thr, smem, stream()>>>(m, n, A, U, s, Vt, pub, keep);
}

__global__ void split_keep_kernel(const double* s, int n, KeepArgs a) {
  if (threadIdx.x == 0) split_keep_device(s, n, a);
}

// Householder QR of a tall block (m rows <= 32 * RPL, n <= 32 * CPW columns,
// m >= n) with warp-level parallelism: warp w holds columns w, w + nw, ...
// (CPW of them) in registers, RPL rows per lane.  Column j's owner forms
// its reflector (LAPACK dgeqrf conventions), publishes it in shared memory,
// ONE CTA barrier, and every owner of later columns applies it (warp
// reduction + axpy).  Mode Q: thin Q (each warp forms its own columns of
// H_0 ... H_{n-1} [I; 0], no barriers) and R; mode R (TSQR leaf): CTA b
// factors rows [b*chunk, b*chunk + rows) and writes its n x n R at rows
// [b*n, (b+1)*n) of the output.  A, Q column-major when cm, else row-major.
#ifdef WQR_MICRO
__device__ unsigned long long g_wqr_t[4];  // owner: form; everyone (warp 1): barrier wait, apply
#define WQR_T0 long long wq_t = clock64();
#define WQR_T(k, cond)                                    \
  if ((cond) && lane == 0) {                              \
    const long long t_ = clock64();                       \
    atomicAdd(&g_wqr_t[k], (unsigned long long)(t_ - wq_t)); \
  }                                                       \
  wq_t = clock64();
#else
#define WQR_T0
#define WQR_T(k, cond)
#endif
template <int RPL, int CPW, bool WANTQ>
__global__ void __launch_bounds__(512)
    wqr_kernel(int m, int n, int chunk, const double* __restrict__ A, double* Q, double* R, int cm,
               const double* __restrict__ P, int pr, double* NP) {
  extern __shared__ double qsm2[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int r0 = blockIdx.x * chunk;
  const int mr = m - r0 < chunk ? m - r0 : chunk;  // rows of this block (>= n, or the whole matrix)
  const int k = mr < n ? mr : n;
  double* vb = qsm2;                  // reflectors, column j at vb[j*mr]
  double* Rs = vb + (size_t)mr * n;   // R column-major n x n
  double* tau = Rs + (size_t)n * n;   // n
  double a[CPW][RPL];
#pragma unroll
  for (int q = 0; q < CPW; ++q) {
    const int c = warp + q * nw;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      a[q][r] = (c < n && i < mr) ? (cm ? A[(size_t)c * m + r0 + i] : A[(size_t)(r0 + i) * n + c]) : 0.0;
    }
  }
  WQR_T0
  for (int j = 0; j < k; ++j) {
    const int ow = j % nw, oq = j / nw;
    WQR_T(3, false)
    if (warp == ow) {
      double ss = 0.0, alpha = 0.0;
#pragma unroll
      for (int q = 0; q < CPW; ++q)
        if (q == oq)
#pragma unroll
          for (int r = 0; r < RPL; ++r) {
            const int i = lane + 32 * r;
            if (i > j && i < mr) ss = fma(a[q][r], a[q][r], ss);
            if (i == j) alpha = a[q][r];
          }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      alpha = __shfl_sync(0xffffffffu, alpha, j & 31);
      double t, sc, beta;
      if (ss == 0.0) {
        t = 0.0;
        sc = 1.0;
        beta = alpha;
      } else {
        const double nrm = sqrt(alpha * alpha + ss);
        beta = alpha >= 0.0 ? -nrm : nrm;
        t = (beta - alpha) / beta;
        sc = 1.0 / (alpha - beta);
      }
#pragma unroll
      for (int q = 0; q < CPW; ++q)
        if (q == oq)
#pragma unroll
          for (int r = 0; r < RPL; ++r) {
            const int i = lane + 32 * r;
            if (i < mr) {
              if (i < j) Rs[(size_t)j * n + i] = a[q][r];
              if (i == j) Rs[(size_t)j * n + i] = beta;
              vb[(size_t)j * mr + i] = i > j ? a[q][r] * sc : (i == j ? 1.0 : 0.0);
            }
          }
      if (lane == 0) tau[j] = t;
    }
    WQR_T(0, warp == ow && blockIdx.x == 0)
    __syncthreads();
    WQR_T(1, warp == (ow + 1) % nw && blockIdx.x == 0)
    const double t = tau[j];
    if (t != 0.0) {
      const double* v = vb + (size_t)j * mr;
      double vv[RPL];
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        vv[r] = (i >= j && i < mr) ? v[i] : 0.0;
      }
      // the CPW columns' dot products and butterfly reductions interleaved
      // (independent chains; each column's arithmetic is unchanged)
      double w[CPW];
#pragma unroll
      for (int q = 0; q < CPW; ++q) {
        w[q] = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) w[q] = fma(vv[r], a[q][r], w[q]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < CPW; ++q) w[q] += __shfl_xor_sync(0xffffffffu, w[q], o);
#pragma unroll
      for (int q = 0; q < CPW; ++q) {
        const int c = warp + q * nw;
        if (c > j && c < n) {
          const double tw = t * w[q];
#pragma unroll
          for (int r = 0; r < RPL; ++r) a[q][r] = fma(-tw, vv[r], a[q][r]);
        }
      }
    }
    WQR_T(2, warp == (ow + 1) % nw && blockIdx.x == 0)
  }
  // columns j >= k (wide leaf, mr < n): their R rows < k are the updated values
#pragma unroll
  for (int q = 0; q < CPW; ++q) {
    const int c = warp + q * nw;
    if (c >= k && c < n)
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        if (i < k) Rs[(size_t)c * n + i] = a[q][r];
      }
  }
  __syncthreads();
  if (!WANTQ) {
    double* Rb = R + (size_t)blockIdx.x * n * n;  // n x n row-major, zero padded
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int rr = e / n, cc = e - rr * n;
      Rb[e] = (rr < k && cc >= rr) ? Rs[(size_t)cc * n + rr] : 0.0;
    }
    return;
  }
  {
    // k x n (one block), or n x n per block (TSQR leaves, rows >= n)
    double* Rb = R + (size_t)blockIdx.x * n * n;
    for (int e = tid; e < k * n; e += blockDim.x) {
      const int rr = e / n, cc = e - rr * n;
      Rb[e] = cc >= rr ? Rs[(size_t)cc * n + rr] : 0.0;
    }
  }
  // thin Q: warp forms its own columns c < k (rows of this block)
#pragma unroll
  for (int q = 0; q < CPW; ++q) {
    const int c = warp + q * nw;
    if (c >= k) continue;
    double x[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) x[r] = (lane + 32 * r == c) ? 1.0 : 0.0;
    for (int j = c; j >= 0; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      const double* v = vb + (size_t)j * mr;
      double w = 0.0, vv[RPL];
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        vv[r] = (i >= j && i < mr) ? v[i] : 0.0;
        w = fma(vv[r], x[r], w);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
      const double tw = tj * w;
#pragma unroll
      for (int r = 0; r < RPL; ++r) x[r] = fma(-tw, vv[r], x[r]);
    }
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i < mr) {
        if (cm)
          Q[(size_t)c * m + r0 + i] = x[r];
        else
          Q[(size_t)(r0 + i) * k + c] = x[r];
      }
    }
  }
  // Absorb R into the neighbouring core, NP (pr x k) = P (pr x n) R^T (one
  // block, m >= n): the GEMM that followed this kernel in the
  // orthonormalisation sweep, with its arithmetic — each 8 x 8 block of NP
  // is the DMMA m8n8k4 chain over k = 0, 4, 8, ... from a zero accumulator
  // (trailing k zero filled), exactly the GEMM tile engine's sequence.
  if (P) {
    const int rb = (pr + 7) / 8, cb = (k + 7) / 8;
    for (int blk = warp; blk < rb * cb; blk += nw) {
      const int i = (blk / cb) * 8 + (lane >> 2), j = (blk % cb) * 8 + (lane >> 2);
      double d0 = 0.0, d1 = 0.0;
      for (int kk = 0; kk < n; kk += 4) {
        const int kc = kk + (lane & 3);
        const double av = (i < pr && kc < n) ? P[(size_t)i * n + kc] : 0.0;
        const double bv = (j < k && kc < n && kc >= j) ? Rs[(size_t)kc * n + j] : 0.0;  // R[j][kc]
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                     : "+d"(d0), "+d"(d1)
                     : "d"(av), "d"(bv));
      }
      const int oc = (blk % cb) * 8 + (lane & 3) * 2;
      if (i < pr) {
        if (oc < k) NP[(size_t)i * k + oc] = d0;
        if (oc + 1 < k) NP[(size_t)i * k + oc + 1] = d1;
      }
    }
  }
}

template <int RPL, int CPW, bool WANTQ>
void launch_wqr(int blocks, int thr, size_t smem, int m, int n, int chunk, const double* A, double* Q,
                double* R, int cm, const double* P, int pr, double* NP) {
  max_dynamic_smem((const void*)wqr_kernel<RPL, CPW, WANTQ>, (int)kSmemCap);
  wqr_kernel<RPL, CPW, WANTQ><<<blocks, thr, smem, stream()>>>(m, n, chunk, A, Q, R, cm, P, pr, NP);
}

// Dispatch: at most 16 warps, CPW = ceil(n / 16) columns each (1, 2 or 4);
// rows per block <= 384 (<= 256 with four columns per warp, registers);
// false if not applicable.
template <bool WANTQ>
bool wqr(int blocks, int m, int n, int chunk, const double* A, double* Q, double* R, int cm,
         const double* P = nullptr, int pr = 0, double* NP = nullptr) {
  const int rows = chunk < m ? chunk : m;
  const int cpw = n <= 16 ? 1 : (n <= 32 ? 2 : 4);
  if (n < 1 || n > 64 || rows > (cpw == 4 ? 256 : 384)) return false;
  const int rpl = (rows + 31) / 32;
  const int nw = (n + cpw - 1) / cpw;
  const int thr = 32 * (nw < 2 ? 2 : nw);
  const size_t smem = ((size_t)rows * n + (size_t)n * n + n) * sizeof(double);
  if (smem > kSmemCap) return false;
#define T2S2_WQR(R_, C_) launch_wqr<R_, C_, WANTQ>(blocks, thr, smem, m, n, chunk, A, Q, R, cm, P, pr, NP)
  if (cpw == 1) {
    if (rpl <= 4) T2S2_WQR(4, 1);
    else if (rpl <= 8) T2S2_WQR(8, 1);
    else T2S2_WQR(12, 1);
  } else if (cpw == 2) {
    if (rpl <= 4) T2S2_WQR(4, 2);
    else if (rpl <= 8) T2S2_WQR(8, 2);
    else T2S2_WQR(12, 2);
  } else {
    if (rpl <= 4) T2S2_WQR(4, 4);
    else T2S2_WQR(8, 4);
  }
#undef T2S2_WQR
  return true;
}

}  // namespace

void qr_r(int m, int n, const double* A, DTensor& R, bool cm) {
  T2S2_REQUIRE(m > 0 && n > 0, kErrShape, "qr_r: empty matrix");
  if (n <= 64 && m >= n) {
    // warp-level TSQR: leaves of <= 384 rows (and >= 2n so the stack shrinks)
    const int k = m < n ? m : n;
    const int cap = n > 32 ? 256 : 384;  // rows per leaf (see wqr)
    int chunk = m;
    if (m > cap) {
      const int leaves = (m + cap - 1) / cap;
      chunk = (m + leaves - 1) / leaves;
      if (chunk < 2 * n) chunk = 2 * n;
    }
    const int blocks = ceil_div(m, chunk);
    if (chunk <= cap && (blocks == 1 || chunk >= 2 * n)) {
      DTensor stacked({blocks * n, n});
      bool ok;
      {
        LaunchScope ls("qr", 2.0 * m * (double)n * n, 8.0 * m * (double)n);
        ok = wqr<false>(blocks, m, n, chunk, A, nullptr, stacked.p, cm ? 1 : 0);
      }
      if (ok) {
        T2S2_CHECK_LAUNCH();
        if (blocks == 1) {
          R = std::move(stacked);  // k == n here (m >= n): the leaf's factor is R
          R.view({k, n});
          return;
        }
        qr_r(blocks * n, n, stacked.p, R);
        return;
      }
    }
  }
  // rows per CTA so that the CTA's block fits the shared-memory budget
  int chunk = (int)(kSmemCap / (sizeof(double) * (size_t)n));
  if (chunk > m) chunk = m;
  if (chunk < m && chunk < 2 * n) {
    // a TSQR leaf would not shrink the row count: one global-memory QR
    DTensor Q;
    qr_thin(m, n, A, Q, R, cm);
    return;
  }
  const int blocks = ceil_div(m, chunk);
  max_dynamic_smem((const void*)qr_r_kernel, (int)kSmemCap);
  DTensor stacked({blocks * n, n});
  {
    LaunchScope ls("qr", 2.0 * m * (double)n * n, 8.0 * m * (double)n);
    qr_r_kernel<<<blocks, threads_for(n), (size_t)chunk * n * sizeof(double), stream()>>>(
        m, n, chunk, A, stacked.p, cm ? 1 : 0);
  }
  T2S2_CHECK_LAUNCH();
  if (blocks == 1) {
    const int k = m < n ? m : n;
    R = DTensor({k, n});
    dcopy(R.p, stacked.p, (size_t)k * n);
    return;
  }
  qr_r(blocks * n, n, stacked.p, R);  // TSQR: reduce the stacked leaf factors
}

void qr_thin(int m, int n, const double* A, DTensor& Q, DTensor& R, bool cm) {
  qr_thin_absorb(m, n, A, Q, R, cm, nullptr, 0, nullptr);
}

bool qr_thin_absorb(int m, int n, const double* A, DTensor& Q, DTensor& R, bool cm, const double* P, int pr,
                    double* NP) {
  T2S2_REQUIRE(m > 0 && n > 0, kErrShape, "qr_thin: empty matrix");
  const int k = m < n ? m : n;
  Q = DTensor({m, k});
  R = DTensor({k, n});
  if (m >= n && m <= (n > 32 ? 256 : 384) && n <= 64) {
    bool ok;
    {
      LaunchScope ls("qr", 4.0 * m * (double)n * k + 2.0 * pr * (double)n * k, 16.0 * m * (double)n);
      ok = wqr<true>(1, m, n, m, A, Q.p, R.p, cm ? 1 : 0, P, pr, NP);
    }
    if (ok) {
      T2S2_CHECK_LAUNCH();
      return P != nullptr;
    }
  }
  qr_thin_general(m, n, A, Q, R, cm, k);
  return false;
}

// the paths beyond the one-CTA warp kernel (Q and R allocated by the caller)
void qr_thin_general(int m, int n, const double* A, DTensor& Q, DTensor& R, bool cm, int k) {
  // tall blocks that do not fit the one-CTA shared-memory kernel (config-4
  // cores, 33*64 x 64): TSQR with Q — warp-level leaves, the stacked leaf
  // R factors factored recursively (Q2, R), Q = diag(Q_leaf) Q2 as one
  // small GEMM per leaf
  if (m > n && n <= 64 && ((size_t)m * n + k) * sizeof(double) > kSmemCap) {
    const int cap = n > 32 ? 256 : 384;
    const int leaves = (m + cap - 1) / cap;
    const int chunk = (m + leaves - 1) / leaves;
    const int blocks = ceil_div(m, chunk);
    const int last = m - (blocks - 1) * chunk;
    if (chunk <= cap && last >= n) {
      DTensor Ql({m, n}), S({blocks * n, n});
      bool ok;
      {
        LaunchScope ls("qr", 4.0 * m * (double)n * n, 16.0 * m * (double)n);
        ok = wqr<true>(blocks, m, n, chunk, A, Ql.p, S.p, cm ? 1 : 0);
      }
      if (ok) {
        T2S2_CHECK_LAUNCH();
        DTensor Q2;
        qr_thin(blocks * n, n, S.p, Q2, R, false);  // Q2 row-major (blocks n) x n, R n x n
        for (int b = 0; b < blocks; ++b) {
          const int r0 = b * chunk, mr = b + 1 < blocks ? chunk : last;
          if (cm)  // Q^T (n x m, ld m) block = Q2_b^T Q_b^T
            gemm(true, false, n, mr, n, 1.0, Q2.p + (size_t)b * n * n, n, Ql.p + r0, m, 0.0,
                 Q.p + r0, m);
          else  // Q rows of the leaf = Q_b Q2_b
            gemm(false, false, mr, n, n, 1.0, Ql.p + (size_t)r0 * n, n, Q2.p + (size_t)b * n * n, n,
                 0.0, Q.p + (size_t)r0 * n, n);
        }
        return;
      }
    }
  }
  double* W = allocator().alloc((size_t)m * n);
  double* Qc = allocator().alloc((size_t)m * k);
  double* tau = allocator().alloc(k);
  {
    LaunchScope ls("qr", 4.0*m*(double)n*(m<n?m:n), 16.0*m*(double)n);
    const size_t need = ((size_t)m * n + k) * sizeof(double);
    if (need <= kSmemCap) {
      max_dynamic_smem((const void*)qr_kernel<true>, (int)kSmemCap);
      qr_kernel<true><<<1, threads_for(n), need, stream()>>>(m, n, A, W, Qc, tau, Q.p, R.p,
                                                              cm ? 1 : 0);
    } else {
      qr_kernel<false><<<1, kQrThreads, 0, stream()>>>(m, n, A, W, Qc, tau, Q.p, R.p, cm ? 1 : 0);
    }
  }
  T2S2_CHECK_LAUNCH();
  allocator().release(W);
  allocator().release(Qc);
  allocator().release(tau);
}

namespace {

// Jacobi SVD of a column-major p x q (p >= q) matrix held in G (clobbered).
void jacobi_svd(int p, int q, double* G, DTensor& U, DTensor& s, DTensor& Vt) {
  U = DTensor({p, q});
  s = DTensor({q});
  Vt = DTensor({q, q});
  double* V = allocator().alloc((size_t)q * q + q);
  int* perm = reinterpret_cast<int*>(allocator().alloc(q));
  {
    LaunchScope ls("svd_jacobi", 0, 0);
    const size_t need = ((size_t)p * q + (size_t)q * q + q) * sizeof(double);
    if (need <= kSmemCap) {
      max_dynamic_smem((const void*)jacobi_kernel<true>, (int)kSmemCap);
      jacobi_kernel<true><<<1, threads_for((q + 1) / 2), need, stream()>>>(p, q, G, V, perm, U.p,
                                                                           s.p, Vt.p);
    } else {
      jacobi_kernel<false><<<1, kQrThreads, 0, stream()>>>(p, q, G, V, perm, U.p, s.p, Vt.p);
    }
  }
  T2S2_CHECK_LAUNCH();
  allocator().release(V);
  allocator().release(reinterpret_cast<double*>(perm));
}

// Tall case (m >= n): A = Q R, R = Ur S Vt, U = Q Ur.
void svd_tall(int m, int n, const double* A, DTensor& U, DTensor& s, DTensor& Vt) {
  DTensor Q, R;
  qr_thin(m, n, A, Q, R);  // Q m x n, R n x n
  double* G = allocator().alloc((size_t)n * n);
  transpose(R.p, G, n, n);  // column-major copy of R
  DTensor Ur;
  jacobi_svd(n, n, G, Ur, s, Vt);
  allocator().release(G);
  U = DTensor({m, n});
  gemm(false, false, m, n, n, 1.0, Q.p, n, Ur.p, n, 0.0, U.p, n);
}

}  // namespace

namespace {
void svd_thin_run(int m, int n, const double* A, DTensor& U, DTensor& s, DTensor& Vt, const ReadTicket* pub,
                  const KeepArgs* keep, bool& published) {
  T2S2_REQUIRE(m > 0 && n > 0, kErrShape, "svd_thin: empty matrix");
  {
    const int mp = m >= n ? m : n, np = m >= n ? n : m;
    // warp-level kernel: np <= 16 columns, mp <= 384 rows
    const size_t wneed = (2 * (size_t)mp * np + 3 * (size_t)np * np + 2 * (size_t)np) * sizeof(double);
    if (np <= 16 && mp <= 384 && wneed <= kSmemCap) {
      U = m >= n ? DTensor({m, n}) : DTensor({m, m});
      s = DTensor({np});
      Vt = m >= n ? DTensor({n, n}) : DTensor({m, n});
      {
        LaunchScope ls("svd_jacobi", 4.0 * mp * (double)np * np, 8.0 * m * (double)n);
        const int thr = 32 * (np < 2 ? 2 : np);
        const ReadTicket tk = pub ? *pub : ReadTicket{};
        const KeepArgs kp = keep ? *keep : KeepArgs{};
        published = true;
        const int rpl = (mp + 31) / 32;
#define T2S2_SVD_WARP(NPX)                                                            \
  do {                                                                            \
    if (rpl <= 4) launch_svd_warp<4, NPX>(m, n, A, U.p, s.p, Vt.p, wneed, thr, tk, kp);   \
    else if (rpl <= 8) launch_svd_warp<8, NPX>(m, n, A, U.p, s.p, Vt.p, wneed, thr, tk, kp); \
    else launch_svd_warp<12, NPX>(m, n, A, U.p, s.p, Vt.p, wneed, thr, tk, kp);           \
  } while (0)
        if (np <= 4) T2S2_SVD_WARP(4);
        else if (np <= 8) T2S2_SVD_WARP(8);
        else if (np <= 12) T2S2_SVD_WARP(12);
        else T2S2_SVD_WARP(16);
#undef T2S2_SVD_WARP
      }
      T2S2_CHECK_LAUNCH();
      return;
    }
    const size_t need = ((size_t)mp * np + 3 * (size_t)np * np + 4 * (size_t)np) * sizeof(double);
    if (need <= kSmemCap && np <= 64) {
      max_dynamic_smem((const void*)svd_small_kernel, (int)kSmemCap);
      U = m >= n ? DTensor({m, n}) : DTensor({m, m});
      s = DTensor({np});
      Vt = m >= n ? DTensor({n, n}) : DTensor({m, n});
      {
        LaunchScope ls("svd_jacobi", 4.0 * mp * (double)np * np, 8.0 * m * (double)n);
        svd_small_kernel<<<1, threads_for(np), need, stream()>>>(m, n, A, U.p, s.p, Vt.p);
      }
      T2S2_CHECK_LAUNCH();
      return;
    }
  }
  if (m >= n) {
    svd_tall(m, n, A, U, s, Vt);
    return;
  }
  // A^T (n x m, tall) = U' S V'^T  =>  A = V' S U'^T
  double* At = allocator().alloc((size_t)m * n);
  transpose(A, At, m, n);
  DTensor U2, Vt2;
  svd_tall(n, m, At, U2, s, Vt2);  // U2 n x m, Vt2 m x m
  allocator().release(At);
  U = DTensor({m, m});
  transpose(Vt2.p, U.p, m, m);
  Vt = DTensor({m, n});
  transpose(U2.p, Vt.p, n, m);
}
}  // namespace

void split_keep(const double* s, int n, const KeepArgs& a) {
  {
    LaunchScope ls("reduce", 0, 0);
    split_keep_kernel<<<1, 32, 0, stream()>>>(s, n, a);
  }
  T2S2_CHECK_LAUNCH();
}

void svd_thin(int m, int n, const double* A, DTensor& U, DTensor& s, DTensor& Vt, const ReadTicket* pub,
              const KeepArgs* keep) {
  bool fused = false;  // the warp kernel published s / decided the rank itself
  svd_thin_run(m, n, A, U, s, Vt, pub, keep, fused);
  if (keep && !fused) split_keep(s.p, s.dim(0), *keep);
  if (pub && !fused) read_publish(s.p, s.size() * sizeof(double), *pub);
}

}  // namespace t2s2
