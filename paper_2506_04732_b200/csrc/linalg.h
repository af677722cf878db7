// Small dense factorisations for TT orthogonalisation, rounding and the
// local solves: Householder QR, one-sided Jacobi SVD, LU with partial
// pivoting.
#pragma once

#include "common.h"

namespace t2s2 {

// Thin QR of a row-major m x n matrix: Q (m x k, orthonormal columns) and
// R (k x n, upper trapezoidal), k = min(m, n).  Householder reflectors in
// the LAPACK dgeqrf/dorgqr convention.
// cm: A (m x n) and Q (m x k) column-major instead.
void qr_thin(int m, int n, const double* A, DTensor& Q, DTensor& R, bool cm = false);
// The same, and NP (pr x k, row-major) = P (pr x n, row-major) R^T from the
// QR kernel itself when the one-CTA warp kernel applies (m >= n): returns
// whether NP was written — otherwise the caller multiplies.  The product has
// the GEMM engine's arithmetic (DMMA chain over k from a zero accumulator).
bool qr_thin_absorb(int m, int n, const double* A, DTensor& Q, DTensor& R, bool cm, const double* P, int pr,
                    double* NP);
void qr_thin_general(int m, int n, const double* A, DTensor& Q, DTensor& R, bool cm, int k);

// R factor only (k x n, k = min(m, n)) of a row-major m x n matrix; tall
// inputs are reduced by a TSQR tree of shared-memory Householder leaves.
void qr_r(int m, int n, const double* A, DTensor& R, bool cm = false);

// Thin SVD A = U diag(s) Vt of a row-major m x n matrix, k = min(m, n),
// singular values descending.  Tall case: QR, then one-sided Jacobi on R.
// Truncation rank of a split decided on the device (tt_solver.py:249-258,
// 268-270): delta = tol * ||s|| / rootd, keep = first k with ||s[k:]|| <= delta
// (at least 1), capped at max_rank; keep_out[0] = keep, mask[j] = j < keep.
// Products and sums are rounded separately, in the reference's order.
struct KeepArgs {
  double tol, rootd;
  int max_rank;
  double* keep_out;
  double* mask;
};
#ifdef __CUDACC__
__device__ __forceinline__ void split_keep_device(const double* s, int n, const KeepArgs& a) {
  double nrm = 0.0;
  for (int k = 0; k < n; ++k) nrm = __dadd_rn(nrm, __dmul_rn(s[k], s[k]));
  const double delta = a.tol * sqrt(nrm) / a.rootd;
  int r = n;
  double acc = 0.0;
  // tails from the back; keep the FIRST k with tail <= delta
  for (int k = n - 1; k >= 0; --k) {
    acc = __dadd_rn(acc, __dmul_rn(s[k], s[k]));
    if (sqrt(acc) <= delta) r = k;
  }
  if (n == 0) r = 1;
  if (r < 1) r = 1;
  if (r > a.max_rank) r = a.max_rank;
  a.keep_out[0] = (double)r;
  for (int j = 0; j < n; ++j) a.mask[j] = j < r ? 1.0 : 0.0;
}
#endif
// One-thread kernel around split_keep_device (s in device memory).
void split_keep(const double* s, int n, const KeepArgs& a);

// pub: an open read ticket (common.h) for the min(m, n) singular values —
// the kernel that finishes s publishes it (as soon as s is known, before U
// and Vt are written), other paths with a publish launch.
// keep: the truncation rank of the split is decided by the same kernel
// (one launch less; other paths run the one-thread kernel).
void svd_thin(int m, int n, const double* A, DTensor& U, DTensor& s, DTensor& Vt,
              const ReadTicket* pub = nullptr, const KeepArgs* keep = nullptr);

// In-place LU with partial pivoting of a column-major N x N matrix (ld=N);
// ipiv 0-based row swaps; *info_dev = 0 or 1 + first zero pivot column.
void lu_factor(int N, double* A, int* ipiv, int* info_dev);
// Solve with the factors for one right-hand side (in place).
void lu_solve(int N, const double* LU, const int* ipiv, double* b);
// One cooperative launch: factor A (clobbered) and overwrite b with the
// solution.  Returns false when N is too large for the smem panel.
// *swapped (optional, not cleared here) is set to 1 if any row was
// interchanged.
bool lu_solve_fused(int N, double* A, double* b, int* piv, int* info_dev, int* swapped = nullptr);
// Verified dense solve by blocked Gauss-Jordan without interchanges (one
// cooperative launch, gj_solve.cu): threshold partial pivoting — while every
// multiplier satisfies |l| <= 8 it eliminates without a pivot search
// (|l| <= 1 throughout means these are GEPP's factors) and overwrites b with
// the solution.  Otherwise (or on a zero pivot) it sets *info_dev = -1 and
// leaves A, b clobbered: rebuild and use the pivoting kernel.  Returns false
// when not applicable (nothing launched).
bool gj_solve_nopivot(int N, double* A, double* b, int* info_dev);

}  // namespace t2s2
