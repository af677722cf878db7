// Device tensor-train operations: orthogonalisation, norm, rounding and
// exact arithmetic (reference: pkg/src/ttss/tensor_train.py).
#pragma once

#include "common.h"

namespace t2s2 {

// Operator trains are handled through their merged-mode vector view
// (r0, m*n, r1) wherever the operation is mode-agnostic.
void right_orthonormalize(std::vector<DTensor>& cores);  // tensor_train.py:307
double tt_norm(const Train& t);                            // tensor_train.py:319
Train tt_round(const Train& t, double tol, int max_rank);  // tensor_train.py:327 / :616
Train tt_add(const Train& a, const Train& b, double sa = 1.0, double sb = 1.0);  // :253
Train tt_scale(const Train& a, double s);                  // :277
Train tt_apply(const Train& op, const Train& v);           // :359
double tt_dot(const Train& a, const Train& b);             // :296
void tt_full(const Train& v, double* host_out, size_t cap);  // :186
double compression_ratio(const Train& v);                    // :377

// Smallest k >= 1 whose singular-value tail ||s[k:]|| <= delta
// (tensor_train.py:143, tt_solver.py:249); host-side on read-back values.
int tail_keep(const std::vector<double>& s, double delta);

// Row/column scaling helpers used by the splits.
void scale_rows(double* X, int rows, int cols, int ld, const double* s);  // X[i,:] *= s[i]
void scale_cols(double* X, int rows, int cols, int ld, const double* s);  // X[:,j] *= s[j]

}  // namespace t2s2
