// Restarted GMRES and Jacobi-preconditioned CG for the local systems that
// exceed the direct-solve size (reference: tt_solver.py:375-414, which calls
// scipy.sparse.linalg.gmres(restart=40, maxiter=10) and cg(maxiter=250)).
//
// The Krylov recurrences follow scipy 1.18's pure-Python implementations
// (modified Gram-Schmidt Arnoldi with LAPACK-style Givens rotations and the
// gh-8400 inner-tolerance control; textbook PCG), with every vector and
// scalar resident on the device.  GMRES: the host polls a convergence flag
// every few iterations; PCG: the loop runs on the device.
#pragma once

#include <functional>

#include "blas.h"
#include "common.h"

namespace t2s2 {

// out = A in.  guard (device int, may be null): when it reads 0 on the
// device the application is skipped (a Krylov loop that converged between
// two host polls does not pay for its trailing matvecs).
using MatVec = std::function<void(const double* in, double* out, const int* guard)>;

// x (device, length n) is the initial guess and receives the result.
// rtol relative to ||b|| (scipy's atol = rtol * ||b||).  Returns inner
// iterations performed.
int gmres(const MatVec& A, int n, const double* b, double* x, double rtol, int restart,
          int maxiter);

// Adds the problems of out = A in to a GEMM batch (stages from 0).
using ProgramBuilder = std::function<void(GemmBatch& gb, const double* in, double* out)>;

// Preconditioner M = diag^{-1}.  The whole iteration loop is one cooperative
// kernel with the matvec program inside it.
int pcg(const ProgramBuilder& A, int n, const double* b, double* x, const double* diag, double rtol,
        int maxiter);

}  // namespace t2s2
