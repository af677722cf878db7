// Restarted GMRES and Jacobi-preconditioned CG for the local systems that
// exceed the direct-solve size (reference: tt_solver.py:375-414, which calls
// scipy.sparse.linalg.gmres(restart=40, maxiter=10) and cg(maxiter=250)).
//
// The Krylov recurrences follow scipy 1.18's pure-Python implementations
// (modified Gram-Schmidt Arnoldi with LAPACK-style Givens rotations and the
// gh-8400 inner-tolerance control; textbook PCG), with every vector and
// scalar resident on the device; the iteration loops run on the device.
#pragma once

#include <functional>

#include "blas.h"
#include "common.h"

namespace t2s2 {

// Adds the problems of out = A in to a GEMM batch (stages from 0).  The
// solvers run the matvec as a program inside their own kernels; an operator
// whose matvec does not fit one program gets it as a separate launch per
// iteration, skipped on the device once the loop has converged.
using ProgramBuilder = std::function<void(GemmBatch& gb, const double* in, double* out)>;

// x (device, length n) is the initial guess and receives the result.
// rtol relative to ||b|| (scipy's atol = rtol * ||b||).  Returns inner
// iterations performed.  One cooperative kernel per restart cycle (the
// column loop with matvec and Arnoldi step); the host runs the restart logic.
int gmres(const ProgramBuilder& A, int n, const double* b, double* x, double rtol, int restart,
          int maxiter);

// Preconditioner M = diag^{-1}.  The whole iteration loop is one cooperative
// kernel with the matvec program inside it.
int pcg(const ProgramBuilder& A, int n, const double* b, double* x, const double* diag, double rtol,
        int maxiter);

}  // namespace t2s2
