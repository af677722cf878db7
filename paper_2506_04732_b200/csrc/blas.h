// Dense fp64 building blocks on device arrays: GEMM, permutation,
// tensordot, vector ops and deterministic reductions.
#pragma once

#include "common.h"

namespace t2s2 {

// C[M,N] = alpha * op(A)[M,K] * op(B)[K,N] + beta * C, row-major with
// leading dimensions; op(X) = X^T when the flag is set.
void gemm(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int lda,
          const double* B, int ldb, double beta, double* C, int ldc);

// Strided batch of the same GEMM (batch strides in elements).
void gemm_batched(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int lda,
                  long long sA, const double* B, int ldb, long long sB, double beta, double* C,
                  int ldc, long long sC, int batch);

// A program of strided-batched GEMMs in stages: the problems of a stage are
// independent, stage s+1 may read what stage s wrote.  One (cooperative)
// launch per program with a grid barrier between stages.
constexpr int kProgMaxProb = 24;
constexpr int kProgMaxStage = 24;
struct GemmProb {
  const double* A;
  const double* B;
  double* C;
  long long sA, sB, sC;
  int M, N, K, lda, ldb, ldc, batch, tiles;
  int ta, tb;
  double alpha, beta;
};
struct GemmProgram {
  int nprob, nstage;
  int stage_first[kProgMaxStage + 1];
  GemmProb p[kProgMaxProb];
};

class GemmBatch {
 public:
  // scratch that lives until run() has enqueued the program
  double* temp(std::vector<int> shape);
  void add(int stage, bool ta, bool tb, int M, int N, int K, const double* A, int lda, long long sA,
           const double* B, int ldb, long long sB, double* C, int ldc, long long sC, int batch = 1,
           double alpha = 1.0, double beta = 0.0);
  void run();

 private:
  struct Item {
    int stage;
    GemmProb g;
  };
  std::vector<Item> items_;
  std::vector<DTensor> temps_;
  double flops_ = 0.0;
};

DTensor permute(const DTensor& a, const std::vector<int>& perm);

// numpy.tensordot semantics: result axes are the free axes of a (in order)
// followed by the free axes of b (in order).
DTensor tensordot(const DTensor& a, const std::vector<int>& axa, const DTensor& b,
                  const std::vector<int>& axb);

void dcopy(double* dst, const double* src, size_t n);
void dfill(double* dst, double v, size_t n);
void dscal(double* x, double s, size_t n);
void daxpy(double a, const double* x, double* y, size_t n);  // y += a x
// y[i] = a*x[i] + b*y[i]
void daxpby(double a, const double* x, double b, double* y, size_t n);

// Deterministic (fixed-shape tree) reductions.  The *_dev variants leave
// the scalar in device memory; the others synchronise and return it.
void ddot_dev(const double* x, const double* y, size_t n, double* out);
double ddot(const double* x, const double* y, size_t n);
double dnrm2(const double* x, size_t n);

// Copy a (rows x cols) block between row-major arrays with leading dims.
void copy2d(double* dst, int ldd, const double* src, int lds, int rows, int cols);

// out (cols x rows) = in^T for a row-major rows x cols matrix.
void transpose(const double* in, double* out, int rows, int cols);

// Small host<->device helpers on the context stream.
void to_host(double* h, const double* d, size_t n);  // synchronises
void to_device(double* d, const double* h, size_t n);
double scalar_to_host(const double* d);

}  // namespace t2s2
