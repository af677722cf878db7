// Dense fp64 building blocks on device arrays: GEMM, permutation,
// tensordot, vector ops and deterministic reductions.
#pragma once

#include <initializer_list>
#include <utility>

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
constexpr int kProgMaxProb = 20;
constexpr int kProgMaxStage = 24;
struct GemmProb {
  // A(i,k) = A[(i / ad) * ahi + (i % ad) * alo + k * ak]: a two-level row
  // index folds a batch (or a split row index) into one large GEMM;
  // B(k,j) = B[k * bk + j * bj]; C(i,j) = C[(i / cd) * chi + (i % cd) * clo + j * cj].
  const double* A;
  const double* B;
  double* C;
  long long sA, sB, sC;  // strides of the explicit batch index
  long long ahi, alo, ak, bk, bj, chi, clo, cj;
  int ad, cd;
  int M, N, K, batch, tiles;
  int big;   // 2: 64x136x16 tiles (65 <= N <= 136), 1: 64x64x16, 0: 32x32x32
  int kind;  // 0 GEMM; 1 split-K reduction: C = alpha sum_j A[j] + beta C (A: batch x M x N)
  double alpha, beta;
  const double* rs;  // optional epilogue scales (beta == 0 only): C(i,j) = alpha acc rs[i] cs[j]
  const double* cs;
};

struct GemmProgram {
  const int* guard;  // device flag: the program does nothing while it reads 0 (null: run)
  int nprob, nstage;
  int stage_first[kProgMaxStage + 1];
  GemmProb p[kProgMaxProb];
};

// Operand with a two-level row index (see GemmProb): element (i, k) at
// p + (i / d) * hi + (i % d) * lo + k * k_stride (+ batch stride).
struct GemmOperand {
  const double* p;
  int d;
  long long hi, lo, k, batch;
};

class GemmBatch {
 public:
  // scratch that lives until run() has enqueued the program
  double* temp(std::vector<int> shape);
  void add(int stage, bool ta, bool tb, int M, int N, int K, const double* A, int lda, long long sA,
           const double* B, int ldb, long long sB, double* C, int ldc, long long sC, int batch = 1,
           double alpha = 1.0, double beta = 0.0);
  // C = alpha op(A) B + beta C with general operand addressing
  void add_general(int stage, int M, int N, int K, const GemmOperand& a, const double* B,
                   long long bk, long long bj, long long sB, const GemmOperand& c, int batch = 1,
                   double alpha = 1.0, double beta = 0.0);
  // scale the rows / columns of the last added problem's result (plain
  // batch-1 problems with beta = 0; after a split-K the scales go to its
  // reduction): the product of copy + scale_rows/cols
  void scale_last(const double* rs, const double* cs);
  void run();
  void set_guard(const int* g) { guard_ = g; }
  // The added problems as ONE program for a kernel that runs it inside its
  // own loop (gemm_device.cuh; the Krylov solvers): false when they do not
  // fit one program.  wide: the program needs the 64x136 instantiation;
  // max_tiles: the largest stage.  The scratch of temp() lives until the
  // batch is destroyed.
  bool build_program(GemmProgram& prog, bool& wide, int& max_tiles, double& flops);

 private:
  const int* guard_ = nullptr;
  struct Item {
    int stage;
    GemmProb g;
  };
  std::vector<Item> items_;
  std::vector<DTensor> temps_;
  double flops_ = 0.0;
};

// dynamic shared memory of a kernel running programs (gemm_device.cuh)
int gemm_program_smem(bool wide);

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
// dst[i, j] = src[i, j] * rs[i] * cs[j] (a null scale is 1; with one scale the
// product is the single rounding of copy2d followed by scale_rows/scale_cols)
void copy_scaled(double* dst, int ldd, const double* src, int lds, int rows, int cols,
                 const double* rs, const double* cs);
// copy2d(d1 <- s1, r1 x c1) and copy_scaled(d2 <- s2 with row scales rs, r2 x c2) in one launch
void copy_and_scaled(double* d1, int ldd1, const double* s1, int lds1, int r1, int c1, double* d2,
                     int ldd2, const double* s2, int lds2, int r2, int c2, const double* rs);
// The data movements that finish a split of a solved core, in ONE launch:
//   0: d0[i, j] = s0[i, j] * rs[i] * cs[j]   (rows0 x cols0; a null scale is 1)
//   1: d1[r, :c1] = a1[r, :c1], d1[r, c1:c1+c2] = b1[r, :c2]   (rows1 rows)
//   2: d2[0 .. n2) = 0
struct SplitFinish {
  double* d0;
  const double* s0;
  int ldd0, lds0, rows0, cols0;
  const double* rs;
  const double* cs;
  double* d1;
  const double* a1;
  const double* b1;
  int ldd1, lda1, ldb1, c1, c2, rows1;
  double* d2;
  long long n2;
};
void split_finish(const SplitFinish& a);
// dst[:, :c1] = s1, dst[:, c1:c1+c2] = s2 (rows x ...), one launch
void copy2d_pair(double* dst, int ldd, const double* s1, int ld1, int c1, const double* s2, int ld2,
                 int c2, int rows);
// fill several arrays with one value in one launch (at most 8)
void fill_many(std::initializer_list<std::pair<double*, size_t>> arrays, double v);
// copies of a set of arrays, eight per launch (instead of one copy-engine node each)
std::vector<DTensor> clone_all(const std::vector<DTensor>& v);
// concatenate up to 4 device arrays into dst in one launch
void pack(double* dst, std::initializer_list<std::pair<const double*, size_t>> parts);

// out (cols x rows) = in^T for a row-major rows x cols matrix.
void transpose(const double* in, double* out, int rows, int cols);

// Small host<->device helpers on the context stream.
void to_host(double* h, const double* d, size_t n);  // synchronises
void to_device(double* d, const double* h, size_t n);
double scalar_to_host(const double* d);

}  // namespace t2s2
