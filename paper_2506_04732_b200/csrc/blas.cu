// Dense fp64 kernels: tiled GEMM (FFMA), permutation, vector ops and
// deterministic reductions.
#include "blas.h"

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

namespace cg = cooperative_groups;

namespace t2s2 {

// ---------------------------------------------------------------------------
// GEMM: 64x64 output tile per CTA, BK = 16, 256 threads, 4x4 per thread.
// Operands are staged through shared memory with bounds checks so the same
// kernel serves the many tiny contractions of the sweep as well as the
// larger trailing updates.
// ---------------------------------------------------------------------------

namespace {

// Tile TM x TN x TK, 256 threads on a 16x16 grid (RM x RN outputs each).
// The next K-tile is fetched into registers while the current one is
// consumed from shared memory, so each tile costs one exposed L2 latency at
// most; small problems use 32x32x32 tiles to spread over more SMs.
// FP64 tensor-core MMA (DMMA, mma.sync m8n8k4): D[8x8] += A[8x4] B[4x8].
// Fragments: lane holds A[lane/4][lane%4], B[lane%4][lane/4],
// C/D[lane/4][2*(lane%4) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// One TM x TN output tile (tile coordinates bx, by of batch entry bz).
template <int TM, int TN, int TK, bool TC>
__device__ __forceinline__ void gemm_tile(bool ta, bool tb, int M, int N, int K, double alpha,
                                          const double* __restrict__ A, int lda, long long sA,
                                          const double* __restrict__ B, int ldb, long long sB,
                                          double beta, double* C, int ldc, long long sC, int bx,
                                          int by, int bz) {
  constexpr int PA = TM * TK / 256, PB = TK * TN / 256, RM = TM / 16, RN = TN / 16;
  __shared__ double As[TK][TM + 1];
  __shared__ double Bs[TK][TN + 1];
  A += bz * sA;
  B += bz * sB;
  C += bz * sC;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int row0 = by * TM, col0 = bx * TN;
  double ra[PA], rb[PB];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int t = 0; t < PA; ++t) {
      const int e = threadIdx.x + t * 256;
      int ar, ak;
      if (ta) {  // A^T: contiguous along rows of op(A) -> consecutive threads walk i
        ar = e % TM;
        ak = e / TM;
      } else {
        ar = e / TK;
        ak = e % TK;
      }
      const int gi = row0 + ar, gk = k0 + ak;
      ra[t] = (gi < M && gk < K) ? (ta ? A[(long long)gk * lda + gi] : A[(long long)gi * lda + gk])
                                 : 0.0;
    }
#pragma unroll
    for (int t = 0; t < PB; ++t) {
      const int e = threadIdx.x + t * 256;
      int bk, bc;
      if (tb) {
        bk = e % TK;
        bc = e / TK;
      } else {
        bk = e / TN;
        bc = e % TN;
      }
      const int gk = k0 + bk, gj = col0 + bc;
      rb[t] = (gk < K && gj < N) ? (tb ? B[(long long)gj * ldb + gk] : B[(long long)gk * ldb + gj])
                                 : 0.0;
    }
  };
  // FFMA path: 16x16 threads, RM x RN outputs each.  TC path: 8 warps on a
  // 4 x 2 grid of (TM/4) x (TN/2) warp tiles of 8x8 DMMA blocks.
  constexpr int WM = TM / 4, WN = TN / 2, MB = WM / 8, NB = WN / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm0 = (warp >> 1) * WM, wn0 = (warp & 1) * WN;
  double acc[RM][RN] = {};
  double tc[MB][NB][2] = {};
  fetch(0);
  for (int k0 = 0; k0 < K; k0 += TK) {
#pragma unroll
    for (int t = 0; t < PA; ++t) {
      const int e = threadIdx.x + t * 256;
      if (ta)
        As[e / TM][e % TM] = ra[t];
      else
        As[e % TK][e / TK] = ra[t];
    }
#pragma unroll
    for (int t = 0; t < PB; ++t) {
      const int e = threadIdx.x + t * 256;
      if (tb)
        Bs[e % TK][e / TK] = rb[t];
      else
        Bs[e / TN][e % TN] = rb[t];
    }
    __syncthreads();
    if (k0 + TK < K) fetch(k0 + TK);
    if (TC) {
#pragma unroll
      for (int kk = 0; kk < TK; kk += 4) {
        const int kr = kk + (lane & 3);
        double af[MB], bf[NB];
#pragma unroll
        for (int i = 0; i < MB; ++i) af[i] = As[kr][wm0 + i * 8 + (lane >> 2)];
#pragma unroll
        for (int j = 0; j < NB; ++j) bf[j] = Bs[kr][wn0 + j * 8 + (lane >> 2)];
#pragma unroll
        for (int i = 0; i < MB; ++i)
#pragma unroll
          for (int j = 0; j < NB; ++j) dmma_8x8x4(tc[i][j][0], tc[i][j][1], af[i], bf[j]);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        double a[RM], b[RN];
#pragma unroll
        for (int i = 0; i < RM; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < RN; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
    }
    __syncthreads();
  }
  if (TC) {
#pragma unroll
    for (int i = 0; i < MB; ++i) {
      const int gi = row0 + wm0 + i * 8 + (lane >> 2);
      if (gi >= M) continue;
#pragma unroll
      for (int j = 0; j < NB; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gj = col0 + wn0 + j * 8 + (lane & 3) * 2 + h;
          if (gj >= N) continue;
          double* c = C + (long long)gi * ldc + gj;
          *c = beta == 0.0 ? alpha * tc[i][j][h] : alpha * tc[i][j][h] + beta * (*c);
        }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const int gi = row0 + ty + 16 * i;
    if (gi >= M) continue;
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int gj = col0 + tx + 16 * j;
      if (gj >= N) continue;
      double* c = C + (long long)gi * ldc + gj;
      *c = beta == 0.0 ? alpha * acc[i][j] : alpha * acc[i][j] + beta * (*c);
    }
  }
}

template <int TM, int TN, int TK, bool TC>
__global__ void __launch_bounds__(256) gemm_kernel(bool ta, bool tb, int M, int N, int K,
                                                   double alpha, const double* __restrict__ A,
                                                   int lda, long long sA,
                                                   const double* __restrict__ B, int ldb,
                                                   long long sB, double beta, double* C, int ldc,
                                                   long long sC) {
  gemm_tile<TM, TN, TK, TC>(ta, tb, M, N, K, alpha, A, lda, sA, B, ldb, sB, beta, C, ldc, sC,
                            blockIdx.x, blockIdx.y, blockIdx.z);
}

// A GEMM program: stages of independent strided-batched GEMMs, one
// cooperative launch, a grid barrier between stages.  Chains of small
// contractions (the interface recurrences of a move, the local right-hand
// sides, the operator applications) run as one kernel instead of one launch
// per GEMM.
__global__ void __launch_bounds__(256) gemm_program_kernel(const __grid_constant__ GemmProgram prog) {
  cg::grid_group grid = cg::this_grid();
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
      const int tn = (g.N + 31) / 32, tm = (g.M + 31) / 32;
      const int bz = tt / (tm * tn), rem = tt - bz * tm * tn;
      gemm_tile<32, 32, 32, true>(g.ta, g.tb, g.M, g.N, g.K, g.alpha, g.A, g.lda, g.sA, g.B, g.ldb,
                                  g.sB, g.beta, g.C, g.ldc, g.sC, rem % tn, rem / tn, bz);
    }
    if (s + 1 < prog.nstage) grid.sync();
  }
}

struct PermArgs {
  int nd;
  int out_shape[8];
  long long in_stride[8];  // stride in the input of output axis k
};

// 32-bit index math (every local tensor has < 2^31 entries).
__global__ void permute_kernel(const double* __restrict__ in, double* __restrict__ out, int n,
                               PermArgs a) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) {
    unsigned rem = (unsigned)o;
    unsigned off = 0;
    for (int k = a.nd - 1; k >= 0; --k) {
      const unsigned d = (unsigned)a.out_shape[k];
      const unsigned q = rem / d;
      off += (rem - q * d) * (unsigned)a.in_stride[k];
      rem = q;
    }
    out[o] = in[off];
  }
}

__global__ void fill_kernel(double* x, double v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = v;
}

__global__ void scal_kernel(double* x, double s, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] *= s;
}

__global__ void axpby_kernel(double a, const double* x, double b, double* y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = a * x[i] + b * y[i];
}

__global__ void copy2d_kernel(double* dst, int ldd, const double* src, int lds, int rows,
                              int cols) {
  long long n = (long long)rows * cols;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (int)n;
       e += gridDim.x * blockDim.x) {
    int r = (int)(e / cols), c = (int)(e % cols);
    dst[(long long)r * ldd + c] = src[(long long)r * lds + c];
  }
}

// Block-level sum of one double per thread (blockDim multiple of 32).
__device__ double block_sum(double v) {
  __shared__ double warp_part[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) warp_part[w] = v;
  __syncthreads();
  int nw = blockDim.x >> 5;
  v = lane < nw ? warp_part[lane] : 0.0;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // valid in warp 0
}

__global__ void dot_partial_kernel(const double* x, const double* y, long long n, double* part) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    s = fma(x[i], y[i], s);
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_final_kernel(const double* part, int n, double* out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) *out = s;
}

__global__ void transpose_kernel(const double* in, double* out, int rows, int cols) {
  long long n = (long long)rows * cols;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (int)n;
       e += gridDim.x * blockDim.x) {
    int r = (int)(e / cols), c = (int)(e % cols);
    out[(long long)c * rows + r] = in[e];
  }
}

int grid_for(long long n, int threads = 256, int cap = 1184) {
  long long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace

void gemm_batched(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int lda,
                  long long sA, const double* B, int ldb, long long sB, double beta, double* C,
                  int ldc, long long sC, int batch) {
  if (M <= 0 || N <= 0 || batch <= 0) return;
  if (K <= 0) {
    // C = beta * C
    for (int b = 0; b < batch; ++b)
      for (int i = 0; i < M; ++i) {
        if (beta == 0.0)
          dfill(C + b * sC + (long long)i * ldc, 0.0, N);
        else
          dscal(C + b * sC + (long long)i * ldc, beta, N);
      }
    return;
  }
  const bool big = (long long)ceil_div(M, 64) * ceil_div(N, 64) * batch >= 74;
  {
    LaunchScope ls("gemm", 2.0*M*N*(double)K*batch, 8.0*batch*((double)M*K+(double)K*N+2.0*M*N));
    if (big) {
      dim3 grid(ceil_div(N, 64), ceil_div(M, 64), batch);
      gemm_kernel<64, 64, 16, true><<<grid, 256, 0, stream()>>>(ta, tb, M, N, K, alpha, A, lda, sA,
                                                                B, ldb, sB, beta, C, ldc, sC);
    } else {
      dim3 grid(ceil_div(N, 32), ceil_div(M, 32), batch);
      gemm_kernel<32, 32, 32, true><<<grid, 256, 0, stream()>>>(ta, tb, M, N, K, alpha, A, lda, sA,
                                                                B, ldb, sB, beta, C, ldc, sC);
    }
  }
  T2S2_CHECK_LAUNCH();
}

double* GemmBatch::temp(std::vector<int> shape) {
  temps_.emplace_back(std::move(shape));
  return temps_.back().p;
}

void GemmBatch::add(int stage, bool ta, bool tb, int M, int N, int K, const double* A, int lda,
                    long long sA, const double* B, int ldb, long long sB, double* C, int ldc,
                    long long sC, int batch, double alpha, double beta) {
  if (M <= 0 || N <= 0 || batch <= 0) return;
  T2S2_REQUIRE(K > 0, kErrShape, "GemmBatch: empty contraction");
  GemmProb g{};
  g.A = A;
  g.B = B;
  g.C = C;
  g.sA = sA;
  g.sB = sB;
  g.sC = sC;
  g.M = M;
  g.N = N;
  g.K = K;
  g.lda = lda;
  g.ldb = ldb;
  g.ldc = ldc;
  g.batch = batch;
  g.ta = ta;
  g.tb = tb;
  g.alpha = alpha;
  g.beta = beta;
  g.tiles = ceil_div(M, 32) * ceil_div(N, 32) * batch;
  items_.push_back({stage, g});
  flops_ += 2.0 * M * N * (double)K * batch;
}

void GemmBatch::run() {
  if (items_.empty()) return;
  std::stable_sort(items_.begin(), items_.end(),
                   [](const Item& x, const Item& y) { return x.stage < y.stage; });
  // split into programs of at most kProgMaxProb problems / kProgMaxStage stages
  size_t i = 0;
  while (i < items_.size()) {
    GemmProgram prog{};
    int last_stage = -1, max_tiles = 0, stage_tiles = 0;
    while (i < items_.size() && prog.nprob < kProgMaxProb) {
      const Item& it = items_[i];
      if (it.stage != last_stage) {
        if (prog.nstage == kProgMaxStage) break;
        prog.stage_first[prog.nstage++] = prog.nprob;
        last_stage = it.stage;
        stage_tiles = 0;
      }
      prog.p[prog.nprob++] = it.g;
      stage_tiles += it.g.tiles;
      max_tiles = stage_tiles > max_tiles ? stage_tiles : max_tiles;
      ++i;
    }
    // a stage cut by the problem limit continues in the next program
    prog.stage_first[prog.nstage] = prog.nprob;
    static int nsm = 0;
    if (nsm == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    int grid = max_tiles < nsm ? max_tiles : nsm;
    if (sm_budget() > 0 && grid > sm_budget()) grid = sm_budget();
    if (grid < 1) grid = 1;
    {
      LaunchScope ls("gemm", flops_ * prog.nprob / (double)items_.size(), 0.0);
      if (prog.nstage == 1) {
        gemm_program_kernel<<<grid, 256, 0, stream()>>>(prog);
      } else {
        void* params[] = {&prog};
        T2S2_CUDA(cudaLaunchCooperativeKernel((void*)gemm_program_kernel, dim3(grid), dim3(256),
                                              params, 0, stream()));
      }
    }
    T2S2_CHECK_LAUNCH();
  }
  items_.clear();
  temps_.clear();  // stream-ordered: safe to recycle once the launch is enqueued
  flops_ = 0.0;
}

void gemm(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int lda,
          const double* B, int ldb, double beta, double* C, int ldc) {
  gemm_batched(ta, tb, M, N, K, alpha, A, lda, 0, B, ldb, 0, beta, C, ldc, 0, 1);
}

DTensor permute(const DTensor& a, const std::vector<int>& perm) {
  int nd = a.ndim();
  T2S2_REQUIRE((int)perm.size() == nd && nd <= 8, kErrShape, "permute: bad axes");
  bool ident = true;
  for (int k = 0; k < nd; ++k) ident = ident && perm[k] == k;
  std::vector<int> os(nd);
  for (int k = 0; k < nd; ++k) os[k] = a.shape[perm[k]];
  DTensor out(os);
  if (ident) {
    dcopy(out.p, a.p, a.size());
    return out;
  }
  std::vector<long long> st(nd);
  long long s = 1;
  for (int k = nd - 1; k >= 0; --k) {
    st[k] = s;
    s *= a.shape[k];
  }
  PermArgs pa{};
  pa.nd = nd;
  for (int k = 0; k < nd; ++k) {
    pa.out_shape[k] = os[k];
    pa.in_stride[k] = st[perm[k]];
  }
  long long n = (long long)a.size();
  {
    LaunchScope ls("permute", 0, 16.0*n);
    permute_kernel<<<grid_for(n), 256, 0, stream()>>>(a.p, out.p, (int)n, pa);
  }
  T2S2_CHECK_LAUNCH();
  return out;
}

DTensor tensordot(const DTensor& a, const std::vector<int>& axa, const DTensor& b,
                  const std::vector<int>& axb) {
  T2S2_REQUIRE(axa.size() == axb.size(), kErrShape, "tensordot: axis count mismatch");
  int na = a.ndim(), nb = b.ndim();
  std::vector<int> fa, fb, norm_a, norm_b;
  std::vector<bool> ca(na, false), cb(nb, false);
  long long K = 1;
  for (size_t i = 0; i < axa.size(); ++i) {
    int ia = axa[i] < 0 ? axa[i] + na : axa[i];
    int ib = axb[i] < 0 ? axb[i] + nb : axb[i];
    T2S2_REQUIRE(a.shape[ia] == b.shape[ib], kErrShape, "tensordot: contracted size mismatch");
    ca[ia] = true;
    cb[ib] = true;
    norm_a.push_back(ia);
    norm_b.push_back(ib);
    K *= a.shape[ia];
  }
  long long M = 1, N = 1;
  std::vector<int> out_shape;
  for (int k = 0; k < na; ++k)
    if (!ca[k]) {
      fa.push_back(k);
      M *= a.shape[k];
      out_shape.push_back(a.shape[k]);
    }
  for (int k = 0; k < nb; ++k)
    if (!cb[k]) {
      fb.push_back(k);
      N *= b.shape[k];
      out_shape.push_back(b.shape[k]);
    }
  // A as (free, contracted) or, if already laid out (contracted, free), transposed.
  std::vector<int> pa_fc = fa, pa_cf = norm_a;
  pa_fc.insert(pa_fc.end(), norm_a.begin(), norm_a.end());
  pa_cf.insert(pa_cf.end(), fa.begin(), fa.end());
  std::vector<int> pb_cf = norm_b, pb_fc = fb;
  pb_cf.insert(pb_cf.end(), fb.begin(), fb.end());
  pb_fc.insert(pb_fc.end(), norm_b.begin(), norm_b.end());
  auto is_id = [](const std::vector<int>& p) {
    for (size_t k = 0; k < p.size(); ++k)
      if (p[k] != (int)k) return false;
    return true;
  };
  DTensor ta_buf, tb_buf;
  const double* Ap;
  const double* Bp;
  bool transA = false, transB = false;
  if (is_id(pa_fc)) {
    Ap = a.p;
  } else if (is_id(pa_cf)) {
    Ap = a.p;
    transA = true;
  } else {
    ta_buf = permute(a, pa_fc);
    Ap = ta_buf.p;
  }
  if (is_id(pb_cf)) {
    Bp = b.p;
  } else if (is_id(pb_fc)) {
    Bp = b.p;
    transB = true;
  } else {
    tb_buf = permute(b, pb_cf);
    Bp = tb_buf.p;
  }
  if (out_shape.empty()) out_shape.push_back(1);
  DTensor out(out_shape);
  int lda = transA ? (int)M : (int)K;
  int ldb = transB ? (int)K : (int)N;
  gemm(transA, transB, (int)M, (int)N, (int)K, 1.0, Ap, lda, Bp, ldb, 0.0, out.p, (int)N);
  return out;
}

void transpose(const double* in, double* out, int rows, int cols) {
  long long n = (long long)rows * cols;
  if (n <= 0) return;
  {
    LaunchScope ls("permute", 0, 16.0*n);
    transpose_kernel<<<grid_for(n), 256, 0, stream()>>>(in, out, rows, cols);
  }
  T2S2_CHECK_LAUNCH();
}

void dcopy(double* dst, const double* src, size_t n) {
  if (n) T2S2_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
}

void dfill(double* dst, double v, size_t n) {
  if (!n) return;
  {
    LaunchScope ls("vector", 0, 8.0*n);
    fill_kernel<<<grid_for((long long)n), 256, 0, stream()>>>(dst, v, (long long)n);
  }
  T2S2_CHECK_LAUNCH();
}

void dscal(double* x, double s, size_t n) {
  if (!n) return;
  {
    LaunchScope ls("vector", n, 16.0*n);
    scal_kernel<<<grid_for((long long)n), 256, 0, stream()>>>(x, s, (long long)n);
  }
  T2S2_CHECK_LAUNCH();
}

void daxpby(double a, const double* x, double b, double* y, size_t n) {
  if (!n) return;
  {
    LaunchScope ls("vector", 3.0*n, 24.0*n);
    axpby_kernel<<<grid_for((long long)n), 256, 0, stream()>>>(a, x, b, y, (long long)n);
  }
  T2S2_CHECK_LAUNCH();
}

void daxpy(double a, const double* x, double* y, size_t n) { daxpby(a, x, 1.0, y, n); }

void copy2d(double* dst, int ldd, const double* src, int lds, int rows, int cols) {
  long long n = (long long)rows * cols;
  if (n <= 0) return;
  {
    LaunchScope ls("vector", 0, 16.0*n);
    copy2d_kernel<<<grid_for(n), 256, 0, stream()>>>(dst, ldd, src, lds, rows, cols);
  }
  T2S2_CHECK_LAUNCH();
}

void ddot_dev(const double* x, const double* y, size_t n, double* out) {
  int g = grid_for((long long)n, 256, 296);
  double* part = allocator().alloc(g);
  {
    LaunchScope ls("reduce", 2.0*n, 16.0*n);
    dot_partial_kernel<<<g, 256, 0, stream()>>>(x, y, (long long)n, part);
  }
  {
    LaunchScope ls("reduce", 0, 0);
    sum_final_kernel<<<1, 256, 0, stream()>>>(part, g, out);
  }
  T2S2_CHECK_LAUNCH();
  allocator().release(part);
}

double scalar_to_host(const double* d) {
  double h = 0.0;
  T2S2_CUDA(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, stream()));
  T2S2_CUDA(cudaStreamSynchronize(stream()));
  return h;
}

double ddot(const double* x, const double* y, size_t n) {
  double* o = allocator().alloc(1);
  ddot_dev(x, y, n, o);
  double h = scalar_to_host(o);
  allocator().release(o);
  return h;
}

double dnrm2(const double* x, size_t n) { return std::sqrt(ddot(x, x, n)); }

void to_host(double* h, const double* d, size_t n) {
  if (n) T2S2_CUDA(cudaMemcpyAsync(h, d, n * sizeof(double), cudaMemcpyDeviceToHost, stream()));
  T2S2_CUDA(cudaStreamSynchronize(stream()));
}

void to_device(double* d, const double* h, size_t n) {
  if (n) T2S2_CUDA(cudaMemcpyAsync(d, h, n * sizeof(double), cudaMemcpyHostToDevice, stream()));
}

DTensor DTensor::clone() const {
  DTensor o(shape);
  dcopy(o.p, p, size());
  return o;
}

Train Train::clone() const {
  Train t;
  t.rows = rows;
  t.cols = cols;
  for (auto& c : cores) t.cores.push_back(c.clone());
  return t;
}

}  // namespace t2s2
