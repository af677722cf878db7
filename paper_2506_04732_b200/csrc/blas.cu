// Dense fp64 kernels: tiled GEMM (DMMA), permutation, vector ops and
// deterministic reductions.
#include "blas.h"
#include "gemm_device.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace t2s2 {

// ---------------------------------------------------------------------------
// GEMM: 32x32x32 or 64x64x16 output tiles per CTA, 256 threads (8 warps of
// DMMA).  Operands are staged through shared memory with bounds checks so the same
// kernel serves the many tiny contractions of the sweep as well as the
// larger trailing updates.
// ---------------------------------------------------------------------------

namespace {

using gemm_device::kGemmSmem;
using gemm_device::kGemmSmemWide;
using gemm_device::kReduceTile;
using gemm_device::kWideN;

// A GEMM program: stages of independent strided-batched GEMMs, one
// cooperative launch, a grid barrier between stages (gemm_device.cuh).
// Chains of small contractions (the interface recurrences of a move, the
// local right-hand sides, the operator applications) run as one kernel
// instead of one launch per GEMM.  Two CTAs per SM (<= 128 registers).
template <bool WIDE>
__global__ void __launch_bounds__(256, 2) gemm_program_kernel(const __grid_constant__ GemmProgram prog) {
  extern __shared__ __align__(16) double gemm_smem[];
  cg::grid_group grid = cg::this_grid();
  if (prog.guard && *prog.guard == 0) return;  // uniform over the grid: flag set by an earlier kernel
  gemm_device::gemm_program_run<WIDE>(prog, gemm_smem, grid);
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

__global__ void copy_scaled_kernel(double* dst, int ldd, const double* src, int lds, int rows,
                                   int cols, const double* rs, const double* cs) {
  const int n = rows * cols;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int r = e / cols, c = e - r * cols;
    double v = src[(long long)r * lds + c];
    if (rs) v *= rs[r];
    if (cs) v *= cs[c];
    dst[(long long)r * ldd + c] = v;
  }
}

// blockIdx.y = 0: d1 = s1 (r1 x c1 block copy); 1: d2[i, j] = s2[i, j] * rs[i]
__global__ void copy_and_scaled_kernel(double* d1, int ldd1, const double* s1, int lds1, int r1, int c1,
                                       double* d2, int ldd2, const double* s2, int lds2, int r2, int c2,
                                       const double* rs) {
  if (blockIdx.y == 0) {
    const int n = r1 * c1;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
      const int r = e / c1, c = e - r * c1;
      d1[(long long)r * ldd1 + c] = s1[(long long)r * lds1 + c];
    }
  } else {
    const int n = r2 * c2;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
      const int r = e / c2, c = e - r * c2;
      d2[(long long)r * ldd2 + c] = s2[(long long)r * lds2 + c] * rs[r];
    }
  }
}

// The three data movements that finish a split, blockIdx.y = 0, 1, 2 (see
// SplitFinish in blas.h); each element gets the arithmetic of copy_scaled /
// copy2d_pair / fill.
__global__ void split_finish_kernel(const __grid_constant__ SplitFinish a) {
  const int stride = gridDim.x * blockDim.x, t0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.y == 0) {
    const int n = a.rows0 * a.cols0;
    for (int e = t0; e < n; e += stride) {
      const int r = e / a.cols0, c = e - r * a.cols0;
      double v = a.s0[(long long)r * a.lds0 + c];
      if (a.rs) v *= a.rs[r];
      if (a.cs) v *= a.cs[c];
      a.d0[(long long)r * a.ldd0 + c] = v;
    }
  } else if (blockIdx.y == 1) {
    const int cols = a.c1 + a.c2, n = a.rows1 * cols;
    for (int e = t0; e < n; e += stride) {
      const int r = e / cols, c = e - r * cols;
      a.d1[(long long)r * a.ldd1 + c] =
          c < a.c1 ? a.a1[(long long)r * a.lda1 + c] : a.b1[(long long)r * a.ldb1 + c - a.c1];
    }
  } else {
    for (long long e = t0; e < a.n2; e += stride) a.d2[e] = 0.0;
  }
}

__global__ void copy2d_pair_kernel(double* dst, int ldd, const double* s1, int ld1, int c1,
                                   const double* s2, int ld2, int c2, int rows) {
  const int cols = c1 + c2, n = rows * cols;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int r = e / cols, c = e - r * cols;
    dst[(long long)r * ldd + c] = c < c1 ? s1[(long long)r * ld1 + c] : s2[(long long)r * ld2 + c - c1];
  }
}

struct Segments {
  double* dst[8];
  const double* src[8];
  long long n[8];
  int k;
  double v;
};

// fill (src == null) or copy segments; blockIdx.y = segment
__global__ void segments_kernel(Segments a) {
  const int q = blockIdx.y;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < a.n[q];
       e += (long long)gridDim.x * blockDim.x)
    a.dst[q][e] = a.src[q] ? a.src[q][e] : a.v;
}

__global__ void dot_partial_kernel(const double* x, const double* y, long long n, double* part) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    s = fma(x[i], y[i], s);
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// (an open read ticket: the sum is also published to the host, see common.h)
__global__ void sum_final_kernel(const double* part, int n, double* out, ReadTicket t) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) *out = s;
  if (t.dst) {
    __syncthreads();
    publish_words(t, reinterpret_cast<const unsigned*>(out), 2);
  }
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
  GemmBatch gb;
  gb.add(0, ta, tb, M, N, K, A, lda, sA, B, ldb, sB, C, ldc, sC, batch, alpha, beta);
  gb.run();
}

double* GemmBatch::temp(std::vector<int> shape) {
  temps_.emplace_back(std::move(shape));
  return temps_.back().p;
}

void GemmBatch::add(int stage, bool ta, bool tb, int M, int N, int K, const double* A, int lda,
                    long long sA, const double* B, int ldb, long long sB, double* C, int ldc,
                    long long sC, int batch, double alpha, double beta) {
  if (batch > 1 && sA == 0) {
    // shared left factor: the batch folds into the rows of one GEMM,
    // C_b^T = B_b^T A^T stacked over b (two-level row index (b, n))
    GemmOperand a2{B, N, sB, tb ? (long long)ldb : 1, tb ? 1 : (long long)ldb, 0};
    GemmOperand c2{C, N, sC, 1, ldc, 0};
    add_general(stage, batch * N, M, K, a2, A, ta ? (long long)lda : 1, ta ? 1 : (long long)lda, 0,
                c2, 1, alpha, beta);
    return;
  }
  GemmOperand a{A, 1 << 30, 0, ta ? 1 : lda, ta ? lda : 1, sA};
  GemmOperand c{C, 1 << 30, 0, ldc, 1, sC};
  add_general(stage, M, N, K, a, B, tb ? 1 : ldb, tb ? ldb : 1, sB, c, batch, alpha, beta);
}

void GemmBatch::add_general(int stage, int M, int N, int K, const GemmOperand& a, const double* B,
                            long long bk, long long bj, long long sB, const GemmOperand& c,
                            int batch, double alpha, double beta) {
  if (M <= 0 || N <= 0 || batch <= 0) return;
  T2S2_REQUIRE(K > 0, kErrShape, "GemmBatch: empty contraction");
  GemmProb g{};
  g.A = a.p;
  g.ad = a.d;
  g.ahi = a.hi;
  g.alo = a.lo;
  g.ak = a.k;
  g.sA = a.batch;
  g.B = B;
  g.bk = bk;
  g.bj = bj;
  g.sB = sB;
  g.C = const_cast<double*>(c.p);
  g.cd = c.d;
  g.chi = c.hi;
  g.clo = c.lo;
  g.cj = c.k;
  g.sC = c.batch;
  g.M = M;
  g.N = N;
  g.K = K;
  g.batch = batch;
  g.alpha = alpha;
  g.beta = beta;
  // 64x64 tiles once a problem fills the GPU with them (more reuse per L2
  // byte); for 64 < N <= 136 — the operator-core stages of a config-4
  // matvec, N = n * rA = 132 — one 64 x 136 tile covers all columns (64-wide
  // tiles would compute 192 columns for 132)
  g.big = M >= 64 && N >= 64 && K >= 64 &&
          (long long)ceil_div(M, 64) * ceil_div(N, 64) * batch >= 148;
  if (g.big && N > 64 && N <= kWideN) g.big = 2;
  g.tiles = g.big == 2 ? ceil_div(M, 64) * batch
            : g.big    ? ceil_div(M, 64) * ceil_div(N, 64) * batch
                       : ceil_div(M, 32) * ceil_div(N, 32) * batch;
  flops_ += 2.0 * M * N * (double)K * batch;
  // split-K for long contractions with too few output tiles to fill the GPU:
  // partial products at stage 2s, their deterministic sum at stage 2s+1
  constexpr int kFill = 592;  // two waves of two CTAs per SM
  if (batch == 1 && K >= 256 && g.tiles < kFill / 2) {
    // chunks of >= 128; 64x64 tiles when the output allows (twice the
    // operand reuse of 32x32)
    const bool big = M >= 64 && N >= 64;
    const int tiles = big ? ceil_div(M, 64) * ceil_div(N, 64) : g.tiles;
    int S = K / 128;
    const int want = ceil_div(kFill, tiles);
    if (S > want) S = want;
    if (S >= 2) {
      g.big = big;
      g.tiles = tiles;
      const int chunk = ceil_div(K, S);
      S = ceil_div(K, chunk);
      double* P = temp({S, M, N});
      for (int j = 0; j < S; ++j) {
        const int k0 = j * chunk, kj = K - k0 < chunk ? K - k0 : chunk;
        GemmProb h = g;
        h.K = kj;
        h.A = a.p + (long long)k0 * a.k;
        h.B = B + (long long)k0 * bk;
        h.C = P + (long long)j * M * N;
        h.cd = 1 << 30;
        h.chi = 0;
        h.clo = N;
        h.cj = 1;
        h.alpha = 1.0;
        h.beta = 0.0;
        items_.push_back({2 * stage, h});
      }
      GemmProb r = g;
      r.kind = 1;
      r.A = P;
      r.batch = S;
      r.tiles = (int)(((long long)M * N + kReduceTile - 1) / kReduceTile);
      items_.push_back({2 * stage + 1, r});
      return;
    }
  }
  items_.push_back({2 * stage, g});
}

void GemmBatch::scale_last(const double* rs, const double* cs) {
  // the last item is the problem itself or, after a split-K, its reduction
  T2S2_REQUIRE(!items_.empty() && items_.back().g.beta == 0.0 &&
                   (items_.back().g.kind == 1 ||
                    (items_.back().g.batch == 1 && items_.back().g.ad == (1 << 30))) &&
                   items_.back().g.cd == (1 << 30),
               kErrShape, "GemmBatch::scale_last: plain beta = 0 problem expected");
  items_.back().g.rs = rs;
  items_.back().g.cs = cs;
}

int gemm_program_smem(bool wide) { return wide ? kGemmSmemWide : kGemmSmem; }

bool GemmBatch::build_program(GemmProgram& prog, bool& wide, int& max_tiles, double& flops) {
  if (items_.empty() || (int)items_.size() > kProgMaxProb) return false;
  std::stable_sort(items_.begin(), items_.end(),
                   [](const Item& x, const Item& y) { return x.stage < y.stage; });
  prog = GemmProgram{};
  prog.guard = guard_;
  int last_stage = -1, stage_tiles = 0;
  max_tiles = 0;
  wide = false;
  for (const Item& it : items_) {
    if (it.stage != last_stage) {
      if (prog.nstage == kProgMaxStage) return false;
      prog.stage_first[prog.nstage++] = prog.nprob;
      last_stage = it.stage;
      stage_tiles = 0;
    }
    prog.p[prog.nprob++] = it.g;
    stage_tiles += it.g.tiles;
    max_tiles = stage_tiles > max_tiles ? stage_tiles : max_tiles;
    wide = wide || (it.g.kind == 0 && it.g.big == 2);
  }
  prog.stage_first[prog.nstage] = prog.nprob;
  flops = flops_;
  return true;
}

void GemmBatch::run() {
  if (items_.empty()) return;
  std::stable_sort(items_.begin(), items_.end(),
                   [](const Item& x, const Item& y) { return x.stage < y.stage; });
  // split into programs of at most kProgMaxProb problems / kProgMaxStage stages
  size_t i = 0;
  while (i < items_.size()) {
    GemmProgram prog{};
    prog.guard = guard_;
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
    const int nsm = num_sms();
    bool wide = false;
    for (int q = 0; q < prog.nprob; ++q) wide = wide || (prog.p[q].kind == 0 && prog.p[q].big == 2);
    const int smem = wide ? kGemmSmemWide : kGemmSmem;
    const void* kern = wide ? (const void*)gemm_program_kernel<true>
                            : (const void*)gemm_program_kernel<false>;
    max_dynamic_smem(kern, smem);
    const int occ = occupancy(kern, 256, smem);
    int grid = max_tiles < nsm * occ ? max_tiles : nsm * occ;
    if (sm_budget() > 0 && grid > sm_budget()) grid = sm_budget();
    if (grid < 1) grid = 1;
    {
      LaunchScope ls("gemm", flops_ * prog.nprob / (double)items_.size(), 0.0);
      if (prog.nstage == 1) {
        if (wide)
          gemm_program_kernel<true><<<grid, 256, smem, stream()>>>(prog);
        else
          gemm_program_kernel<false><<<grid, 256, smem, stream()>>>(prog);
      } else {
        void* params[] = {&prog};
        T2S2_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(256), params, smem,
                                              stream()));
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
  if (!n) return;
  LaunchScope ls("copy", 0, 16.0 * n);  // a copy-engine node on the stream, counted like a launch
  T2S2_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
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

void copy_scaled(double* dst, int ldd, const double* src, int lds, int rows, int cols,
                 const double* rs, const double* cs) {
  long long n = (long long)rows * cols;
  if (n <= 0) return;
  {
    LaunchScope ls("vector", (double)n, 16.0 * n);
    copy_scaled_kernel<<<grid_for(n), 256, 0, stream()>>>(dst, ldd, src, lds, rows, cols, rs, cs);
  }
  T2S2_CHECK_LAUNCH();
}

void copy_and_scaled(double* d1, int ldd1, const double* s1, int lds1, int r1, int c1, double* d2,
                     int ldd2, const double* s2, int lds2, int r2, int c2, const double* rs) {
  const long long n1 = (long long)r1 * c1, n2 = (long long)r2 * c2;
  if (n1 <= 0 || n2 <= 0) {
    copy2d(d1, ldd1, s1, lds1, r1, c1);
    copy_scaled(d2, ldd2, s2, lds2, r2, c2, rs, nullptr);
    return;
  }
  {
    LaunchScope ls("vector", (double)n2, 16.0 * (n1 + n2));
    copy_and_scaled_kernel<<<dim3(grid_for(n1 > n2 ? n1 : n2), 2), 256, 0, stream()>>>(
        d1, ldd1, s1, lds1, r1, c1, d2, ldd2, s2, lds2, r2, c2, rs);
  }
  T2S2_CHECK_LAUNCH();
}

void split_finish(const SplitFinish& a) {
  const long long n0 = (long long)a.rows0 * a.cols0, n1 = (long long)a.rows1 * (a.c1 + a.c2);
  long long most = n0 > n1 ? n0 : n1;
  most = a.n2 > most ? a.n2 : most;
  if (most <= 0) return;
  T2S2_REQUIRE(n0 < (1LL << 31) && n1 < (1LL << 31), kErrShape, "split_finish: block too large");
  {
    LaunchScope ls("vector", (double)n0, 16.0 * (n0 + n1) + 8.0 * a.n2);
    split_finish_kernel<<<dim3(grid_for(most), a.n2 > 0 ? 3 : 2), 256, 0, stream()>>>(a);
  }
  T2S2_CHECK_LAUNCH();
}

void copy2d_pair(double* dst, int ldd, const double* s1, int ld1, int c1, const double* s2, int ld2,
                 int c2, int rows) {
  long long n = (long long)rows * (c1 + c2);
  if (n <= 0) return;
  {
    LaunchScope ls("vector", 0, 16.0 * n);
    copy2d_pair_kernel<<<grid_for(n), 256, 0, stream()>>>(dst, ldd, s1, ld1, c1, s2, ld2, c2, rows);
  }
  T2S2_CHECK_LAUNCH();
}

static void run_segments(Segments& a, long long most) {
  if (a.k == 0) return;
  {
    LaunchScope ls("vector", 0, 8.0 * most);
    segments_kernel<<<dim3(grid_for(most), a.k), 256, 0, stream()>>>(a);
  }
  T2S2_CHECK_LAUNCH();
}

void fill_many(std::initializer_list<std::pair<double*, size_t>> arrays, double v) {
  Segments a{};
  a.v = v;
  long long most = 0;
  for (const auto& pr : arrays) {
    if (!pr.second) continue;
    if (a.k == 8) {
      run_segments(a, most);
      a.k = 0;
      most = 0;
    }
    a.dst[a.k] = pr.first;
    a.src[a.k] = nullptr;
    a.n[a.k++] = (long long)pr.second;
    most = std::max(most, (long long)pr.second);
  }
  run_segments(a, most);
}

void pack(double* dst, std::initializer_list<std::pair<const double*, size_t>> parts) {
  Segments a{};
  long long most = 0, off = 0;
  for (const auto& pr : parts) {
    if (!pr.second) continue;
    a.dst[a.k] = dst + off;
    a.src[a.k] = pr.first;
    a.n[a.k++] = (long long)pr.second;
    off += (long long)pr.second;
    most = std::max(most, (long long)pr.second);
  }
  run_segments(a, most);
}

static void ddot_launch(const double* x, const double* y, size_t n, double* out, const ReadTicket& t) {
  int g = grid_for((long long)n, 256, 296);
  double* part = allocator().alloc(g);
  {
    LaunchScope ls("reduce", 2.0*n, 16.0*n);
    dot_partial_kernel<<<g, 256, 0, stream()>>>(x, y, (long long)n, part);
  }
  {
    LaunchScope ls("reduce", 0, 0);
    sum_final_kernel<<<1, 256, 0, stream()>>>(part, g, out, t);
  }
  T2S2_CHECK_LAUNCH();
  allocator().release(part);
}

void ddot_dev(const double* x, const double* y, size_t n, double* out) {
  ddot_launch(x, y, n, out, ReadTicket{});
}

double scalar_to_host(const double* d) {
  double h = 0.0;
  host_read(&h, d, sizeof(double));
  return h;
}

double ddot(const double* x, const double* y, size_t n) {
  // the final sum publishes itself: no separate read launch
  double* o = allocator().alloc(1);
  const ReadTicket t = read_open(sizeof(double));
  ddot_launch(x, y, n, o, t);
  double h = 0.0;
  read_close(&h, sizeof(double), t);
  allocator().release(o);
  return h;
}

double dnrm2(const double* x, size_t n) { return std::sqrt(ddot(x, x, n)); }

void to_host(double* h, const double* d, size_t n) { host_read(h, d, n * sizeof(double)); }

void to_device(double* d, const double* h, size_t n) {
  if (n) T2S2_CUDA(cudaMemcpyAsync(d, h, n * sizeof(double), cudaMemcpyHostToDevice, stream()));
}

std::vector<DTensor> clone_all(const std::vector<DTensor>& v) {
  std::vector<DTensor> out;
  out.reserve(v.size());
  Segments a{};
  long long most = 0;
  for (const DTensor& t : v) {
    out.emplace_back(t.shape);
    if (!t.size()) continue;
    if (a.k == 8) {
      run_segments(a, most);
      a.k = 0;
      most = 0;
    }
    a.dst[a.k] = out.back().p;
    a.src[a.k] = t.p;
    a.n[a.k] = (long long)t.size();
    most = a.n[a.k] > most ? a.n[a.k] : most;
    a.k++;
  }
  run_segments(a, most);
  return out;
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
