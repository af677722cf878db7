// Device tensor-train operations (reference: pkg/src/ttss/tensor_train.py).
#include <cmath>

#include "blas.h"
#include "linalg.h"
#include "tt.h"

namespace t2s2 {
namespace {

__global__ void scale_rows_kernel(double* X, int rows, int cols, int ld, const double* s) {
  long long n = (long long)rows * cols;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (int)n;
       e += gridDim.x * blockDim.x) {
    int r = (int)(e / cols), c = (int)(e % cols);
    X[(long long)r * ld + c] *= s[r];
  }
}

__global__ void scale_cols_kernel(double* X, int rows, int cols, int ld, const double* s) {
  long long n = (long long)rows * cols;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (int)n;
       e += gridDim.x * blockDim.x) {
    int r = (int)(e / cols), c = (int)(e % cols);
    X[(long long)r * ld + c] *= s[c];
  }
}

// The cores of a TT sum written in one pass and ONE launch (blockIdx.y = the
// core): out (r0o, mid, r1o) holds fa * a at offsets (0, 0), fb * b at offsets
// (ob0, ob1), zeros elsewhere (the blocks are disjoint: block diagonal, or
// side by side in the first and last cores).
constexpr int kSumCores = 8;
struct SumCore {
  double* out;
  const double* a;
  const double* b;
  double fa, fb;
  int r0o, mid, r1o, r0a, r1a, r0b, r1b, ob0, ob1;
};
struct SumCores {
  SumCore c[kSumCores];
};
__global__ void sum_cores_kernel(const __grid_constant__ SumCores args) {
  const SumCore& k = args.c[blockIdx.y];
  const int n = k.r0o * k.mid * k.r1o;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int j = e % k.r1o;
    const int t = e / k.r1o;
    const int m = t % k.mid, i = t / k.mid;
    double v = 0.0;
    if (i < k.r0a && j < k.r1a) {
      v = k.fa * k.a[((long long)i * k.mid + m) * k.r1a + j];
    } else {
      const int ib = i - k.ob0, jb = j - k.ob1;
      if (ib >= 0 && jb >= 0 && ib < k.r0b && jb < k.r1b)
        v = k.fb * k.b[((long long)ib * k.mid + m) * k.r1b + jb];
    }
    k.out[e] = v;
  }
}

int grid_of(long long n) {
  long long g = (n + 255) / 256;
  if (g < 1) g = 1;
  if (g > 1184) g = 1184;
  return (int)g;
}

// Shape of a core with its bonds replaced.
std::vector<int> with_bonds(const DTensor& c, int r0, int r1) {
  std::vector<int> s = c.shape;
  s.front() = r0;
  s.back() = r1;
  return s;
}

long long mid_size(const DTensor& c) { return (long long)c.size() / ((long long)c.dim(0) * c.dim(-1)); }

}  // namespace

void scale_rows(double* X, int rows, int cols, int ld, const double* s) {
  if ((long long)rows * cols <= 0) return;
  {
    LaunchScope ls("vector", (double)rows*cols, 16.0*rows*cols);
    scale_rows_kernel<<<grid_of((long long)rows * cols), 256, 0, stream()>>>(X, rows, cols, ld, s);
  }
  T2S2_CHECK_LAUNCH();
}

void scale_cols(double* X, int rows, int cols, int ld, const double* s) {
  if ((long long)rows * cols <= 0) return;
  {
    LaunchScope ls("vector", (double)rows*cols, 16.0*rows*cols);
    scale_cols_kernel<<<grid_of((long long)rows * cols), 256, 0, stream()>>>(X, rows, cols, ld, s);
  }
  T2S2_CHECK_LAUNCH();
}

int tail_keep(const std::vector<double>& s, double delta) {
  const int n = (int)s.size();
  if (n == 0) return 1;
  // tails[k] = ||s[k:]||, accumulated from the back like the reference
  std::vector<double> tails(n);
  double acc = 0.0;
  for (int k = n - 1; k >= 0; --k) {
    acc += s[k] * s[k];
    tails[k] = std::sqrt(acc);
  }
  int r = n;
  for (int k = 0; k < n; ++k)
    if (tails[k] <= delta) {
      r = k;
      break;
    }
  return r < 1 ? 1 : r;
}

// Right-to-left QR sweep: reads the cores of `in` (core l - 1 after it has
// absorbed R_l), never writes them; returns the new cores.
static std::vector<DTensor> right_orthonormalized(const std::vector<DTensor>& in) {
  const int d = (int)in.size();
  std::vector<DTensor> out(d);
  DTensor absorbed;  // core l with R_{l+1} multiplied in
  for (int l = d - 1; l > 0; --l) {
    const DTensor& c = l == d - 1 ? in[l] : absorbed;
    const int r0 = c.dim(0), r1 = c.dim(-1);
    const long long mid = mid_size(c);
    const int rows = (int)(mid * r1);
    // the row-major r0 x rows unfolding is the column-major rows x r0 matrix
    // whose QR we need; Q comes back column-major = the new core row-major
    DTensor Q, R;
    const int k = rows < r0 ? rows : r0;
    const DTensor& p = in[l - 1];
    const int pr = (int)((long long)p.size() / r0);
    DTensor np(with_bonds(p, p.dim(0), k));
    // Q rows x k (column-major), R k x r0; the QR kernel multiplies R into
    // the neighbouring core itself when it is the one-CTA warp kernel
    if (!qr_thin_absorb(rows, r0, c.p, Q, R, true, p.p, pr, np.p))
      gemm(false, true, pr, k, r0, 1.0, p.p, r0, R.p, r0, 0.0, np.p, k);
    DTensor nc = std::move(Q);
    nc.view(with_bonds(c, k, r1));
    out[l] = std::move(nc);
    absorbed = std::move(np);
  }
  out[0] = d == 1 ? in[0].clone() : std::move(absorbed);
  return out;
}

void right_orthonormalize(std::vector<DTensor>& cores) {
  if (cores.size() > 1) cores = right_orthonormalized(cores);
}

double tt_norm(const Train& t) {
  // ||t|| through the right-orthonormalisation R chain (tensor_train.py:
  // 307-324) without forming the orthonormal cores: only the triangular
  // factors travel to the left.
  if (t.d() == 1) return dnrm2(t.cores[0].p, t.cores[0].size());
  DTensor Rp;  // k x r1 factor of the part to the right of the current bond
  for (int l = t.d() - 1; l >= 0; --l) {
    const DTensor& c = t.cores[l];
    const int r0 = c.dim(0), r1 = c.dim(-1);
    const int mid = (int)(c.size() / ((size_t)r0 * r1));
    const int k = l == t.d() - 1 ? r1 : Rp.dim(0);
    DTensor Y;
    const double* Yp = c.p;  // the last core is its own Y (r1 = k = 1 column block), read only
    if (l < t.d() - 1) {
      Y = DTensor({r0 * mid, k});
      gemm(false, true, r0 * mid, k, r1, 1.0, c.p, r1, Rp.p, r1, 0.0, Y.p, k);
      Yp = Y.p;
    }
    if (l == 0) return dnrm2(Yp, (size_t)r0 * mid * k);
    qr_r(mid * k, r0, Yp, Rp, true);  // Y row-major r0 x (mid k) = column-major (mid k) x r0
  }
  return 0.0;
}

Train tt_round(const Train& t, double tol, int max_rank) {
  T2S2_REQUIRE(tol >= 0, kErrValue, "tolerance must be >= 0");
  Train out;
  out.rows = t.rows;
  out.cols = t.cols;
  const int d = t.d();
  if (d == 1) return t.clone();
  const long long cap_all = max_rank > 0 ? max_rank : 1000000000LL;
  std::vector<int> in_ranks = t.ranks();
  std::vector<DTensor> w = right_orthonormalized(t.cores);
  const double nrm = dnrm2(w[0].p, w[0].size());
  if (nrm == 0.0) {
    for (int l = 0; l < d; ++l) {
      DTensor z(with_bonds(t.cores[l], 1, 1));
      dfill(z.p, 0.0, z.size());
      out.cores.push_back(std::move(z));
    }
    return out;
  }
  const double delta = tol * nrm / std::sqrt((double)(d - 1));
  for (int l = 0; l < d - 1; ++l) {
    DTensor& c = w[l];
    const int r0 = c.dim(0), r1 = c.dim(-1);
    const int m = (int)((long long)c.size() / r1);
    DTensor U, s, Vt;
    const int kk = m < r1 ? m : r1;
    std::vector<double> hs(kk);
    {
      // the SVD kernel publishes the singular values itself
      const ReadTicket tk = read_open(kk * sizeof(double));
      svd_thin(m, r1, c.p, U, s, Vt, &tk);
      read_close(hs.data(), kk * sizeof(double), tk);
    }
    long long cap = cap_all < in_ranks[l + 1] ? cap_all : in_ranks[l + 1];
    int r = tail_keep(hs, delta);
    if (r > cap) r = (int)cap;
    DTensor nc(with_bonds(c, r0, r));
    DTensor carry({r, r1});
    copy_and_scaled(nc.p, r, U.p, kk, m, r, carry.p, r1, Vt.p, r1, r, r1, s.p);
    DTensor& nx = w[l + 1];
    const int rest = (int)((long long)nx.size() / r1);
    DTensor nn(with_bonds(nx, r, nx.dim(-1)));
    gemm(false, false, r, rest, r1, 1.0, carry.p, r1, nx.p, rest, 0.0, nn.p, rest);
    w[l] = std::move(nc);
    w[l + 1] = std::move(nn);
  }
  out.cores = std::move(w);
  return out;
}

Train tt_add(const Train& a, const Train& b, double sa, double sb) {
  T2S2_REQUIRE(a.d() == b.d() && a.rows == b.rows && a.cols == b.cols, kErrShape,
               "tt_add: mode mismatch");
  const int d = a.d();
  Train out;
  out.rows = a.rows;
  out.cols = a.cols;
  if (d == 1) {
    const DTensor& ca = a.cores[0];
    DTensor o(ca.shape);
    dcopy(o.p, b.cores[0].p, o.size());
    daxpby(sa, ca.p, sb, o.p, o.size());
    out.cores.push_back(std::move(o));
    return out;
  }
  SumCores args{};
  int nb = 0;
  long long largest = 0, bytes = 0;
  auto flush = [&]() {
    if (nb == 0) return;
    {
      LaunchScope ls("vector", 0, (double)bytes);
      sum_cores_kernel<<<dim3(grid_of(largest), nb), 256, 0, stream()>>>(args);
    }
    T2S2_CHECK_LAUNCH();
    nb = 0;
    largest = bytes = 0;
  };
  for (int l = 0; l < d; ++l) {
    const DTensor& ca = a.cores[l];
    const DTensor& cb = b.cores[l];
    const int r0 = l == 0 ? 1 : ca.dim(0) + cb.dim(0);
    const int r1 = l == d - 1 ? 1 : ca.dim(-1) + cb.dim(-1);
    DTensor o(with_bonds(ca, r0, r1));
    const long long no = (long long)o.size();
    T2S2_REQUIRE(no < (1LL << 31), kErrShape, "tt_add: core too large");
    args.c[nb++] = SumCore{o.p, ca.p, cb.p, l == 0 ? sa : 1.0, l == 0 ? sb : 1.0, r0, (int)mid_size(ca),
                           r1, ca.dim(0), ca.dim(-1), cb.dim(0), cb.dim(-1),
                           l == 0 ? 0 : ca.dim(0), l == d - 1 ? 0 : ca.dim(-1)};
    largest = no > largest ? no : largest;
    bytes += 8 * (no + (long long)ca.size() + (long long)cb.size());
    out.cores.push_back(std::move(o));
    if (nb == kSumCores) flush();
  }
  flush();
  return out;
}

Train tt_scale(const Train& a, double s) {
  Train o = a.clone();
  dscal(o.cores[0].p, s, o.cores[0].size());
  return o;
}

Train tt_apply(const Train& op, const Train& v) {
  T2S2_REQUIRE(op.is_op() && !v.is_op() && op.cols == v.rows, kErrShape,
               "tt_apply: operator columns do not match vector modes");
  // out_l[(a,c), m, (b,e)] = sum_n op_l[a, m, n, b] v_l[c, n, e]: every core is
  // one batched GEMM (batch c, rows (a, m, b), columns e) that reads the cores
  // where they lie and writes the result core in place, all cores in ONE
  // single-stage program — one launch instead of two permutations, a GEMM and
  // a permutation per core, with the same contraction order over n.
  Train out;
  out.rows = op.rows;
  GemmBatch gb;
  for (int l = 0; l < op.d(); ++l) {
    const DTensor& co = op.cores[l];  // (a, m, n, b)
    const DTensor& cv = v.cores[l];   // (c, n, e)
    const int A = co.dim(0), M = co.dim(1), N = co.dim(2), B = co.dim(3);
    const int C = cv.dim(0), E = cv.dim(2);
    DTensor p({A * C, M, B * E});
    // A(i = (a m, b), n) at (i / B) * N B + (i % B) + n B; B(n, e) of batch c;
    // C(i = (a, m b), e) at (i / (M B)) * C M B E + (i % (M B)) * E + e, batch stride M B E
    const GemmOperand a{co.p, B, (long long)N * B, 1, B, 0};
    const GemmOperand c{p.p, M * B, (long long)C * M * B * E, E, 1, (long long)M * B * E};
    gb.add_general(0, A * M * B, E, N, a, cv.p, E, 1, (long long)N * E, c, C);
    out.cores.push_back(std::move(p));
  }
  gb.run();
  return out;
}

double tt_dot(const Train& a, const Train& b) {
  T2S2_REQUIRE(a.d() == b.d() && a.rows == b.rows, kErrShape, "tt_dot: mode mismatch");
  DTensor phi({1, 1});
  dfill(phi.p, 1.0, 1);
  for (int l = 0; l < a.d(); ++l) {
    DTensor t = tensordot(phi, {0}, a.cores[l], {0});    // (rb, n, ra1)
    phi = tensordot(t, {0, 1}, b.cores[l], {0, 1});       // (ra1, rb1)
  }
  return scalar_to_host(phi.p);
}

void tt_full(const Train& v, double* host_out, size_t cap) {
  size_t total = 1;
  for (int n : v.rows) total *= (size_t)n;
  T2S2_REQUIRE(total <= cap, kErrCapacity, "tt_full: output buffer too small");
  const DTensor& c0 = v.cores[0];
  DTensor acc({(int)(c0.size() / c0.dim(-1)), c0.dim(-1)});
  dcopy(acc.p, c0.p, c0.size());
  for (int l = 1; l < v.d(); ++l) {
    const DTensor& c = v.cores[l];
    const int r0 = c.dim(0);
    const int rest = (int)(c.size() / r0);
    const int rows = (int)(acc.size() / r0);
    DTensor nx({rows, rest});
    gemm(false, false, rows, rest, r0, 1.0, acc.p, r0, c.p, rest, 0.0, nx.p, rest);
    acc = std::move(nx);
  }
  to_host(host_out, acc.p, total);
}

double compression_ratio(const Train& v) {
  double dense = 1.0, stored = 0.0;
  for (int l = 0; l < v.d(); ++l) {
    dense *= (double)v.rows[l] * (v.is_op() ? v.cols[l] : 1);
    stored += (double)v.cores[l].size();
  }
  return stored / dense;
}

}  // namespace t2s2
