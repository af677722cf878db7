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

// One core of a TT sum written in one pass: out (r0o, mid, r1o) holds
// fa * a at offsets (0, 0), fb * b at offsets (ob0, ob1), zeros elsewhere
// (the blocks are disjoint: block diagonal, or side by side in the first
// and last cores).
__global__ void sum_core_kernel(double* out, int r0o, int mid, int r1o, const double* a, int r0a,
                                int r1a, double fa, const double* b, int r0b, int r1b, double fb,
                                int ob0, int ob1) {
  const long long n = (long long)r0o * mid * r1o;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e % r1o);
    const long long t = e / r1o;
    const int m = (int)(t % mid), i = (int)(t / mid);
    double v = 0.0;
    if (i < r0a && j < r1a) {
      v = fa * a[((long long)i * mid + m) * r1a + j];
    } else {
      const int ib = i - ob0, jb = j - ob1;
      if (ib >= 0 && jb >= 0 && ib < r0b && jb < r1b) v = fb * b[((long long)ib * mid + m) * r1b + jb];
    }
    out[e] = v;
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

void right_orthonormalize(std::vector<DTensor>& cores) {
  const int d = (int)cores.size();
  for (int l = d - 1; l > 0; --l) {
    DTensor& c = cores[l];
    const int r0 = c.dim(0), r1 = c.dim(-1);
    const long long mid = mid_size(c);
    const int rows = (int)(mid * r1);
    // the row-major r0 x rows unfolding is the column-major rows x r0 matrix
    // whose QR we need; Q comes back column-major = the new core row-major
    DTensor Q, R;
    qr_thin(rows, r0, c.p, Q, R, true);  // Q rows x k (column-major), R k x r0
    const int k = rows < r0 ? rows : r0;
    DTensor nc(with_bonds(c, k, r1));
    dcopy(nc.p, Q.p, (size_t)rows * k);
    DTensor& p = cores[l - 1];
    const int pr = (int)((long long)p.size() / r0);
    DTensor np(with_bonds(p, p.dim(0), k));
    gemm(false, true, pr, k, r0, 1.0, p.p, r0, R.p, r0, 0.0, np.p, k);
    cores[l] = std::move(nc);
    cores[l - 1] = std::move(np);
  }
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
    DTensor Y({r0 * mid, k});
    if (l == t.d() - 1)
      dcopy(Y.p, c.p, c.size());
    else
      gemm(false, true, r0 * mid, k, r1, 1.0, c.p, r1, Rp.p, r1, 0.0, Y.p, k);
    if (l == 0) return dnrm2(Y.p, Y.size());
    qr_r(mid * k, r0, Y.p, Rp, true);  // Y row-major r0 x (mid k) = column-major (mid k) x r0
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
  std::vector<DTensor> w;
  for (auto& c : t.cores) w.push_back(c.clone());
  right_orthonormalize(w);
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
    svd_thin(m, r1, c.p, U, s, Vt);
    const int kk = s.dim(0);
    std::vector<double> hs(kk);
    to_host(hs.data(), s.p, kk);
    long long cap = cap_all < in_ranks[l + 1] ? cap_all : in_ranks[l + 1];
    int r = tail_keep(hs, delta);
    if (r > cap) r = (int)cap;
    DTensor nc(with_bonds(c, r0, r));
    copy2d(nc.p, r, U.p, kk, m, r);
    DTensor carry({r, r1});
    copy_scaled(carry.p, r1, Vt.p, r1, r, r1, s.p, nullptr);
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
  for (int l = 0; l < d; ++l) {
    const DTensor& ca = a.cores[l];
    const DTensor& cb = b.cores[l];
    const int mid = (int)mid_size(ca);
    const double fa = l == 0 ? sa : 1.0, fb = l == 0 ? sb : 1.0;
    if (d == 1) {
      DTensor o(ca.shape);
      dcopy(o.p, cb.p, o.size());
      daxpby(fa, ca.p, fb, o.p, o.size());
      out.cores.push_back(std::move(o));
      continue;
    }
    const int r0 = l == 0 ? 1 : ca.dim(0) + cb.dim(0);
    const int r1 = l == d - 1 ? 1 : ca.dim(-1) + cb.dim(-1);
    DTensor o(with_bonds(ca, r0, r1));
    const int ob0 = l == 0 ? 0 : ca.dim(0), ob1 = l == d - 1 ? 0 : ca.dim(-1);
    const long long no = (long long)o.size();
    {
      LaunchScope ls("vector", 0, 8.0 * (no + (long long)ca.size() + (long long)cb.size()));
      sum_core_kernel<<<grid_of(no), 256, 0, stream()>>>(o.p, r0, mid, r1, ca.p, ca.dim(0),
                                                         ca.dim(-1), fa, cb.p, cb.dim(0),
                                                         cb.dim(-1), fb, ob0, ob1);
    }
    T2S2_CHECK_LAUNCH();
    out.cores.push_back(std::move(o));
  }
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
  Train out;
  out.rows = op.rows;
  for (int l = 0; l < op.d(); ++l) {
    const DTensor& co = op.cores[l];  // (a, m, n, b)
    const DTensor& cv = v.cores[l];   // (c, n, e)
    DTensor t = tensordot(co, {2}, cv, {1});  // (a, m, b, c, e)
    DTensor p = permute(t, {0, 3, 1, 2, 4});   // (a, c, m, b, e)
    p.view({co.dim(0) * cv.dim(0), co.dim(1), co.dim(3) * cv.dim(2)});
    out.cores.push_back(std::move(p));
  }
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
