// Microbenchmark + check of the panel column loop (development tool, not
// part of the engine): packed 32-bit pivot keys (one REDUX per level), only
// the warps that own rows take part (named barrier), U rows of a register
// sub-panel solved from preloaded values.  Verifies P A = L U on the host.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int kThreads = 512;
constexpr int kMaxPanel = 32;

__device__ __forceinline__ void bar_n(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

template <int RPT, int SUB>
__device__ __forceinline__ void factor_columns2(int rows, int w, double* sm, int* s_piv, int nthr, long long* prof) {
  long long c0 = clock64(), c_steps = 0, c_sub = 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = nthr >> 5;
  const unsigned full = 0xffffffffu;
  __shared__ unsigned rk[2][16];
  __shared__ __align__(16) double pub[2][16][SUB + 2];  // candidate row, slot SUB = 1/pivot
  __shared__ double Lp[SUB][SUB];                       // multipliers of the pivot rows
  __shared__ __align__(16) double Us[kMaxPanel][SUB];   // U rows right of the sub-panel
  int row[RPT];
  bool live[RPT];
  unsigned tag[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    row[k] = tid + k * nthr;
    live[k] = row[k] < rows;
    tag[k] = 4095u - (unsigned)row[k];
  }
  for (int j0 = 0; j0 < w; j0 += SUB) {
    const int nsub = w - j0 < SUB ? w - j0 : SUB;
    double a[RPT][SUB];
    int pv[SUB];
#pragma unroll
    for (int k = 0; k < RPT; ++k)
#pragma unroll
      for (int t = 0; t < SUB; ++t) a[k][t] = (row[k] < rows && t < nsub) ? sm[(j0 + t) * rows + row[k]] : 0.0;
#pragma unroll
    for (int t = 0; t < SUB; ++t) {
      pv[t] = 0;
      if (t >= nsub) break;
      const int buf = (j0 + t) & 1;
      unsigned key = 0u;
      int bk = 0;
#pragma unroll
      for (int k = 0; k < RPT; ++k)
        if (live[k]) {
          const unsigned kk = (((unsigned)__double2hiint(fabs(a[k][t])) >> 11) << 12) | tag[k];
          if (kk > key) {
            key = kk;
            bk = k;
          }
        }
      const unsigned wk = __reduce_max_sync(full, key);
      if (key == wk && key != 0u) {
        double* dst = pub[buf][warp];
#pragma unroll
        for (int q = 0; q < SUB; ++q) {
          double v = a[0][q];
#pragma unroll
          for (int k = 1; k < RPT; ++k)
            if (k == bk) v = a[k][q];
          dst[q] = v;
          if (q == t) dst[SUB] = v != 0.0 ? __drcp_rn(v) : 1.0;
        }
      }
      if (lane == 0) rk[buf][warp] = wk;
      bar_n(nthr);
      const unsigned g = __reduce_max_sync(full, lane < nw ? rk[buf][lane] : 0u);
      const int p = 4095 - (int)(g & 4095u);
      pv[t] = p;
      const double* src = pub[buf][(p & (nthr - 1)) >> 5];
      double prow[SUB];
#pragma unroll
      for (int q = 0; q < SUB; ++q) prow[q] = q > t ? src[q] : 0.0;
      const double inv = src[SUB];
      if (tid < t) Lp[t][tid] = src[tid];
      if (tid == 0) s_piv[j0 + t] = p;
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        if (row[k] == p) live[k] = false;
        if (live[k]) {
          const double l = a[k][t] * inv;
          a[k][t] = l;
#pragma unroll
          for (int q = 0; q < SUB; ++q)
            if (q > t) a[k][q] = fma(-l, prow[q], a[k][q]);
        }
      }
    }
    {
      const long long c1 = clock64();
      c_steps += c1 - c0;
      c0 = c1;
    }
#pragma unroll
    for (int k = 0; k < RPT; ++k)
#pragma unroll
      for (int t = 0; t < SUB; ++t)
        if (row[k] < rows && t < nsub) sm[(j0 + t) * rows + row[k]] = a[k][t];
    const int je = j0 + nsub;
    if (je < w) {
      bar_n(nthr);
      // U rows of the sub-panel's pivots right of it: one thread per column
      for (int c = je + tid; c < w; c += nthr) {
        double x[SUB];
#pragma unroll
        for (int t = 0; t < SUB; ++t) x[t] = t < nsub ? sm[c * rows + pv[t]] : 0.0;
#pragma unroll
        for (int t = 1; t < SUB; ++t)
#pragma unroll
          for (int q = 0; q < t; ++q) x[t] = fma(-Lp[t][q], x[q], x[t]);
#pragma unroll
        for (int t = 0; t < SUB; ++t) {
          Us[c][t] = x[t];
          if (t < nsub) sm[c * rows + pv[t]] = x[t];
        }
      }
      bar_n(nthr);
      // rank-nsub update of the live rows, columns je..w-1
      int c = je;
      for (; c + 1 < w; c += 2) {
        double u0[SUB], u1[SUB], x0[RPT], x1[RPT];
#pragma unroll
        for (int t = 0; t < SUB; ++t) {
          u0[t] = Us[c][t];
          u1[t] = Us[c + 1][t];
        }
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          x0[k] = live[k] ? sm[c * rows + row[k]] : 0.0;
          x1[k] = live[k] ? sm[(c + 1) * rows + row[k]] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < RPT; ++k)
#pragma unroll
          for (int t = 0; t < SUB; ++t) {
            x0[k] = fma(-a[k][t], u0[t], x0[k]);
            x1[k] = fma(-a[k][t], u1[t], x1[k]);
          }
#pragma unroll
        for (int k = 0; k < RPT; ++k)
          if (live[k]) {
            sm[c * rows + row[k]] = x0[k];
            sm[(c + 1) * rows + row[k]] = x1[k];
          }
      }
      if (c < w) {
        double ut[SUB];
#pragma unroll
        for (int t = 0; t < SUB; ++t) ut[t] = Us[c][t];
#pragma unroll
        for (int k = 0; k < RPT; ++k)
          if (live[k]) {
            double x = sm[c * rows + row[k]];
#pragma unroll
            for (int t = 0; t < SUB; ++t) x = fma(-a[k][t], ut[t], x);
            sm[c * rows + row[k]] = x;
          }
      }
    }
    {
      const long long c1 = clock64();
      c_sub += c1 - c0;
      c0 = c1;
    }
  }
  if (threadIdx.x == 0) {
    prof[1] = c_steps;
    prof[2] = c_sub;
  }
}

template <int RPT, int SUB, int NT>
__global__ void __launch_bounds__(NT, 1) fc2_kernel(double* A, int* piv, int rows, int w, int nthr, int getenv_reps,
                                                          long long* cyc) {
  extern __shared__ double sm[];
  __shared__ int s_piv[kMaxPanel];
  for (int e = threadIdx.x; e < rows * w; e += blockDim.x) sm[e] = A[e];
  __syncthreads();
  long long t0 = clock64();
  const int reps = getenv_reps;
  for (int it = 0; it < reps; ++it)
    if ((int)threadIdx.x < nthr) factor_columns2<RPT, SUB>(rows, w, sm, s_piv, nthr, cyc);
  __syncthreads();
  long long t1 = clock64();
  for (int e = threadIdx.x; e < rows * w; e += blockDim.x) A[e] = sm[e];
  if ((int)threadIdx.x < w) piv[threadIdx.x] = s_piv[threadIdx.x];
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// host check: rebuild P A = L U from the in-place panel
double check(const std::vector<double>& A0, const std::vector<double>& F, const int* piv, int rows, int w) {
  std::vector<int> pos(rows, -1);
  for (int j = 0; j < w; ++j) {
    if (piv[j] < 0 || piv[j] >= rows || pos[piv[j]] >= 0) return 1e300;
    pos[piv[j]] = j;
  }
  double err = 0.0, nrm = 0.0;
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < w; ++c) {
      // row r: L entries at columns < min(pos, w), U of pivot row j at column c >= j
      const int lim = pos[r] >= 0 ? pos[r] : w;
      double s = 0.0;
      for (int q = 0; q <= c && q < lim; ++q) s += F[q * rows + r] * F[c * rows + piv[q]];
      if (pos[r] >= 0 && c >= pos[r]) s += F[c * rows + r];
      err = fmax(err, fabs(s - A0[c * rows + r]));
      nrm = fmax(nrm, fabs(A0[c * rows + r]));
    }
  return err / nrm;
}

int g_reps = 1;
template <int RPT, int SUB, int NT>
void run(int rows, int w, double* A, int* piv, long long* c, const std::vector<double>& hA) {
  int nthr = 32;
  while (nthr * RPT < rows) nthr *= 2;
  if (nthr > NT) return;
  cudaFuncSetAttribute(fc2_kernel<RPT, SUB, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  long long h = 0, hh[3];
  std::vector<double> F(rows * w);
  int hp[kMaxPanel];
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(A, hA.data(), (size_t)rows * w * 8, cudaMemcpyHostToDevice);
    fc2_kernel<RPT, SUB, NT><<<1, NT, (size_t)rows * w * 8>>>(A, piv, rows, w, nthr, g_reps, c);
    cudaMemcpy(hh, c, 24, cudaMemcpyDeviceToHost);
    h = hh[0];
  }
  cudaMemcpy(F.data(), A, (size_t)rows * w * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hp, piv, w * 4, cudaMemcpyDeviceToHost);
  std::vector<double> A0(hA.begin(), hA.begin() + rows * w);
  printf("NT %d SUB %d rows %4d w %2d RPT %d nthr %3d: %6.0f cycles/column (steps %5.0f sub %5.0f) err %.1e (%s)\n", NT, SUB, rows, w, RPT, nthr,
         (double)h / w, (double)hh[1] / w, (double)hh[2] / w, check(A0, F, hp, rows, w), cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  if (argc > 1) g_reps = atoi(argv[1]);
  double* A;
  int* piv;
  long long* c;
  cudaMalloc(&A, 2600 * 32 * 8);
  cudaMalloc(&piv, 64 * 4);
  cudaMalloc(&c, 32);
  std::vector<double> hA(2600 * 32);
  srand(1);
  for (auto& v : hA) v = (double)rand() / RAND_MAX - 0.5;
  const int rs[] = {33, 66, 132, 264, 528, 792, 1188, 1584, 1848, 2112};
  for (int rows : rs) {
    int w = (int)((200 * 1024 - 8 * rows) / (8 * rows));
    if (w > 32) w = 32;
    if (rows <= 1 * 512 && rows > (1 - 1) * 512 / 2) run<1, 8, 512>(rows, w, A, piv, c, hA);
    if (rows <= 2 * 512 && rows > (2 - 1) * 512 / 2) run<2, 8, 512>(rows, w, A, piv, c, hA);
    if (rows <= 1 * 512 && rows > (1 - 1) * 512 / 2) run<1, 4, 512>(rows, w, A, piv, c, hA);
    if (rows <= 2 * 512 && rows > (2 - 1) * 512 / 2) run<2, 4, 512>(rows, w, A, piv, c, hA);
    if (rows <= 3 * 512 && rows > (3 - 1) * 512 / 2) run<3, 4, 512>(rows, w, A, piv, c, hA);
    if (rows <= 4 * 512 && rows > (4 - 1) * 512 / 2) run<4, 4, 512>(rows, w, A, piv, c, hA);
    if (rows <= 5 * 512 && rows > (5 - 1) * 512 / 2) run<5, 4, 512>(rows, w, A, piv, c, hA);
    if (rows <= 1 * 256 && rows > (1 - 1) * 256 / 2) run<1, 8, 256>(rows, w, A, piv, c, hA);
    if (rows <= 2 * 256 && rows > (2 - 1) * 256 / 2) run<2, 8, 256>(rows, w, A, piv, c, hA);
    if (rows <= 3 * 256 && rows > (3 - 1) * 256 / 2) run<3, 8, 256>(rows, w, A, piv, c, hA);
    if (rows <= 4 * 256 && rows > (4 - 1) * 256 / 2) run<4, 8, 256>(rows, w, A, piv, c, hA);
    if (rows <= 5 * 256 && rows > (5 - 1) * 256 / 2) run<5, 8, 256>(rows, w, A, piv, c, hA);
    if (rows <= 6 * 256 && rows > (6 - 1) * 256 / 2) run<6, 8, 256>(rows, w, A, piv, c, hA);
    if (rows <= 7 * 256 && rows > (7 - 1) * 256 / 2) run<7, 8, 256>(rows, w, A, piv, c, hA);
    if (rows <= 8 * 256 && rows > (8 - 1) * 256 / 2) run<8, 8, 256>(rows, w, A, piv, c, hA);
    if (rows <= 9 * 256 && rows > (9 - 1) * 256 / 2) run<9, 8, 256>(rows, w, A, piv, c, hA);
    if (rows <= 10 * 256 && rows > (10 - 1) * 256 / 2) run<10, 8, 256>(rows, w, A, piv, c, hA);
    if (rows <= 2 * 256 && rows > (2 - 1) * 256 / 2) run<2, 4, 256>(rows, w, A, piv, c, hA);
    if (rows <= 3 * 256 && rows > (3 - 1) * 256 / 2) run<3, 4, 256>(rows, w, A, piv, c, hA);
    if (rows <= 4 * 256 && rows > (4 - 1) * 256 / 2) run<4, 4, 256>(rows, w, A, piv, c, hA);
    if (rows <= 5 * 256 && rows > (5 - 1) * 256 / 2) run<5, 4, 256>(rows, w, A, piv, c, hA);
    if (rows <= 6 * 256 && rows > (6 - 1) * 256 / 2) run<6, 4, 256>(rows, w, A, piv, c, hA);
    if (rows <= 8 * 256 && rows > (8 - 1) * 256 / 2) run<8, 4, 256>(rows, w, A, piv, c, hA);
    if (rows <= 10 * 256 && rows > (10 - 1) * 256 / 2) run<10, 4, 256>(rows, w, A, piv, c, hA);
  }
  return 0;
}
