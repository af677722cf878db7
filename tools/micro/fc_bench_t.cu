#include <cstdio>
#include <cuda_runtime.h>
constexpr int kThreads = 512;
constexpr int kMaxPanel = 32;
__device__ __forceinline__ void amax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

constexpr int SUB = 8;

template <int RPT>
__device__ __forceinline__ void factor_columns(int rows, int w, double* sm, int* s_piv, long long* g_t) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = kThreads / 32;
  __shared__ unsigned rh[2][nw], rl[2][nw];
  __shared__ int ri[2][nw];
  __shared__ double pub[2][nw][SUB];  // each warp's candidate pivot row (sub-panel part)
  __shared__ double pinv[2][nw];      // and the reciprocal of its pivot entry
  bool live[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) live[k] = tid + k * kThreads < rows;
  for (int j0 = 0; j0 < w; j0 += SUB) {
    const int nsub = w - j0 < SUB ? w - j0 : SUB;
    double a[RPT][SUB];
#pragma unroll
    for (int k = 0; k < RPT; ++k)
#pragma unroll
      for (int t = 0; t < SUB; ++t)
        a[k][t] = (tid + k * kThreads < rows && t < nsub) ? sm[(j0 + t) * rows + tid + k * kThreads]
                                                         : 0.0;
#pragma unroll
    for (int t = 0; t < SUB; ++t) {
      if (t >= nsub) break;
      const int j = j0 + t;
      const int buf = j & 1;
      long long c0 = clock64();
      // local candidate: largest |a| among live own rows (first row on ties)
      unsigned long long kb = 0ull;
      int bi = 0x7fffffff, bk = 0;
#pragma unroll
      for (int k = 0; k < RPT; ++k)
        if (live[k]) {
          const unsigned long long b = __double_as_longlong(fabs(a[k][t]));
          if (b > kb || bi == 0x7fffffff) {
            kb = b;
            bi = tid + k * kThreads;
            bk = k;
          }
        }
      const unsigned hi = bi == 0x7fffffff ? 0u : (unsigned)(kb >> 32);
      const unsigned lo = bi == 0x7fffffff ? 0u : (unsigned)kb;
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      const int mi = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bi : 0x7fffffff);
      if (bi == mi && mi != 0x7fffffff) {
        // the warp winner publishes its row's sub-panel values (cols > t)
        // and the reciprocal of its candidate pivot (slot t)
#pragma unroll
        for (int q = 0; q < SUB; ++q) {
          double v = 0.0;
#pragma unroll
          for (int k = 0; k < RPT; ++k)
            if (k == bk) v = a[k][q];
          if (q > t) pub[buf][warp][q] = v;
          if (q == t) {
            pub[buf][warp][q] = v;
            pinv[buf][warp] = v != 0.0 ? __drcp_rn(v) : 1.0;
          }
        }
      }
      long long c1 = clock64(); g_t[0] += c1 - c0;
      if (lane == 0) {
        rh[buf][warp] = mh;
        rl[buf][warp] = ml;
        ri[buf][warp] = mi;
      }
      long long c2a = clock64();
      __syncthreads();
      const unsigned h2 = lane < nw ? rh[buf][lane] : 0u;
      const unsigned l2 = lane < nw ? rl[buf][lane] : 0u;
      const int i2 = lane < nw ? ri[buf][lane] : 0x7fffffff;
      const unsigned gh = __reduce_max_sync(0xffffffffu, h2);
      const unsigned gl = __reduce_max_sync(0xffffffffu, h2 == gh ? l2 : 0u);
      const int p = __reduce_min_sync(0xffffffffu, (h2 == gh && l2 == gl) ? i2 : 0x7fffffff);
      const int pw = __ffs(__ballot_sync(0xffffffffu, lane < nw && i2 == p)) - 1;  // winner warp
      long long c3 = clock64(); g_t[1] += c3 - c2a;
      double prow[SUB];
#pragma unroll
      for (int q = 0; q < SUB; ++q) prow[q] = q >= t ? pub[buf][pw][q] : 0.0;
      if (tid == 0) s_piv[j] = p;
      const double inv = pinv[buf][pw];
      long long c4 = clock64(); g_t[2] += c4 - c3;
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        if (tid + k * kThreads == p) live[k] = false;
        if (live[k]) {
          const double l = a[k][t] * inv;
          a[k][t] = l;
#pragma unroll
          for (int q = 0; q < SUB; ++q)
            if (q > t) a[k][q] = fma(-l, prow[q], a[k][q]);
        }
      }
      g_t[3] += clock64() - c4;
    }
    // sub-panel back to shared memory (pivot rows keep their U entries,
    // the others their multipliers)
#pragma unroll
    for (int k = 0; k < RPT; ++k)
#pragma unroll
      for (int t = 0; t < SUB; ++t)
        if (tid + k * kThreads < rows && t < nsub) sm[(j0 + t) * rows + tid + k * kThreads] = a[k][t];
    const int je = j0 + nsub;
    if (je < w) {
      __syncthreads();
      // U entries of the sub-panel's pivot rows right of it (one thread per
      // column): u_t = a[p_t][c] - sum_{q<t} l[p_t][q] u_q
      for (int c = je + tid; c < w; c += kThreads) {
        double u[SUB];
#pragma unroll
        for (int t = 0; t < SUB; ++t) {
          u[t] = 0.0;
          if (t < nsub) {
            const int pt = s_piv[j0 + t];
            double x = sm[c * rows + pt];
#pragma unroll
            for (int q = 0; q < SUB; ++q)
              if (q < t) x = fma(-sm[(j0 + q) * rows + pt], u[q], x);
            u[t] = x;
            sm[c * rows + pt] = x;
          }
        }
      }
      __syncthreads();
      // rank-nsub update of the live rows, columns je..w-1
      for (int c = je; c < w; ++c) {
        double ut[SUB];
#pragma unroll
        for (int t = 0; t < SUB; ++t) ut[t] = t < nsub ? sm[c * rows + s_piv[j0 + t]] : 0.0;
#pragma unroll
        for (int k = 0; k < RPT; ++k)
          if (live[k]) {
            double x = sm[c * rows + tid + k * kThreads];
#pragma unroll
            for (int t = 0; t < SUB; ++t) x = fma(-a[k][t], ut[t], x);
            sm[c * rows + tid + k * kThreads] = x;
          }
      }
      __syncthreads();
    }
  }
}

template <int RPT>
__global__ void __launch_bounds__(kThreads, 1) fc_kernel(double* A, int rows, int w, long long* cyc) {
  extern __shared__ double sm[];
  __shared__ int s_piv[kMaxPanel];
  for (int e = threadIdx.x; e < rows * w; e += blockDim.x) sm[e] = A[e];
  __syncthreads();
  long long t0 = clock64();
  long long gt[4] = {0,0,0,0};
  factor_columns<RPT>(rows, w, sm, s_piv, gt);
  __syncthreads();
  long long t1 = clock64();
  for (int e = threadIdx.x; e < rows * w; e += blockDim.x) A[e] = sm[e];
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; for (int i = 0; i < 4; ++i) cyc[1 + i] = gt[i]; }
}
template <int RPT> void run(int rows, int w, double* A, long long* c, double* hA) {
  cudaFuncSetAttribute(fc_kernel<RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  long long h[5] = {0};
  for (int it = 0; it < 2; ++it) {
    cudaMemcpy(A, hA, (size_t)rows * w * 8, cudaMemcpyHostToDevice);
    fc_kernel<RPT><<<1, kThreads, (size_t)rows * w * 8>>>(A, rows, w, c);
    cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  }
  printf("rows %4d w %2d RPT %d: %7.0f cyc/col | local+redux %5.0f barrier+redux2 %5.0f prow %4.0f update %4.0f (%s)\n", rows, w, RPT, (double)h[0] / w,
         (double)h[1]/w, (double)h[2]/w, (double)h[3]/w, (double)h[4]/w, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  double* A; long long* c; cudaMalloc(&A, 2600 * 32 * 8); cudaMalloc(&c, 64);
  double* hA = new double[2600 * 32];
  for (int i = 0; i < 2600 * 32; ++i) hA[i] = (double)((i * 7919) % 1013) / 1013.0 - 0.5;
  run<1>(66, 32, A, c, hA);
  run<1>(264, 32, A, c, hA);
  run<2>(792, 31, A, c, hA);
  run<3>(1386, 17, A, c, hA);
  run<4>(1584, 15, A, c, hA);
  run<4>(1584, 8, A, c, hA);
  return 0;
}
