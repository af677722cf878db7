// Microbenchmark: per-column cost of in-smem partial-pivoting panel
// factorisation in one CTA (development tool, not part of the engine).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void amax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

template <int RPT>
__global__ void panel(double* A, int rows, int w, long long* cyc, int mode) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  __shared__ double rv[2][32];
  __shared__ int ri[2][32];
  for (int e = tid; e < rows * w; e += blockDim.x) sm[e] = A[e];
  __syncthreads();
  unsigned live = 0;
  for (int k = 0; k < RPT; ++k) if (tid + k * (int)blockDim.x < rows) live |= 1u << k;
  long long t0 = clock64(), targ = 0, tupd = 0;
  for (int j = 0; j < w; ++j) {
    long long a0 = clock64();
    const int oj = j * rows;
    double best = -1.0; int bi = rows;
#pragma unroll
    for (int k = 0; k < RPT; ++k)
      if (live & (1u << k)) { const int r = tid + k * blockDim.x; amax_merge(best, bi, fabs(sm[oj + r]), r); }
    if (mode & 1) {
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        amax_merge(best, bi, v2, i2);
      }
    }
    if (lane == 0) { rv[j & 1][warp] = best; ri[j & 1][warp] = bi; }
    __syncthreads();
    best = lane < nw ? rv[j & 1][lane] : -1.0;
    bi = lane < nw ? ri[j & 1][lane] : rows;
    if (mode & 1) {
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        amax_merge(best, bi, v2, i2);
      }
    }
    long long a1 = clock64();
    targ += a1 - a0;
    const int p = bi < rows ? bi : 0;
    const double pv = sm[oj + p];
    if ((p - tid) % (int)blockDim.x == 0 && p >= tid) live &= ~(1u << ((p - tid) / blockDim.x));
    const double inv = pv != 0.0 ? 1.0 / pv : 1.0;
    double lk[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      lk[k] = 0.0;
      if (live & (1u << k)) { const int r = tid + k * blockDim.x; lk[k] = sm[oj + r] * inv; sm[oj + r] = lk[k]; }
    }
    if (mode & 2) {
      for (int c = j + 1; c < w; c += 4) {
        const int nb = w - c < 4 ? w - c : 4;
        double u[4], v[RPT][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = q < nb ? sm[(c + q) * rows + p] : 0.0;
#pragma unroll
        for (int k = 0; k < RPT; ++k)
#pragma unroll
          for (int q = 0; q < 4; ++q) v[k][q] = ((live >> k) & 1u) && q < nb ? sm[(c + q) * rows + tid + k * blockDim.x] : 0.0;
#pragma unroll
        for (int k = 0; k < RPT; ++k)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (((live >> k) & 1u) && q < nb) sm[(c + q) * rows + tid + k * blockDim.x] = fma(-lk[k], u[q], v[k][q]);
      }
    }
    tupd += clock64() - a1;
  }
  long long t1 = clock64();
  __syncthreads();
  for (int e = tid; e < rows * w; e += blockDim.x) A[e] = sm[e];
  if (tid == 0) { cyc[0] = t1 - t0; cyc[1] = targ; cyc[2] = tupd; }
}

int main() {
  int rows_list[] = {66, 792, 1600};
  double* A; long long* cyc; long long h[3];
  cudaMalloc(&A, 2000 * 32 * 8); cudaMalloc(&cyc, 64);
  cudaFuncSetAttribute(panel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  for (int rows : rows_list) {
    int w = 200 * 1024 / (8 * rows); if (w > 32) w = 32;
    double* hA = new double[rows * w];
    for (int i = 0; i < rows * w; ++i) hA[i] = (double)((i * 7919) % 1000) / 1000.0 - 0.5;
    for (int threads : {128, 256, 512}) for (int mode : {0, 1, 2, 3}) {
      if (rows > 5 * threads) continue;
      cudaMemcpy(A, hA, rows * w * 8, cudaMemcpyHostToDevice);
      panel<5><<<1, threads, rows * w * 8>>>(A, rows, w, cyc, mode);
      cudaMemcpy(A, hA, rows * w * 8, cudaMemcpyHostToDevice);
      panel<5><<<1, threads, rows * w * 8>>>(A, rows, w, cyc, mode);
      cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
      printf("rows %4d w %2d threads %3d mode %d (shfl=%d upd=%d): %6.0f cyc/col (argmax %5.0f upd %5.0f)  err=%s\n", rows, w, threads, mode, mode & 1, (mode >> 1) & 1,
             (double)h[0] / w, (double)h[1] / w, (double)h[2] / w, cudaGetErrorString(cudaGetLastError()));
    }
    delete[] hA;
  }
  return 0;
}
