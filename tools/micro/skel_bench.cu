// What does one "column step" skeleton cost? (development microbenchmark)
#include <cstdio>
__device__ __forceinline__ void amax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}
__global__ void skel(const double* A, int w, long long* cyc, int mode) {
  __shared__ double sm[4096];
  __shared__ double rv[2][32];
  __shared__ int ri[2][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int e = tid; e < 4096; e += blockDim.x) sm[e] = A[e];
  __syncthreads();
  double acc = 0.0;
  long long t0 = clock64();
  for (int j = 0; j < w; ++j) {
    double best = fabs(sm[(j * 67 + tid) & 4095]);
    int bi = tid;
    if (mode >= 1) {
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        amax_merge(best, bi, v2, i2);
      }
    }
    if (mode >= 2) {
      if (lane == 0) { rv[j & 1][warp] = best; ri[j & 1][warp] = bi; }
      __syncthreads();
      best = lane < nw ? rv[j & 1][lane] : -1.0;
      bi = lane < nw ? ri[j & 1][lane] : 0;
    }
    if (mode >= 3) {
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        amax_merge(best, bi, v2, i2);
      }
    }
    acc += best + bi;
  }
  long long t1 = clock64();
  if (tid == 0) { cyc[0] = t1 - t0; cyc[1] = (long long)acc; }
}
int main() {
  double* A; long long* c; long long h[2];
  cudaMalloc(&A, 4096 * 8); cudaMemset(A, 0, 4096 * 8); cudaMalloc(&c, 16);
  for (int threads : {32, 128, 512}) for (int mode = 0; mode < 4; ++mode) {
    skel<<<1, threads>>>(A, 64, c, mode); skel<<<1, threads>>>(A, 64, c, mode);
    cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("threads %3d mode %d: %6.1f cycles per column\n", threads, mode, h[0] / 64.0);
  }
}
