// Ping-pong latency: one thread publishes a value through shared memory,
// a named barrier, every thread reads it (development tool).
#include <cstdio>
template <int M>
__global__ void k(double* out, long long* cyc) {
  __shared__ double s[2][32];
  double v = threadIdx.x * 1e-3 + 1.0;
  if (threadIdx.x < 64) s[threadIdx.x >> 5][threadIdx.x & 31] = v;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int st = 0; st < 256; ++st) {
    const int par = st & 1;
    const double r = s[par][st & 31];
    v = fma(v, r, 1e-9);
    if (M == 1) v = 1.0 / v;
    if (threadIdx.x == ((st + 1) & 127)) s[par ^ 1][(st + 1) & 31] = v;
    asm volatile("bar.sync 1, 128;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = v;
}
int main() {
  double* d; long long* c; long long h;
  cudaMalloc(&d, 8 * 1024); cudaMalloc(&c, 8);
  k<0><<<1, 128>>>(d, c); k<0><<<1, 128>>>(d, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("publish->bar->read->fma: %.1f cycles/step\n", h / 256.0);
  k<1><<<1, 128>>>(d, c); k<1><<<1, 128>>>(d, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("  + 1.0/v: %.1f cycles/step\n", h / 256.0);
  return 0;
}
