// Single-warp 32x32 LU in shared memory, variants (development tool).
#include <cstdio>
template <int M>
__global__ void k(const double* A, double* out, long long* cyc) {
  __shared__ double D[32 * 33];
  const int i = threadIdx.x;
  for (int c = 0; c < 32; ++c) D[c * 33 + i] = A[c * 32 + i] + (i == c ? 40.0 : 0.0);
  __syncwarp();
  long long t0 = clock64();
#pragma unroll 1
  for (int st = 0; st < 32; ++st) {
    const double piv = D[st * 33 + st];
    const double rinv = (M == 1) ? piv : 1.0 / piv;
    if (i > st) {
      const double l = D[st * 33 + i] * rinv;
      D[st * 33 + i] = l;
      if (M != 2) {
#pragma unroll 4
        for (int c = st + 1; c < 32; ++c) D[c * 33 + i] = fma(-l, D[c * 33 + st], D[c * 33 + i]);
      }
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (i == 0) cyc[0] = t1 - t0;
  for (int c = 0; c < 32; ++c) out[c * 32 + i] = D[c * 33 + i];
}
// register-resident variant: lane i holds row i, full unroll (for reference)
__global__ void kr(const double* A, double* out, long long* cyc) {
  const int i = threadIdx.x;
  double d[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) d[c] = A[c * 32 + i] + (i == c ? 40.0 : 0.0);
  long long t0 = clock64();
#pragma unroll
  for (int st = 0; st < 32; ++st) {
    const double piv = __shfl_sync(0xffffffffu, d[st], st);
    const double l = d[st] * (1.0 / piv);
    const double ml = i > st ? -l : 0.0;
    if (i > st) d[st] = l;
#pragma unroll
    for (int c = st + 1; c < 32; ++c) d[c] = fma(ml, __shfl_sync(0xffffffffu, d[c], st), d[c]);
  }
  long long t1 = clock64();
  if (i == 0) cyc[0] = t1 - t0;
#pragma unroll
  for (int c = 0; c < 32; ++c) out[c * 32 + i] = d[c];
}
// register-resident, rolled: lane i holds row i, the active column is
// always d[0] (the row is shifted left after each step)
__global__ void krot(const double* A, double* out, long long* cyc) {
  __shared__ double D[32 * 33];
  const int i = threadIdx.x;
  double d[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) d[c] = A[c * 32 + i] + (i == c ? 40.0 : 0.0);
  long long t0 = clock64();
#pragma unroll 1
  for (int st = 0; st < 32; ++st) {
    const double piv = __shfl_sync(0xffffffffu, d[0], st);
    const double l = d[0] * (1.0 / piv);
    const bool below = i > st;
    const double ml = below ? -l : 0.0;
    D[st * 33 + i] = below ? l : d[0];
#pragma unroll
    for (int c = 1; c < 32; ++c) d[c - 1] = fma(ml, __shfl_sync(0xffffffffu, d[c], st), d[c]);
    d[31] = 0.0;
  }
  long long t1 = clock64();
  if (i == 0) cyc[0] = t1 - t0;
  __syncwarp();
  for (int c = 0; c < 32; ++c) out[c * 32 + i] = D[c * 33 + i];
}
int main() {
  double *A, *o; long long* c; long long h;
  cudaMalloc(&A, 8 * 1024); cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8);
  cudaMemset(A, 0, 8 * 1024);
  const char* nm[3] = {"smem rolled", "smem rolled, no division", "smem rolled, no update loop"};
  for (int r = 0; r < 2; ++r) {
    k<0><<<1, 32>>>(A, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld\n", nm[0], h);
    k<1><<<1, 32>>>(A, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld\n", nm[1], h);
    k<2><<<1, 32>>>(A, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("%s: %lld\n", nm[2], h);
    kr<<<1, 32>>>(A, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("registers unrolled: %lld\n", h);
    krot<<<1, 32>>>(A, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("registers rolled (shifted rows): %lld\n", h);
  }
  return 0;
}
