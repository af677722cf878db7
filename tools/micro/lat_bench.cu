#include <cstdio>
template <int M>
__global__ void k(unsigned* out, double* dout, long long* cyc) {
  unsigned v = threadIdx.x * 2654435761u;
  double d = 1.0 + threadIdx.x * 1e-3;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 256; ++i) {
    if (M == 0) v = __reduce_max_sync(0xffffffffu, v) ^ threadIdx.x;
    else if (M == 1) v = __shfl_xor_sync(0xffffffffu, v, 1) ^ threadIdx.x;
    else if (M == 2) d = __drcp_rn(d);
    else if (M == 3) d = fma(d, 1.0000001, 1e-9);
    else if (M == 4) { __syncthreads(); v ^= 1; }
    else if (M == 5) v = __ballot_sync(0xffffffffu, (v & 1)) ^ threadIdx.x;
    else if (M == 6) d = 1.0 / d;
    else if (M == 7) v = v * 3u + 1u;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = v; dout[threadIdx.x] = d;
}
template <int M> void run(const char* name, int threads, unsigned* o, double* d, long long* c) {
  long long h;
  k<M><<<1, threads>>>(o, d, c); k<M><<<1, threads>>>(o, d, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-18s %6.1f cycles per dependent op\n", name, h / 256.0);
}
int main() {
  unsigned* o; double* d; long long* c;
  cudaMalloc(&o, 4096); cudaMalloc(&d, 8192); cudaMalloc(&c, 8);
  run<0>("REDUX.MAX", 32, o, d, c); run<1>("SHFL", 32, o, d, c); run<2>("drcp_rn", 32, o, d, c);
  run<3>("DFMA", 32, o, d, c); run<4>("syncthreads(512)", 512, o, d, c); run<5>("ballot", 32, o, d, c);
  run<6>("ddiv", 32, o, d, c); run<7>("IMAD", 32, o, d, c);
}
