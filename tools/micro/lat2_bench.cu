// Latency of single primitives on B200 (development tool).
#include <cstdio>
__device__ __forceinline__ double rcp_approx(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int M>
__global__ void k(double* dout, long long* cyc, int nthr) {
  __shared__ double sm[1024];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  double d = 1.0 + threadIdx.x * 1e-3, e = 0.5, f = 0.25;
  int idx = threadIdx.x & 7;
  long long t0 = clock64();
  if (threadIdx.x < nthr) {
#pragma unroll 16
  for (int i = 0; i < 256; ++i) {
    if (M == 0) d = fma(d, 1.0000001, 1e-9);
    else if (M == 1) d = d * 1.0000001;
    else if (M == 2) d = 1.0 / d;
    else if (M == 3) d = __drcp_rn(d);
    else if (M == 4) d = rcp_approx(d);
    else if (M == 5) { d = sm[idx]; idx = (int)d & 7; }
    else if (M == 6) { __syncthreads(); }
    else if (M == 7) dmma(d, e, d, f);
    else if (M == 8) { dmma(d, e, f, f); }
    else if (M == 9) d = sqrt(d) + 1.0;
    else if (M == 10) d = rsqrt(d) + 1.0;
    else if (M == 11) { int x = (int)d; d = (double)((x * 7 + 3) % 13) + 1.0; }
  }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  dout[threadIdx.x] = d + e;
}
template <int M>
void run(const char* name, int thr, int nthr) {
  double* d; long long* c; long long h;
  cudaMalloc(&d, 8 * 1024); cudaMalloc(&c, 8);
  k<M><<<1, thr>>>(d, c, nthr); k<M><<<1, thr>>>(d, c, nthr);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %6.1f cycles/op\n", name, h / 256.0);
}
int main() {
  run<0>("dfma dependent", 32, 32);
  run<1>("dmul dependent", 32, 32);
  run<2>("1.0/d dependent", 32, 32);
  run<3>("__drcp_rn dependent", 32, 32);
  run<4>("rcp.approx.f64 dependent", 32, 32);
  run<5>("lds dependent", 32, 32);
  run<6>("__syncthreads 256", 256, 256);
  run<6>("__syncthreads 1024", 1024, 1024);
  run<7>("dmma dependent (1 warp)", 32, 32);
  run<8>("dmma acc-only chain (1 warp)", 32, 32);
  run<8>("dmma acc chain (8 warps)", 256, 256);
  run<8>("dmma acc chain (16 warps)", 512, 512);
  run<0>("dfma dep (32 warps)", 1024, 1024);
  run<9>("sqrt dependent", 32, 32);
  run<10>("rsqrt dependent", 32, 32);
  run<11>("int mod + cvt dependent", 32, 32);
  return 0;
}
