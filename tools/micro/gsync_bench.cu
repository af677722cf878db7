// Grid barrier cost: cooperative_groups grid.sync() vs a spin barrier on a
// counter + generation word (development tool).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_barrier(unsigned* bar, unsigned nb) {
  // bar[0] = arrivals, bar[1] = generation
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acquire(bar + 1);
    __threadfence();
    const unsigned a = atomicAdd(bar, 1u);
    if (a == nb - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_acquire(bar + 1) == g) {
      }
    }
  }
  __syncthreads();
}

__global__ void k_cg(int reps, long long* cyc) {
  cg::grid_group grid = cg::this_grid();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) grid.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / reps;
}
__global__ void k_spin(int reps, long long* cyc, unsigned* bar) {
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) spin_barrier(bar, gridDim.x);
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / reps;
}

int main() {
  long long* cyc;
  unsigned* bar;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&bar, 8);
  cudaMemset(bar, 0, 8);
  long long h;
  for (int G : {2, 3, 16, 75, 148}) {
    int reps = 200;
    void* p1[] = {&reps, &cyc};
    cudaLaunchCooperativeKernel((void*)k_cg, G, 256, p1, 0, 0);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    long long hc = h;
    void* p2[] = {&reps, &cyc, &bar};
    cudaLaunchCooperativeKernel((void*)k_spin, G, 256, p2, 0, 0);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int one = 3;
    void* p3[] = {&one, &cyc};
    cudaEventRecord(e0);
    for (int i = 0; i < 100; ++i) cudaLaunchCooperativeKernel((void*)k_cg, G, 256, p3, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    void* p4[] = {&one, &cyc, &bar};
    cudaEventRecord(e0);
    for (int i = 0; i < 100; ++i) cudaLaunchCooperativeKernel((void*)k_spin, G, 256, p4, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms2; cudaEventElapsedTime(&ms2, e0, e1);
    printf("G=%3d  grid.sync %5lld cycles  spin %5lld cycles | launch+3 syncs: cg %.1f us, spin %.1f us (%s)\n",
           G, hc, h, ms * 10, ms2 * 10, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
