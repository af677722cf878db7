// Grid barrier cost on B200: cooperative_groups grid.sync() against a
// monotonic arrival counter (fence + red.add, volatile spin, fence) — the
// barrier of csrc/grid_barrier.cuh.  Each round every CTA writes a word and
// reads its neighbour's after the barrier (checked), so the barrier is timed
// with the memory ordering it has to provide.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gbar tools/micro/gbar_bench.cu && /tmp/gbar
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
struct Bar {
  unsigned* ctr;
  unsigned target, G;
};
__device__ __forceinline__ void bar_sync(Bar& b) {
  __syncthreads();
  if (threadIdx.x == 0) {
    b.target += b.G;
    __threadfence();
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(b.ctr) : "memory");
    while ((int)(ld_relaxed(b.ctr) - b.target) < 0) {
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void k_cg(int reps, long long* cyc, unsigned* data, int* bad) {
  cg::grid_group grid = cg::this_grid();
  const unsigned G = gridDim.x, me = blockIdx.x;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) data[me] = r + 1;
    grid.sync();
    if (threadIdx.x == 32 && data[(me + 1) % G] != (unsigned)(r + 1)) atomicAdd(bad, 1);
    grid.sync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / (2 * reps);
}
__global__ void k_bar(int reps, long long* cyc, unsigned* ctr, unsigned* data, int* bad) {
  Bar b{ctr, 0u, gridDim.x};
  const unsigned G = gridDim.x, me = blockIdx.x;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) data[me] = r + 1;
    bar_sync(b);
    if (threadIdx.x == 32 && data[(me + 1) % G] != (unsigned)(r + 1)) atomicAdd(bad, 1);
    bar_sync(b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / (2 * reps);
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// one thread-block cluster = the whole grid; the hardware cluster barrier with release/acquire
__global__ void k_cluster(int reps, long long* cyc, unsigned* data, int* bad) {
  const unsigned G = gridDim.x, me = blockIdx.x;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) data[me] = r + 1;
    cluster_sync();
    if (threadIdx.x == 32 && data[(me + 1) % G] != (unsigned)(r + 1)) atomicAdd(bad, 1);
    cluster_sync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / (2 * reps);
}

int main() {
  long long* cyc;
  unsigned *ctr, *data;
  int* bad;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&ctr, 4);
  cudaMalloc(&data, 4 * 1024);
  cudaMalloc(&bad, 4);
  cudaMemset(bad, 0, 4);
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int G : {2, 4, 8, 16}) {
    int reps = 500;
    long long hc = 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cluster, reps, cyc, data, bad);
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
    int hbad = 0;
    cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost);
    printf("cluster of %2d CTAs: barrier.cluster %5lld cycles   stale reads %d (%s / %s)\n", G, hc, hbad,
           cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
  }
  for (int G : {2, 6, 16, 40, 75, 148, 296}) {
    int reps = 500;
    long long hc = 0, hb = 0;
    void* p1[] = {&reps, &cyc, &data, &bad};
    cudaLaunchCooperativeKernel((void*)k_cg, G, 256, p1, 0, 0);
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
    cudaMemset(ctr, 0, 4);
    void* p2[] = {&reps, &cyc, &ctr, &data, &bad};
    cudaLaunchCooperativeKernel((void*)k_bar, G, 256, p2, 0, 0);
    cudaMemcpy(&hb, cyc, 8, cudaMemcpyDeviceToHost);
    int hbad = 0;
    cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost);
    printf("G=%3d  grid.sync %5lld cycles   counter barrier %5lld cycles   stale reads %d (%s)\n", G, hc,
           hb, hbad, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
