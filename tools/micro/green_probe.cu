// Feasibility probe: SM partitions (green contexts) for concurrent
// independent solves.  Splits the device's SMs into G groups, and in G host
// threads creates a green context per group, makes it current, allocates
// with cudaMallocAsync on a stream of that context, and runs cooperative
// kernels (grid = the group's SM count, a grid barrier inside) concurrently.
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a green_probe.cu -lcuda -o green_probe
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                   \
  do {                                                                          \
    CUresult r_ = (x);                                                          \
    if (r_ != CUDA_SUCCESS) {                                                   \
      const char* s_;                                                           \
      cuGetErrorString(r_, &s_);                                                \
      printf("%s failed: %s (line %d)\n", #x, s_, __LINE__);                    \
      return;                                                                   \
    }                                                                           \
  } while (0)
#define RK(x)                                                                   \
  do {                                                                          \
    cudaError_t r_ = (x);                                                       \
    if (r_ != cudaSuccess) {                                                    \
      printf("%s failed: %s (line %d)\n", #x, cudaGetErrorString(r_), __LINE__); \
      return;                                                                   \
    }                                                                           \
  } while (0)

__global__ void spin_kernel(double* x, int n, int rounds) {
  cg::grid_group g = cg::this_grid();
  for (int r = 0; r < rounds; ++r) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
      x[i] = x[i] * 0.999 + 1.0;
    g.sync();
  }
}

void worker(CUgreenCtx gctx, int sms, int id, double* out_ms) {
  CUcontext c;
  CK(cuCtxFromGreenCtx(&c, gctx));
  CK(cuCtxSetCurrent(c));
  cudaStream_t s;
  RK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double* x = nullptr;
  const int n = 1 << 22;
  RK(cudaMallocAsync(&x, n * sizeof(double), s));
  RK(cudaMemsetAsync(x, 0, n * sizeof(double), s));
  int dev_sms = 0;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, 0);
  int rounds = 2000;
  void* args[] = {&x, (void*)&n, &rounds};
  auto t0 = std::chrono::steady_clock::now();
  for (int k = 0; k < 5; ++k)
    RK(cudaLaunchCooperativeKernel((void*)spin_kernel, dim3(sms), dim3(256), args, 0, s));
  RK(cudaStreamSynchronize(s));
  *out_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  double h = 0;
  RK(cudaMemcpy(&h, x, sizeof h, cudaMemcpyDeviceToHost));
  printf("group %d: %d SMs (device attr says %d), 5 cooperative launches %.1f ms, x[0]=%.3f\n", id,
         sms, dev_sms, *out_ms, h);
  RK(cudaFreeAsync(x, s));
  RK(cudaStreamSynchronize(s));
}

int main(int argc, char** argv) {
  const int G = argc > 1 ? atoi(argv[1]) : 4;
  cuInit(0);
  CUdevice dev;
  cuDeviceGet(&dev, 0);
  cudaFree(0);  // primary context
  CUdevResource all;
  if (cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) {
    printf("no SM resource\n");
    return 1;
  }
  printf("device SMs %u\n", all.sm.smCount);
  std::vector<CUdevResource> parts(G);
  unsigned ng = G;
  CUdevResource rest;
  const unsigned per = all.sm.smCount / G;
  CUresult r = cuDevSmResourceSplitByCount(parts.data(), &ng, &all, &rest, 0, per);
  if (r != CUDA_SUCCESS) {
    const char* s;
    cuGetErrorString(r, &s);
    printf("split failed: %s\n", s);
    return 1;
  }
  printf("split into %u groups of %u SMs (+%u remaining)\n", ng, parts[0].sm.smCount,
         rest.sm.smCount);
  std::vector<CUgreenCtx> g(ng);
  for (unsigned i = 0; i < ng; ++i) {
    CUdevResourceDesc d;
    if (cuDevResourceGenerateDesc(&d, &parts[i], 1) != CUDA_SUCCESS ||
        cuGreenCtxCreate(&g[i], d, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
      printf("green ctx %u failed\n", i);
      return 1;
    }
  }
  std::vector<double> ms(ng);
  // serial reference: one group alone
  worker(g[0], parts[0].sm.smCount, 0, &ms[0]);
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (unsigned i = 0; i < ng; ++i) th.emplace_back(worker, g[i], (int)parts[i].sm.smCount, (int)i, &ms[i]);
  for (auto& t : th) t.join();
  printf("all %u groups concurrently: %.1f ms wall\n", ng,
         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  for (auto& x : g) cuGreenCtxDestroy(x);
  return 0;
}
