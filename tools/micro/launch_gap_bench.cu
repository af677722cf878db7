// Dependent-launch gap on B200: 2000 back-to-back small kernels on one
// stream, each reading what the previous one wrote, launched (a) plainly,
// (b) with programmatic dependent launch (PDL: the next grid is launched
// early and waits in griddepcontrol.wait), (c) as one CUDA graph.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a launch_gap_bench.cu -o launch_gap_bench
#include <cuda_runtime.h>

#include <cstdio>

__global__ void step_kernel(double* x, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 0.5 + 1.0;
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}

int main() {
  const int n = 1 << 14, reps = 2000;
  double* x;
  cudaMalloc(&x, n * sizeof(double));
  cudaMemset(x, 0, n * sizeof(double));
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int grid : {1, 64, 148}) {
    const int blocks = grid, thr = 128;
    // (a) plain
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0, s);
      for (int r = 0; r < reps; ++r) step_kernel<<<blocks, thr, 0, s>>>(x, n, 0);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
    }
    float ms_plain;
    cudaEventElapsedTime(&ms_plain, e0, e1);
    // (b) PDL
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(thr);
    cfg.stream = s;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    float ms_pdl = 0;
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0, s);
      for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, step_kernel, x, n, 1);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms_pdl, e0, e1);
    // (c) graph
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int r = 0; r < reps; ++r) step_kernel<<<blocks, thr, 0, s>>>(x, n, 0);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    float ms_graph = 0;
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms_graph, e0, e1);
    printf("grid %3d: plain %.2f us/kernel | PDL %.2f us/kernel | graph %.2f us/kernel | %s\n", grid,
           1e3 * ms_plain / reps, 1e3 * ms_pdl / reps, 1e3 * ms_graph / reps,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
