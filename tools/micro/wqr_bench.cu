// Phase timing of the warp-level Householder QR leaf (development tool):
// cycles per column the owner warp spends forming a reflector, the next
// column's owner waits at the CTA barrier, and applies the reflector.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2506_04732_b200/csrc \
//     tools/micro/wqr_bench.cu build/{als,api,blas,iterative,lu,lu_fused,tt,gj_solve,partition}.o -o build/micro/wqr_bench
#include <cstdlib>
#include <vector>
#define WQR_MICRO
#include "../../paper_2506_04732_b200/csrc/linalg.cu"

template <int RPL, int CPW>
static void run(int m, int n) {
  using namespace t2s2;
  std::vector<double> h((size_t)m * n);
  srand(3);
  for (auto& v : h) v = rand() / (double)RAND_MAX - 0.5;
  double *A, *R;
  cudaMalloc(&A, h.size() * 8);
  cudaMalloc(&R, (size_t)n * n * 8);
  cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const int nw = (n + CPW - 1) / CPW, thr = 32 * (nw < 2 ? 2 : nw);
  const size_t smem = ((size_t)m * n + (size_t)n * n + n) * sizeof(double);
  auto k = wqr_kernel<RPL, CPW, false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k<<<1, thr, smem>>>(m, n, m, A, nullptr, R, 1, nullptr, 0, nullptr);
  unsigned long long z[4] = {};
  cudaMemcpyToSymbol(g_wqr_t, z, sizeof z);
  const int reps = 20;
  cudaEventRecord(e0);
  for (int w = 0; w < reps; ++w) k<<<1, thr, smem>>>(m, n, m, A, nullptr, R, 1, nullptr, 0, nullptr);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaMemcpyFromSymbol(z, g_wqr_t, sizeof z);
  const double den = (double)reps * n;
  printf("%4d x %2d  RPL %2d CPW %d  %3d threads  %6.1f us  per column: form %5.0f  barrier wait %5.0f  apply %5.0f cycles (%s)\n",
         m, n, RPL, CPW, thr, ms * 1e3 / reps, z[0] / den, z[1] / den, z[2] / den, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<4, 1>(99, 3);
  run<4, 1>(128, 12);
  run<12, 1>(352, 12);
  run<4, 2>(76, 21);
  run<12, 2>(314, 29);
  run<8, 4>(231, 35);
  run<4, 4>(105, 35);
  return 0;
}
