// Micro-benchmark of the one-CTA thin SVD on split-sized matrices
// (development tool).  Links against the engine objects:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2506_04732_b200/csrc \
//     tools/micro/svd_bench.cu build/{als,api,blas,iterative,lu,lu_fused,tt,gj_solve}.o -o tools/micro/svd_bench
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cmath>
#define SVD_MICRO
#include "../../paper_2506_04732_b200/csrc/linalg.cu"

// ||A - U S Vt|| / ||A|| and max |U^T U - I|, |V V^T - I| (host)
static void check(int m, int n, const std::vector<double>& A, double* dU, double* ds, double* dVt,
                  double& rec, double& ou, double& ov) {
  const int np = m < n ? m : n;
  const int uc = m >= n ? n : m;  // U columns
  std::vector<double> U((size_t)m * uc), s(np), Vt((size_t)np * n);
  cudaMemcpy(U.data(), dU, U.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(s.data(), ds, s.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(Vt.data(), dVt, Vt.size() * 8, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      double v = 0;
      for (int k = 0; k < np; ++k) v += U[(size_t)i * uc + k] * s[k] * Vt[(size_t)k * n + j];
      num += (v - A[(size_t)i * n + j]) * (v - A[(size_t)i * n + j]);
      den += A[(size_t)i * n + j] * A[(size_t)i * n + j];
    }
  rec = std::sqrt(num / den);
  ou = 0; ov = 0;
  for (int a = 0; a < np; ++a)
    for (int b = 0; b < np; ++b) {
      double x = 0, y = 0;
      for (int i = 0; i < m; ++i) x += U[(size_t)i * uc + a] * U[(size_t)i * uc + b];
      for (int j = 0; j < n; ++j) y += Vt[(size_t)a * n + j] * Vt[(size_t)b * n + j];
      ou = std::max(ou, std::fabs(x - (a == b)));
      ov = std::max(ov, std::fabs(y - (a == b)));
    }
}

int main(int argc, char** argv) {
  using namespace t2s2;
  const int shapes[][2] = {{66, 4}, {132, 8}, {264, 8}, {198, 11}, {231, 11}, {264, 16}, {8, 264},
                           {33, 1}, {1, 33}, {4, 33}, {12, 66}, {100, 3}, {384, 16}, {16, 384}, {2, 50}, {33, 16}, {132, 12}, {396, 12}, {627, 12}};
  for (auto& sh : shapes) {
    const int m = sh[0], n = sh[1];
    std::vector<double> h((size_t)m * n);
    srand(1);
    // low-rank-ish: rank n-2 plus 1e-13 noise, like a core near convergence
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) {
        double v = 0;
        for (int k = 0; k < n - 2; ++k) v += std::sin(0.37 * (i + 1) * (k + 1)) * std::cos(0.11 * (j + 1) * (k + 2)) / (1 + k * k);
        h[(size_t)i * n + j] = v + 1e-13 * ((rand() % 1000) / 1000.0 - 0.5);
        if (getenv("GRADED")) h[(size_t)i * n + j] = std::pow(10.0, -0.9 * (j % 17)) * std::sin(1.0 + 0.731 * i * (j + 1) + 0.1 * j * j) + 1e-3 * std::cos(0.3 * i + j);
      }
    double* A;
    cudaMalloc(&A, h.size() * 8);
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    const int mp = m >= n ? m : n, np = m >= n ? n : m;
    const size_t need = ((size_t)mp * np + 3 * (size_t)np * np + 4 * (size_t)np) * sizeof(double);
    cudaFuncSetAttribute(svd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap);
    double *U, *s, *Vt;
    cudaMalloc(&U, (size_t)mp * mp * 8);
    cudaMalloc(&s, np * 8);
    cudaMalloc(&Vt, (size_t)mp * np * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) svd_small_kernel<<<1, threads_for(np), need>>>(m, n, A, U, s, Vt);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int w = 0; w < reps; ++w) svd_small_kernel<<<1, threads_for(np), need>>>(m, n, A, U, s, Vt);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<double> hs(np), hs2(np), hu((size_t)mp * mp), hu2((size_t)mp * mp);
    cudaMemcpy(hs.data(), s, np * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hu.data(), U, (size_t)m * (m >= n ? n : m) * 8, cudaMemcpyDeviceToHost);
    double r1, u1, v1;
    check(m, n, h, U, s, Vt, r1, u1, v1);
    printf("   old: rec %.1e orthU %.1e orthV %.1e\n", r1, u1, v1);
    // the warp-level kernel
    const size_t wneed = (2 * (size_t)mp * np + 3 * (size_t)np * np + 2 * (size_t)np) * sizeof(double);
    auto wk = np <= 4 ? (mp <= 128 ? svd_warp_kernel<4, 4> : mp <= 256 ? svd_warp_kernel<8, 4> : svd_warp_kernel<12, 4>)
            : np <= 8 ? (mp <= 128 ? svd_warp_kernel<4, 8> : mp <= 256 ? svd_warp_kernel<8, 8> : svd_warp_kernel<12, 8>)
            : np <= 12 ? (mp <= 128 ? svd_warp_kernel<4, 12> : mp <= 256 ? svd_warp_kernel<8, 12> : svd_warp_kernel<12, 12>)
                      : (mp <= 128 ? svd_warp_kernel<4, 16> : mp <= 256 ? svd_warp_kernel<8, 16> : svd_warp_kernel<12, 16>);
    cudaFuncSetAttribute(wk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap);
    const int thr = 32 * (np < 2 ? 2 : np);
    for (int w = 0; w < 3; ++w) wk<<<1, thr, wneed>>>(m, n, A, U, s, Vt, t2s2::ReadTicket{});
    cudaEventRecord(e0);
    for (int w = 0; w < reps; ++w) wk<<<1, thr, wneed>>>(m, n, A, U, s, Vt, t2s2::ReadTicket{});
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms2;
    cudaEventElapsedTime(&ms2, e0, e1);
    cudaMemcpy(hs2.data(), s, np * 8, cudaMemcpyDeviceToHost);
    double r2, u2, v2;
    check(m, n, h, U, s, Vt, r2, u2, v2);
    printf("   new: rec %.1e orthU %.1e orthV %.1e\n", r2, u2, v2);
    cudaMemcpy(hu2.data(), U, (size_t)m * (m >= n ? n : m) * 8, cudaMemcpyDeviceToHost);
    double ds = 0, du = 0;
    for (int j = 0; j < np; ++j) ds = std::max(ds, std::fabs(hs[j] - hs2[j]) / hs[0]);
    // U columns up to sign, only for well-separated singular values (first n-2)
    const int ucols = m >= n ? n : m;
    for (int j = 0; j + 2 < np; ++j) {
      double dp = 0, dm = 0;
      for (int i = 0; i < m; ++i) {
        dp = std::max(dp, std::fabs(hu[(size_t)i * ucols + j] - hu2[(size_t)i * ucols + j]));
        dm = std::max(dm, std::fabs(hu[(size_t)i * ucols + j] + hu2[(size_t)i * ucols + j]));
      }
      du = std::max(du, std::min(dp, dm));
    }
    long long tw[8]; int sww;
    cudaMemcpyFromSymbol(tw, g_svd_t, sizeof(tw));
    cudaMemcpyFromSymbol(&sww, g_svd_sweeps, sizeof(int));
    printf("        svd_warp %7.1f us   max |ds|/s0 %.1e  max |dU| %.1e | qr %lld jacobi(warp0) %lld (%d sweeps) q+out %lld\n", ms2 * 1e3 / reps, ds, du, tw[1]-tw[0], tw[2]-tw[1], sww, tw[3]-tw[2]);
    cudaMemcpy(hs.data(), s, np * 8, cudaMemcpyDeviceToHost);
    long long t[8]; int sw;
    cudaMemcpyFromSymbol(t, g_svd_t, sizeof(t));
    cudaMemcpyFromSymbol(&sw, g_svd_sweeps, sizeof(int));
    printf("%4d x %-4d svd_small %7.1f us  qr %lld jacobi %lld (%d sweeps) sort+ur %lld formq %lld | s0 %.3e s_last %.3e  (%s)\n", m, n, ms * 1e3 / reps,
           t[1]-t[0], t[2]-t[1], sw, t[3]-t[2], t[4]-t[3], hs[0], hs[np - 1], cudaGetErrorString(cudaGetLastError()));
    cudaFree(A); cudaFree(U); cudaFree(s); cudaFree(Vt);
  }
  return 0;
}
