// Timeline of one Gauss-Jordan solve (development tool): per phase, when a
// few CTAs wait, work and signal (globaltimer).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DGJ_MICRO -DGJ_TIMELINE \
//        -I paper_2506_04732_b200/csrc tools/micro/gj_timeline.cu -o tools/micro/gj_timeline_bench
//   tools/micro/gj_timeline_bench [N]
#include "../../paper_2506_04732_b200/csrc/gj_solve.cu"

#include <vector>

using namespace t2s2;

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 1848;
  const int npan = (N + kP - 1) / kP;
  std::vector<double> A((size_t)N * N), b(N);
  unsigned long long st = 7;
  auto rnd = [&] { st = st * 6364136223846793005ull + 1442695040888963407ull; return (double)(st >> 11) / 9007199254740992.0 - 0.5; };
  for (int c = 0; c < N; ++c) {
    double sum = 0;
    for (int r = 0; r < N; ++r) { A[(size_t)c * N + r] = rnd(); sum += fabs(A[(size_t)c * N + r]); }
    A[(size_t)c * N + c] += sum;
  }
  for (int r = 0; r < N; ++r) b[r] = rnd();
  double *dA, *db, *inv, *wbuf;
  int* info;
  unsigned* sync;
  unsigned long long* prof;
  cudaMalloc(&dA, sizeof(double) * N * N);
  cudaMalloc(&db, sizeof(double) * N);
  cudaMalloc(&inv, sizeof(double) * npan * kInv);
  cudaMalloc(&wbuf, sizeof(double) * 3 * kP * (N + 1));
  cudaMalloc(&info, 8);
  cudaMalloc(&sync, 4 * (npan + 3));
  cudaMalloc(&prof, 8 * 5 * 128 * 4);
  const int smem = sizeof(Smem);
  cudaFuncSetAttribute(gj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int G = 148;
  std::vector<unsigned long long> h(5 * 128 * 4);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dA, A.data(), sizeof(double) * N * N, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), sizeof(double) * N, cudaMemcpyHostToDevice);
    cudaMemset(sync, 0, 4 * (npan + 3));
    cudaMemset(prof, 0, 8 * 5 * 128 * 4);
    GjArgs a{N, dA, db, inv, wbuf, info, sync, prof};
    void* params[] = {&a};
    cudaLaunchCooperativeKernel((void*)gj_kernel, dim3(G), dim3(kThr), params, smem, 0);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h.data(), prof, 8 * h.size(), cudaMemcpyDeviceToHost);
  auto at = [&](int slot, int p, int k) { return (double)h[((size_t)slot * 128 + p) * 4 + k]; };
  const double t0 = at(0, 0, 0);
  printf("N=%d npan=%d  (us relative to CTA 0's phase-0 start)\n", N, npan);
  printf("phase | CTA0: wait-feeders special diag | start->published | workers (cta 1, 5, G/2, G-1): wait-arrivals wait-published work\n");
  double sw = 0, ss = 0, sd = 0, wa[4] = {}, wp[4] = {}, ww[4] = {};
  int cnt = 0;
  for (int p = 0; p + 1 < npan; ++p) {
    const double w = (at(0, p, 1) - at(0, p, 0)) / 1e3, sp = (at(0, p, 2) - at(0, p, 1)) / 1e3, d = (at(0, p, 3) - at(0, p, 2)) / 1e3;
    if (p % 8 == 4) {
      printf("%3d | %6.2f %6.2f %6.2f | %8.2f |", p, w, sp, d, (at(0, p, 3) - t0) / 1e3);
      for (int s = 1; s < 5; ++s)
        printf("  %5.2f %5.2f %6.2f", (at(s, p, 1) - at(s, p, 0)) / 1e3, (at(s, p, 2) - at(s, p, 1)) / 1e3, (at(s, p, 3) - at(s, p, 2)) / 1e3);
      printf("\n");
    }
    sw += w; ss += sp; sd += d; ++cnt;
    for (int s = 1; s < 5; ++s) { wa[s-1] += (at(s, p, 1) - at(s, p, 0)) / 1e3; wp[s-1] += (at(s, p, 2) - at(s, p, 1)) / 1e3; ww[s-1] += (at(s, p, 3) - at(s, p, 2)) / 1e3; }
  }
  printf("mean over %d phases: CTA0 wait %.2f special %.2f diag %.2f | total %.1f us\n", cnt, sw / cnt, ss / cnt, sd / cnt, (at(0, npan - 2, 3) - t0) / 1e3);
  for (int s = 0; s < 4; ++s) printf("  worker %d: wait-arrivals %.2f wait-published %.2f work %.2f\n", s, wa[s] / cnt, wp[s] / cnt, ww[s] / cnt);
  {
    // CTA 0's special tile in clock cycles (sum over the three repetitions):
    // info load, operand loads issued, first barrier, W + multiplier products, update product
    unsigned long long acc[8];
    cudaMemcpyFromSymbol(acc, g_sp_acc, sizeof acc);
    const double den = 3.0 * (npan - 1);
    printf("special tile cycles per phase: info %.0f  issue-loads %.0f  barrier(load latency) %.0f  W+check %.0f (products %.0f)  update %.0f\n",
           acc[1] / den, acc[2] / den, acc[3] / den, (acc[4] + acc[6]) / den, acc[6] / den, acc[5] / den);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
