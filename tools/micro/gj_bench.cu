// Micro-benchmark of the Gauss-Jordan solve's pieces (development tool):
// gj_diag on one CTA, one tile task, and an empty grid barrier.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DGJ_MICRO \
//        -I paper_2506_04732_b200/csrc tools/micro/gj_bench.cu -o tools/micro/gj_bench
#include "../../paper_2506_04732_b200/csrc/gj_solve.cu"

using namespace t2s2;

__global__ void diag_loop(GjArgs a, int reps, long long* cyc) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem& s = *reinterpret_cast<Smem*>(smraw);
  for (int e = threadIdx.x; e < kP * 33; e += kThr) s.dg[e] = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < kP * kP; e += kThr) {
      const int c = e >> 5, i = e & 31;
      s.dg[c * 33 + i] = __ldcg(a.A + e) + (i == c ? 40.0 : 0.0);
    }
    gj_diag(a, 0, kP, s);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = (t1 - t0) / reps;
}

__global__ void tile_loop(GjArgs a, int reps, int want_w, long long* cyc) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem& s = *reinterpret_cast<Smem*>(smraw);
  const Phase ph(a.N, 1);
  load_inv(a, 1, s);
  TileRegs R;
  Task k = task_of(ph, 3 + blockIdx.x % 8);
  tile_load(a, ph, k, true, R);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const bool w = want_w || r == 0;
    tile_stage(R, w, s, r & 1);
    double cv[4][2][2];
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 2; ++j)
        for (int h = 0; h < 2; ++h) cv[i][j][h] = R.cv[i][j][h];
    __syncthreads();
    tile_load(a, ph, k, want_w, R);
    tile_compute(a, ph, k, cv, w, false, false, false, s, r & 1);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / reps;
}

// the special tile (next diagonal block, 32 x 32) followed by its factorisation
__global__ void special_loop(GjArgs a, int reps, long long* cyc) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem& s = *reinterpret_cast<Smem*>(smraw);
  const Phase ph(a.N, 1);
  long long tt = 0, td = 0;
  for (int r = 0; r < reps; ++r) {
    long long t0 = clock64();
    special_tile(a, ph, s, false);
    __syncthreads();
    long long t1 = clock64();
    for (int e = threadIdx.x; e < kP * 33; e += kThr) s.dg[e] += (e % 34 == 0) ? 40.0 : 0.0;
    __syncthreads();
    long long t2 = clock64();
    gj_diag(a, 2, kP, s);
    long long t3 = clock64();
    tt += t1 - t0;
    td += t3 - t2;
  }
  if (threadIdx.x == 0) {
    cyc[0] = tt / reps;
    cyc[1] = td / reps;
  }
}

__global__ void sync_loop(int reps, long long* cyc) {
  cg::grid_group grid = cg::this_grid();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) grid.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / reps;
}

// timing of the phases of one gj_diag call, thread 0 (clock64 stamps)
__global__ void diag_parts(GjArgs a, long long* out) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Smem& s = *reinterpret_cast<Smem*>(smraw);
  for (int e = threadIdx.x; e < kP * kP; e += kThr) {
    const int c = e >> 5, i = e & 31;
    s.dg[c * 33 + i] = __ldcg(a.A + e) + (i == c ? 40.0 : 0.0);
  }
  __syncthreads();
  long long t0 = clock64();
  gj_diag(a, 0, kP, s);
  long long t1 = clock64();
  __syncthreads();
  long long t2 = clock64();
  for (int r = 0; r < 32; ++r) __syncthreads();
  long long t3 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t3 - t2; }
}

int main() {
  const int N = 1024;
  double *A, *b, *inv, *wbuf;
  int* info;
  long long* cyc;
  cudaMalloc(&A, sizeof(double) * N * N);
  cudaMalloc(&b, sizeof(double) * N);
  cudaMalloc(&inv, sizeof(double) * 64 * kInv);
  cudaMalloc(&wbuf, sizeof(double) * 3 * kP * (N + 1));
  cudaMalloc(&info, 4);
  cudaMalloc(&cyc, 16);
  cudaMemset(A, 0, sizeof(double) * N * N);
  cudaMemset(inv, 0, sizeof(double) * 64 * kInv);
  cudaMemset(wbuf, 0, sizeof(double) * 3 * kP * (N + 1));
  GjArgs a{N, A, b, inv, wbuf, info, nullptr, nullptr};
  const int smem = sizeof(Smem);
  cudaFuncSetAttribute(diag_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(tile_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h;
  cudaFuncSetAttribute(diag_parts, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int it = 0; it < 3; ++it) {
    diag_parts<<<1, kThr, smem>>>(a, cyc);
    long long hh[2];
    cudaMemcpy(hh, cyc, 16, cudaMemcpyDeviceToHost);
    printf("diag_parts: gj_diag %lld cycles, 32 bare barriers %lld\n", hh[0], hh[1]);
    long long dt[8];
    cudaMemcpyFromSymbol(dt, g_diag_t, sizeof(dt));
    printf("   lu %lld inverses %lld dinv+store %lld | b0: leaf %lld panel %lld\n", dt[1]-dt[0], dt[2]-dt[1], dt[3]-dt[2], dt[4]-dt[6], dt[5]-dt[4]);
  }
  cudaFuncSetAttribute(special_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int it = 0; it < 2; ++it) {
    special_loop<<<1, kThr, smem>>>(a, 50, cyc);
    long long hh[2];
    cudaMemcpy(hh, cyc, 16, cudaMemcpyDeviceToHost);
    printf("special tile %lld cycles, then gj_diag %lld cycles (steady state)\n", hh[0], hh[1]);
  }
  for (int it = 0; it < 2; ++it) {
    diag_loop<<<1, kThr, smem>>>(a, 100, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("gj_diag: %lld cycles/call\n", h);
    for (int w = 0; w < 2; ++w) {
      tile_loop<<<148, kThr, smem>>>(a, 100, w, cyc);
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("gj_tile (148 CTAs, want_w=%d): %lld cycles/tile\n", w, h);
    }
    int reps = 1000;
    void* params[] = {&reps, &cyc};
    cudaLaunchCooperativeKernel((void*)sync_loop, 148, kThr, params, 0, 0);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("grid.sync (148 x %d): %lld cycles\n", kThr, h);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
