// Cost of the pieces of one gj_diag step (development tool).
#include <cstdio>
struct S {
  alignas(32) double rowd[2][32];
  alignas(32) double rowx[2][32];
  double cold[2][32], colz[2][32], rinv[32];
};
template <int M>
__global__ void k(double* out, long long* cyc) {
  __shared__ S s;
  const int tid = threadIdx.x, i = tid & 31, g = tid >> 5, j0 = 4 * g;
  if (tid < 32) {
    for (int p = 0; p < 2; ++p) { s.rowd[p][tid] = 1e-3 * tid; s.rowx[p][tid] = 2e-3 * tid; s.cold[p][tid] = 0.5; s.colz[p][tid] = 0.25; }
    s.rinv[tid] = 1.0;
  }
  double dv[4] = {1, 2, 3, 4}, xv[4] = {1, 0, 0, 1}, zv[4] = {0, 1, 1, 0};
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int st = 0; st < 32; ++st) {
    const int par = st & 1, nx = st + 1;
    if (M & 1) {
      const double rinv = s.rinv[st], cd = s.cold[par][i], cz = s.colz[par][i];
      const double4 u4 = *reinterpret_cast<const double4*>(&s.rowd[par][j0]);
      const double4 x4 = *reinterpret_cast<const double4*>(&s.rowx[par][j0]);
      const double ur[4] = {u4.x, u4.y, u4.z, u4.w}, xr[4] = {x4.x, x4.y, x4.z, x4.w};
      const double l = i > st ? cd * rinv : 0.0;
      const double y = i <= st ? cz * rinv : 0.0;
      if (M & 2) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = j0 + q;
          const bool ahead = j > st;
          dv[q] = fma(ahead ? -l : 0.0, ur[q], dv[q]);
          zv[q] = fma(ahead ? -y : 0.0, ur[q], zv[q]);
          xv[q] = fma(ahead ? 0.0 : -l, xr[q], xv[q]);
        }
      } else {
        dv[0] += l + ur[0] + ur[1] + ur[2] + ur[3]; xv[0] += y + xr[0] + xr[1] + xr[2] + xr[3];
      }
    }
    if ((M & 4) && nx < 32) {
      const int qn = nx - j0;
      if (qn >= 0 && qn < 4) {
        const double dc = qn == 0 ? dv[0] : qn == 1 ? dv[1] : qn == 2 ? dv[2] : dv[3];
        if (i == nx) s.rinv[nx] = (M & 8) ? 1.0 / dc : dc;
        s.cold[par ^ 1][i] = dc;
        s.colz[par ^ 1][i] = dc;
      }
      if (i == nx) {
        *reinterpret_cast<double4*>(&s.rowd[par ^ 1][j0]) = make_double4(dv[0], dv[1], dv[2], dv[3]);
        *reinterpret_cast<double4*>(&s.rowx[par ^ 1][j0]) = make_double4(xv[0], xv[1], xv[2], xv[3]);
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  out[tid] = dv[0] + dv[1] + dv[2] + dv[3] + xv[0] + xv[1] + xv[2] + xv[3] + zv[0] + zv[1] + zv[2] + zv[3];
}
template <int M> void run(const char* n) {
  double* d; long long* c; long long h;
  cudaMalloc(&d, 8 * 1024); cudaMalloc(&c, 8);
  k<M><<<1, 256>>>(d, c); k<M><<<1, 256>>>(d, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %7.1f cycles/step\n", n, h / 32.0);
}
int main() {
  run<0>("barrier only");
  run<1>("loads + l,y");
  run<3>("loads + fma");
  run<7>("loads + fma + stores");
  run<15>("loads + fma + stores + division");
  run<5>("loads + stores (no fma)");
  return 0;
}
