// Micro-benchmark: 32x32 no-pivot factorisation by one warp in shared
// memory, variants of the reciprocal (development tool).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void diag_kernel(double* A, int reps, long long* cyc) {
  __shared__ double D[33 * 32];
  const int lane = threadIdx.x;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int c = 0; c < 32; ++c) D[c * 33 + lane] = A[c * 32 + lane] + (lane == c ? 40.0 : 0.0);
    __syncwarp();
    for (int s = 0; s < 32; ++s) {
      const double piv = D[s * 33 + s];
      double rinv;
      if (MODE == 0) rinv = 1.0 / piv;
      else if (MODE == 1) rinv = __drcp_rn(piv);
      else rinv = 1.0 / (float)piv;  // lower bound: fp32 reciprocal
      if (lane > s) {
        const double l = D[s * 33 + lane] * rinv;
        D[s * 33 + lane] = l;
        for (int c = s + 1; c < 32; ++c) D[c * 33 + lane] = fma(-l, D[c * 33 + s], D[c * 33 + lane]);
      }
      __syncwarp();
    }
    for (int c = 0; c < 32; ++c) A[c * 32 + lane] = D[c * 33 + lane] * 1e-3;
  }
  long long t1 = clock64();
  if (lane == 0) *cyc = (t1 - t0) / reps;
}

// V1: row in registers, pivot row by shuffles (full unroll)
__global__ void diag_reg(double* A, int reps, long long* cyc) {
  const int lane = threadIdx.x;
  long long t0 = clock64();
  for (int rr = 0; rr < reps; ++rr) {
    double r[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) r[c] = A[c * 32 + lane] + (lane == c ? 40.0 : 0.0);
#pragma unroll
    for (int s = 0; s < 32; ++s) {
      const double piv = __shfl_sync(0xffffffffu, r[s], s);
      const double l = r[s] * (1.0 / piv);
      if (lane > s) r[s] = l;
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c > s) {
          const double u = __shfl_sync(0xffffffffu, r[c], s);
          if (lane > s) r[c] = fma(-l, u, r[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < 32; ++c) A[c * 32 + lane] = r[c] * 1e-3;
  }
  long long t1 = clock64();
  if (lane == 0) *cyc = (t1 - t0) / reps;
}

// V2: shared memory, 8 columns per batch (loads before stores)
__global__ void diag_smem8(double* A, int reps, long long* cyc) {
  __shared__ double D[33 * 32];
  const int lane = threadIdx.x;
  long long t0 = clock64();
  for (int rr = 0; rr < reps; ++rr) {
    for (int c = 0; c < 32; ++c) D[c * 33 + lane] = A[c * 32 + lane] + (lane == c ? 40.0 : 0.0);
    __syncwarp();
    for (int s = 0; s < 32; ++s) {
      const double piv = D[s * 33 + s];
      const double rinv = 1.0 / piv;
      const double l = D[s * 33 + lane] * rinv;
      const bool act = lane > s;
      if (act) D[s * 33 + lane] = l;
      for (int c0 = (s + 1) & ~7; c0 < 32; c0 += 8) {
        double u[8], x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          u[q] = D[(c0 + q) * 33 + s];
          x[q] = D[(c0 + q) * 33 + lane];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (act && c0 + q > s) D[(c0 + q) * 33 + lane] = fma(-l, u[q], x[q]);
      }
      __syncwarp();
    }
    for (int c = 0; c < 32; ++c) A[c * 32 + lane] = D[c * 33 + lane] * 1e-3;
  }
  long long t1 = clock64();
  if (lane == 0) *cyc = (t1 - t0) / reps;
}

// V3: 256 threads, ping-pong buffers, one barrier per column (as np_diag)
__global__ void __launch_bounds__(256, 1) diag_pp(double* A, int reps, long long* cyc) {
  __shared__ double D0[33 * 32], D1[33 * 32], rinv[33];
  const int tid = threadIdx.x;
  long long t0 = clock64();
  for (int rr = 0; rr < reps; ++rr) {
    for (int e = tid; e < 1024; e += 256) {
      const int c = e >> 5, i = e & 31;
      D0[c * 33 + i] = A[c * 32 + i] + (i == c ? 40.0 : 0.0);
    }
    __syncthreads();
    if (tid == 0) rinv[0] = 1.0 / D0[0];
    __syncthreads();
    const int j = tid & 31, i0 = tid >> 5;
    double* Dc = D0;
    double* Dn = D1;
    for (int s = 0; s < 32; ++s) {
      const double ri = rinv[s];
      const double us = Dc[j * 33 + s];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = i0 + 8 * q;
        const double x = Dc[j * 33 + i];
        double v = x;
        if (i > s) {
          const double l = Dc[s * 33 + i] * ri;
          if (j > s) v = fma(-l, us, x);
          if (j == s) v = l;
        }
        Dn[j * 33 + i] = v;
        if (i == s + 1 && j == s + 1) rinv[s + 1] = 1.0 / v;
      }
      __syncthreads();
      double* t = Dc; Dc = Dn; Dn = t;
    }
    for (int e = tid; e < 1024; e += 256) {
      const int c = e >> 5, i = e & 31;
      A[c * 32 + i] = Dc[c * 33 + i] * 1e-3;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) *cyc = (t1 - t0) / reps;
}

__global__ void div_lat(double* out, double x, int n, long long* cyc) {
  double v = x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = 1.0 / (v + 1.0);
  long long t1 = clock64();
  *out = v;
  *cyc = (t1 - t0) / n;
}
__global__ void fma_lat(double* out, double x, int n, long long* cyc) {
  double v = x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = fma(v, 0.999, 1e-3);
  long long t1 = clock64();
  *out = v;
  *cyc = (t1 - t0) / n;
}

int main() {
  double* A; long long* c; double* o;
  cudaMalloc(&A, 32 * 32 * 8); cudaMalloc(&c, 8); cudaMalloc(&o, 8);
  cudaMemset(A, 0, 32 * 32 * 8);
  long long h;
  diag_kernel<0><<<1, 32>>>(A, 10, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("diag div   %lld cyc\n", h);
  diag_kernel<1><<<1, 32>>>(A, 10, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("diag drcp  %lld cyc\n", h);
  diag_kernel<2><<<1, 32>>>(A, 10, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("diag frcp  %lld cyc\n", h);
  diag_reg<<<1, 32>>>(A, 10, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("diag reg   %lld cyc\n", h);
  diag_smem8<<<1, 32>>>(A, 10, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("diag smem8 %lld cyc\n", h);
  diag_pp<<<1, 256>>>(A, 10, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("diag pp256 %lld cyc\n", h);
  div_lat<<<1, 1>>>(o, 0.5, 1000, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("ddiv latency %lld cyc\n", h);
  fma_lat<<<1, 1>>>(o, 0.5, 1000, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("dfma latency %lld cyc\n", h);
  return 0;
}
