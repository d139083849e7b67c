// Probe: (1) f64 mma.m8n8k4 fragment layout, (2) fast ES-weight accuracy vs
// CUDA exp/sqrt, (3) DMMA dependent-chain latency.  nvcc -arch=sm_100a.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include "../paper_2605_10729_b200/csrc/pif_internal.cuh"
#include "../paper_2605_10729_b200/csrc/es_fast.cuh"

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// assumed layout: A[row=lane>>2][col=lane&3]; B[row=lane&3][col=lane>>2];
// D[row=lane>>2][col=2*(lane&3)+i]
__global__ void layout_k(const double* A, const double* B, double* D) {
  int l = threadIdx.x;
  double a = A[(l >> 2) * 4 + (l & 3)];
  double b = B[(l & 3) * 8 + (l >> 2)];
  double d0 = 0, d1 = 0;
  dmma(d0, d1, a, b);
  D[(l >> 2) * 8 + 2 * (l & 3)] = d0;
  D[(l >> 2) * 8 + 2 * (l & 3) + 1] = d1;
}
__global__ void weights_k(const double* c, const double* i, int n, double beta, double* err) {
  __shared__ double tab[32];
  if (threadIdx.x < 32) tab[threadIdx.x] = pif::kExp2Table[threadIdx.x];
  __syncthreads();
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double a = pif::es_weight(c[t], i[t], 0.25, beta);
  double b = pif::es_weight_fast(c[t], i[t], 0.25, beta, tab);
  err[2 * t] = fabs(a - b);
  err[2 * t + 1] = a > 0 ? fabs(a - b) / a : 0;
}
__global__ void lat_k(double* out, long long* cyc, int chains) {
  double d[8][2]; double a = threadIdx.x * 1e-3, b = 0.999;
  for (int j = 0; j < 8; ++j) d[j][0] = d[j][1] = 0;
  long long t0 = clock64();
  for (int it = 0; it < 1024; ++it) {
    if (chains == 1) { dmma(d[0][0], d[0][1], a, b); }
    else { for (int j = 0; j < 8; ++j) dmma(d[j][0], d[j][1], a, b); }
  }
  long long t1 = clock64();
  double s = 0; for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double hA[32], hB[32], hD[64], ref[64];
  for (int r = 0; r < 8; ++r) for (int c = 0; c < 4; ++c) hA[r * 4 + c] = r * 10 + c + 1;
  for (int r = 0; r < 4; ++r) for (int c = 0; c < 8; ++c) hB[r * 8 + c] = r * 0.5 + c * 3 - 2;
  for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) { double s = 0; for (int k = 0; k < 4; ++k) s += hA[r*4+k]*hB[k*8+c]; ref[r*8+c] = s; }
  double *dA, *dB, *dD; cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dD, 512);
  cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  layout_k<<<1, 32>>>(dA, dB, dD); cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
  double md = 0; for (int k = 0; k < 64; ++k) md = fmax(md, fabs(hD[k] - ref[k]));
  printf("layout max|D-ref| = %g  (%s)\n", md, md == 0 ? "layout OK" : "LAYOUT WRONG");
  const int n = 1 << 22;
  double *hc = (double*)malloc(8 * n), *hi = (double*)malloc(8 * n), *he = (double*)malloc(16 * n);
  srand(1);
  for (int t = 0; t < n; ++t) { double c = 256.0 * rand() / RAND_MAX; double i0 = ceil(c - 4); hc[t] = c; hi[t] = i0 + (t & 7); }
  hc[0] = 4.0; hi[0] = 0.0;  // t = 1 exactly
  double *dc, *di, *de; cudaMalloc(&dc, 8 * n); cudaMalloc(&di, 8 * n); cudaMalloc(&de, 16 * n);
  cudaMemcpy(dc, hc, 8 * n, cudaMemcpyHostToDevice); cudaMemcpy(di, hi, 8 * n, cudaMemcpyHostToDevice);
  for (double beta : {2.30 * 4, 2.30 * 8, 2.30 * 13, 2.30 * 17}) {
    weights_k<<<(n + 255) / 256, 256>>>(dc, di, n, beta, de);
    cudaMemcpy(he, de, 16 * n, cudaMemcpyDeviceToHost);
    double ma = 0, mr = 0; for (int t = 0; t < n; ++t) { ma = fmax(ma, he[2*t]); mr = fmax(mr, he[2*t+1]); }
    printf("fast weights beta=%.1f: max abs err %.3e  max rel err %.3e\n", beta, ma, mr);
  }
  long long* dcyc; cudaMalloc(&dcyc, 8); long long cyc;
  lat_k<<<1, 32>>>(dD, dcyc, 1); cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
  printf("DMMA dependent chain: %.1f cycles/DMMA\n", cyc / 1024.0);
  lat_k<<<1, 32>>>(dD, dcyc, 8); cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
  printf("DMMA 8 chains, 1 warp: %.1f cycles/DMMA\n", cyc / 8192.0);
  cudaError_t e = cudaDeviceSynchronize(); printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
