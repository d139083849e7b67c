// Microbenchmark of the gather sub-batch: 48 f64 DMMAs against a 48-double
// register window, adding one ingredient at a time.  One warp per block;
// blocks/SM chosen by the caller.  Prints cycles per DMMA per warp and TF/s.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void k(const double *in, double *out, int iters, long long *cyc) {
    __shared__ double wx[8][33], wz[32][9];
    const int lane = threadIdx.x & 31, r = lane >> 2, c4 = lane & 3;
    for (int i = lane; i < 8 * 33; i += 32) (&wx[0][0])[i] = in[i % 64] * 1e-3;
    for (int i = lane; i < 32 * 9; i += 32) (&wz[0][0])[i] = in[(i + 7) % 64] * 1e-3;
    __syncwarp();
    double g[8][2][3];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int d = 0; d < 3; ++d) g[a][h][d] = in[(a * 6 + h * 3 + d + lane) & 63];
    double acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int j = (it * 8) & 31;
        double D[2][3][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int d = 0; d < 3; ++d) D[h][d][0] = D[h][d][1] = 0.0;
        double A[8][2];
        if (MODE == 0) {
#pragma unroll
            for (int a = 0; a < 8; ++a) A[a][0] = A[a][1] = 1e-3 * (a + 1);
        } else {
            const int pb = (j + r) & 31;
            const double bz0 = wz[pb][(c4 - it) & 7], bz1 = wz[pb][(c4 + 4 - it) & 7];
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const double w = wx[a][pb];
                A[a][0] = w * bz0;
                A[a][1] = w * bz1;
            }
        }
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int d = 0; d < 3; ++d) dmma(D[h][d][0], D[h][d][1], A[a][h], g[a][h][d]);
        double e[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) e[d] = D[0][d][0] + D[1][d][0] + D[0][d][1] + D[1][d][1];
        if (MODE == 2) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                e[d] += __shfl_xor_sync(0xffffffffu, e[d], 1);
                e[d] += __shfl_xor_sync(0xffffffffu, e[d], 2);
            }
        }
        acc += e[0] + e[1] + e[2];
    }
    long long t1 = clock64();
    out[blockIdx.x * 32 + lane] = acc;
    if (lane == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double *in, *out; long long *cyc;
    cudaMalloc(&in, 64 * 8); cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
    double h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0 + i * 0.01;
    cudaMemcpy(in, h, 512, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096;
    for (int mode = 0; mode < 3; ++mode)
        for (int wps : {1, 2, 3, 4, 8}) {   // warps per SMSP
            int blocks = 148 * 4 * wps;
            float ms; long long c;
            auto launch = [&]() {
                if (mode == 0) k<0><<<blocks, 32>>>(in, out, iters, cyc);
                if (mode == 1) k<1><<<blocks, 32>>>(in, out, iters, cyc);
                if (mode == 2) k<2><<<blocks, 32>>>(in, out, iters, cyc);
            };
            launch();
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            double fl = 2.0 * 256 * 48 * (double)iters * blocks * 32 / 32;
            printf("mode %d warps/SMSP %d: %.1f cycles/DMMA/warp, %.1f TF/s\n", mode, wps,
                   c / (48.0 * iters), fl / (ms * 1e-3) / 1e12);
        }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
