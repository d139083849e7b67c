// FP64 pipe probe: the roofline denominator for the FP64-bound PIF kernels.
// MEASURED_PEAKS.json carries HBM and bf16 tensor peaks only, so bench.py
// measures the DFMA peak live on the same GPU with this kernel (8 independent
// FMA chains per thread, 148 x 8 blocks of 256 threads).
#include "pif_internal.cuh"

namespace {
__global__ void dfma_probe_kernel(double *out, double s, int iters) {
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma(a[j], s, 0.5);
    }
    double t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += a[j];
    if (t == 123.456) out[0] = t;
}
}  // namespace

extern "C" int pif_probe_fp64(double *scratch, int blocks, int threads, int iters, void *stream,
                              double *flops_out) {
    if (!scratch || blocks < 1 || threads < 32 || iters < 1) {
        pif::set_error("invalid probe arguments");
        return PIF_ERR_VALUE;
    }
    dfma_probe_kernel<<<blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        scratch, 0.999, iters);
    if (flops_out) *flops_out = 2.0 * 8.0 * (double)blocks * threads * (double)iters;
    return pif::fail_cuda(cudaGetLastError(), "dfma_probe_kernel");
}
