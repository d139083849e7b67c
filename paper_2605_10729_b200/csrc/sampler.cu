// Device-resident initial-condition samplers.
//
// The reference draws every particle attribute from its own counter-based
// stream, np.random.Generator(Philox(SeedSequence((seed, attr)))) (bench.py:67-68),
// indexed by global particle id, so any rank decomposition sees one global
// ensemble.  Philox4x64-10 is counter based: uint64 number j of a stream is
// word j & 3 of Philox(counter0 + 1 + j / 4, key), so each GPU thread computes
// its particle's draws directly, no state walk.  The host supplies counter0 and
// key (numpy derives them from the SeedSequence); uniforms are
// (raw >> 11) * 2^-53 like Generator.random.
//
// On top of the stream, the reference's transforms (bench.py:71-122):
//  * Landau positions: Newton inversion of (x + (alpha/k) sin kx)/L = u from
//    x = uL, per element frozen at the first iterate with |f| <= 1e-12, 60
//    checks, bisection rescue (200 halvings), then the periodic wrap;
//  * normals: Box-Muller sqrt(-2 log1p(-u1)) cos(2 pi u2) on rows 0 / 1 of a
//    (2, n) draw; Penning positions: the first in-box candidate of
//    mean + std * normal over REJECTION_BUDGET rows.
// Arithmetic is unfused (__dadd_rn / __dmul_rn / __ddiv_rn) in numpy's order;
// sin/cos/log1p are CUDA's (<= 1-2 ulp), so ensembles equal the host's to a
// few ulps rather than bit for bit (tests/test_gpu_parity.py checks this).

#include <cstdint>

#include "pif_internal.cuh"

namespace pif {
namespace {

struct PhiloxStream {
    unsigned long long ctr[4];
    unsigned long long key[2];
};

__device__ __forceinline__ unsigned long long philox_word(const PhiloxStream &s,
                                                         unsigned long long j) {
    const unsigned long long M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    const unsigned long long W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
    // counter = counter0 + 1 + j/4 as a 256-bit integer
    unsigned long long c[4];
    unsigned long long add = 1ull + (j >> 2), carry;
    c[0] = s.ctr[0] + add;
    carry = c[0] < add;
#pragma unroll
    for (int i = 1; i < 4; ++i) {
        c[i] = s.ctr[i] + carry;
        carry = carry && c[i] == 0;
    }
    unsigned long long k0 = s.key[0], k1 = s.key[1];
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += W0;
            k1 += W1;
        }
        const unsigned long long hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
        const unsigned long long hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
        const unsigned long long n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
    }
    return c[j & 3];
}

__device__ __forceinline__ double uniform(const PhiloxStream &s, unsigned long long j) {
    return (double)(philox_word(s, j) >> 11) * (1.0 / 9007199254740992.0);
}

// np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)
__device__ __forceinline__ double box_muller(double u1, double u2) {
    const double r = sqrt(__dmul_rn(-2.0, log1p(-u1)));
    return __dmul_rn(r, cos(__dmul_rn(6.283185307179586, u2)));
}

// (x + a sin(kx)) / L - u
__device__ __forceinline__ double landau_residual(double x, double a, double k, double L,
                                                  double u) {
    return __dsub_rn(__ddiv_rn(__dadd_rn(x, __dmul_rn(a, sin(__dmul_rn(k, x)))), L), u);
}

__global__ void landau_axis_kernel(PhiloxStream s, int64_t lo, int64_t count, double alpha,
                                   double k, double L, double *__restrict__ out, int64_t stride,
                                   int *__restrict__ status) {
    const double a = alpha / k;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double u = uniform(s, (unsigned long long)(lo + i));
        double x = __dmul_rn(u, L);
        bool done = false;
        for (int it = 0; it < 60; ++it) {
            const double f = landau_residual(x, a, k, L, u);
            if (fabs(f) <= 1e-12) {
                done = true;
                break;
            }
            const double fp = __ddiv_rn(__dadd_rn(1.0, __dmul_rn(alpha, cos(__dmul_rn(k, x)))), L);
            x = __dsub_rn(x, __ddiv_rn(f, fp));
        }
        if (!done) {   // bisection rescue (bench.py:94-106)
            double lo_b = 0.0, hi_b = L;
            for (int it = 0; it < 200; ++it) {
                const double mid = __dmul_rn(0.5, __dadd_rn(lo_b, hi_b));
                if (landau_residual(mid, a, k, L, u) > 0.0) hi_b = mid;
                else lo_b = mid;
            }
            x = __dmul_rn(0.5, __dadd_rn(lo_b, hi_b));
            if (fabs(landau_residual(x, a, k, L, u)) > 1e-10) atomicOr(status, 1);
        }
        out[i * stride] = wrap_coord(x, L);
    }
}

// budget == 0: plain N(0,1) (rows 0 / 1 of a (2, n_total) draw);
// budget > 0: first in-box mean + std * normal over rows i / budget + i of a
// (2 budget, n_total) draw (bench.py:113-122)
__global__ void normal_kernel(PhiloxStream s, int64_t n_total, int64_t lo, int64_t count,
                              double mean, double std_dev, int budget, double L,
                              double *__restrict__ out, int64_t stride, int *__restrict__ status) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long g = (unsigned long long)(lo + i), n = (unsigned long long)n_total;
        double v;
        if (budget == 0) {
            v = box_muller(uniform(s, g), uniform(s, n + g));
        } else {
            v = 0.0;
            bool found = false;
            for (int r = 0; r < budget && !found; ++r) {
                const double z = box_muller(uniform(s, (unsigned long long)r * n + g),
                                            uniform(s, (unsigned long long)(budget + r) * n + g));
                const double c = __dadd_rn(mean, __dmul_rn(std_dev, z));
                if (c >= 0.0 && c < L) {
                    v = c;
                    found = true;
                }
            }
            if (!found) atomicOr(status, 2);
        }
        out[i * stride] = v;
    }
}

int grid_for(int64_t count, int device) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int64_t blocks = (count + 255) / 256;
    return (int)(blocks < 8LL * sms ? (blocks > 0 ? blocks : 1) : 8LL * sms);
}

PhiloxStream make_stream(const uint64_t *ctr, const uint64_t *key) {
    PhiloxStream s;
    for (int i = 0; i < 4; ++i) s.ctr[i] = ctr[i];
    for (int i = 0; i < 2; ++i) s.key[i] = key[i];
    return s;
}

}  // namespace

}  // namespace pif

extern "C" int pif_sample_landau_axis(const uint64_t *counter, const uint64_t *key, int64_t lo,
                                      int64_t count, double alpha, double k, double L,
                                      double *out, int64_t stride, int *status, void *stream) {
    if (count < 0 || (count > 0 && (!counter || !key || !out || !status)) || stride < 1 ||
        !(k > 0) || !(L > 0) || !(alpha >= 0 && alpha < 1)) {
        pif::set_error("invalid Landau sampler arguments");
        return PIF_ERR_VALUE;
    }
    if (count == 0) return PIF_OK;
    int dev = 0;
    cudaGetDevice(&dev);
    pif::landau_axis_kernel<<<pif::grid_for(count, dev), 256, 0,
                              reinterpret_cast<cudaStream_t>(stream)>>>(
        pif::make_stream(counter, key), lo, count, alpha, k, L, out, stride, status);
    return pif::fail_cuda(cudaGetLastError(), "landau_axis_kernel");
}

extern "C" int pif_sample_normal(const uint64_t *counter, const uint64_t *key, int64_t n_total,
                                 int64_t lo, int64_t count, double mean, double std_dev,
                                 int budget, double L, double *out, int64_t stride, int *status,
                                 void *stream) {
    if (count < 0 || (count > 0 && (!counter || !key || !out || !status)) || stride < 1 ||
        budget < 0 || lo < 0 || lo + count > n_total) {
        pif::set_error("invalid normal sampler arguments");
        return PIF_ERR_VALUE;
    }
    if (count == 0) return PIF_OK;
    int dev = 0;
    cudaGetDevice(&dev);
    pif::normal_kernel<<<pif::grid_for(count, dev), 256, 0,
                         reinterpret_cast<cudaStream_t>(stream)>>>(
        pif::make_stream(counter, key), n_total, lo, count, mean, std_dev, budget, L, out, stride,
        status);
    return pif::fail_cuda(cudaGetLastError(), "normal_kernel");
}
