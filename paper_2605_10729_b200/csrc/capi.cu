// C ABI of libpifb200 (include/pif_b200.h): plan lifetime, argument checks,
// device selection and dispatch to the kernel launchers.
#include <cub/cub.cuh>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "pif_internal.cuh"

namespace pif {

static thread_local std::string g_error;

void set_error(const std::string &msg) { g_error = msg; }

int fail_cuda(cudaError_t e, const char *where) {
    if (e == cudaSuccess) return PIF_OK;
    set_error(std::string(where) + ": " + cudaGetErrorString(e));
    return PIF_ERR_CUDA;
}

int fail_cufft(cufftResult r, const char *where) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "%s: cufft error %d", where, (int)r);
    set_error(buf);
    return PIF_ERR_CUDA;
}

namespace {

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

template <typename T>
int dalloc(Plan &p, T **ptr, size_t count) {
    cudaError_t e = cudaMalloc(reinterpret_cast<void **>(ptr), sizeof(T) * count);
    if (e != cudaSuccess) return fail_cuda(e, "cudaMalloc");
    p.bytes += (int64_t)(sizeof(T) * count);
    return PIF_OK;
}

void release(Plan &p) {
    void *ptrs[] = {p.deconv, p.kvec, p.grid, p.spec, p.field, p.field3, p.emodes, p.cgrid,
                    p.cell_count, p.cell_start, p.scan_tmp, p.work, p.partials, p.maxbits,
                    p.shape_tab, p.items, p.seg_parts, p.seg_off, p.max_parts, p.ring_scratch, p.wcache,
                    p.dbuf, p.det_keys, p.det_iota, p.det_tmp, p.cell_start2, p.perm2,
                    p.items2, p.seg_parts2, p.seg_off2};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    if (p.max_parts_host) cudaFreeHost(p.max_parts_host);
    if (p.d2z) cufftDestroy(p.d2z);
    if (p.z2d3) cufftDestroy(p.z2d3);
    if (p.fft_ev) {
        for (int i = 0; i < 4 * p.fft_slots; ++i) cudaEventDestroy(p.fft_ev[i]);
        delete[] p.fft_ev;
        p.fft_ev = nullptr;
        p.fft_slots = 0;
    }
    if (p.z2z) cufftDestroy(p.z2z);
}

bool soa_ok(const pif_soa_t *s, bool vel) {
    if (!s || s->count < 0) return false;
    if (s->count == 0) return true;
    if (!s->x || !s->y || !s->z || !s->id) return false;
    if (vel && (!s->vx || !s->vy || !s->vz)) return false;
    return s->count < (int64_t)INT32_MAX;
}

int bad(const char *msg) {
    set_error(msg);
    return PIF_ERR_VALUE;
}

}  // namespace

int ensure_complex(Plan &p) {
    if (p.cgrid) return PIF_OK;
    DeviceGuard g(p.device);
    int rc = dalloc(p, &p.cgrid, p.n3);
    if (rc != PIF_OK) return rc;
    cufftResult r = cufftPlan3d(&p.z2z, p.n, p.n, p.n, CUFFT_Z2Z);
    if (r != CUFFT_SUCCESS) return fail_cufft(r, "cufftPlan3d(Z2Z)");
    return PIF_OK;
}

// Chebyshev interpolation (extended precision) of weight a as a function of
// u = 2f - 1, converted to monomials; each polynomial is verified on a fine grid
// and replaced by the exact formula (exact_mask) if it misses 4e-15.
void build_es_poly(int w, double beta, EsPolyHost *P, double *max_err) {
    std::memset(P, 0, sizeof(*P));
    double worst = 0.0;
    const int D = kEsDegHost;
    const long double pi = 3.141592653589793238462643383279502884L;
    const long double B = (long double)beta;
    auto phi = [&](long double t) {
        long double u = 1.0L - t * t;
        if (u < 0) u = 0;
        return expl(B * (sqrtl(u) - 1.0L));
    };
    // rows a = 1 .. (w-1)/2; weight w-1-a is the mirror p_a(-u) (es_fast.cuh)
    for (int a = 1; 2 * a <= w - 1 && a <= 6; ++a) {
        long double y[kEsDegHost + 1], cheb[kEsDegHost + 1];
        for (int k = 0; k <= D; ++k) {
            const long double un = cosl(pi * (k + 0.5L) / (D + 1));
            const long double f = 0.5L * (un + 1.0L);
            y[k] = phi(1.0L - (2.0L / w) * (a + f));
        }
        for (int j = 0; j <= D; ++j) {
            long double s = 0;
            for (int k = 0; k <= D; ++k) s += y[k] * cosl(pi * j * (k + 0.5L) / (D + 1));
            cheb[j] = (2.0L / (D + 1)) * s;
        }
        cheb[0] *= 0.5L;
        long double mono[kEsDegHost + 1] = {0}, t0[kEsDegHost + 1] = {0},
                    t1[kEsDegHost + 1] = {0}, t2[kEsDegHost + 1];
        t0[0] = 1.0L;
        t1[1] = 1.0L;
        for (int k = 0; k <= D; ++k) mono[k] += cheb[0] * t0[k] + cheb[1] * t1[k];
        for (int j = 2; j <= D; ++j) {
            for (int k = 0; k <= D; ++k) t2[k] = -t0[k] + (k ? 2.0L * t1[k - 1] : 0.0L);
            for (int k = 0; k <= D; ++k) {
                mono[k] += cheb[j] * t2[k];
                t0[k] = t1[k];
                t1[k] = t2[k];
            }
        }
        for (int k = 0; k <= D; ++k) P->c[a - 1][k] = (double)mono[k];
        // check exactly the device evaluation: E(u^2) +/- u O(u^2), both weights
        const double *cf = P->c[a - 1];
        double err = 0.0;
        for (int i = 0; i <= 4000; ++i) {
            const double f = i / 4000.0 * (1.0 - 1e-12);
            const double u = 2.0 * f - 1.0, v = u * u;
            double e = cf[D], o = cf[D - 1];
            for (int k = D / 2 - 1; k >= 0; --k) {
                e = std::fma(e, v, cf[2 * k]);
                if (k < (D - 1) / 2) o = std::fma(o, v, cf[2 * k + 1]);
            }
            const double pa = std::fma(u, o, e), pb = std::fma(-u, o, e);
            const long double fl = (long double)f;
            const double ea = std::fabs(pa - (double)phi(1.0L - (2.0L / w) * (a + fl)));
            const double eb = std::fabs(pb - (double)phi(1.0L - (2.0L / w) * (w - 1 - a + fl)));
            err = std::max(err, std::max(ea, eb));
        }
        if (err > 4e-15) {
            P->exact_mask |= 1 << (a - 1);
        } else if (err > worst) {
            worst = err;
        }
    }
    if (max_err) *max_err = worst;
}

}  // namespace pif

using pif::Plan;

struct pif_plan_s {
    Plan p;
};

extern "C" {

const char *pif_last_error(void) { return pif::g_error.c_str(); }

int pif_abi_version(void) { return 1; }

int pif_plan_create(const pif_plan_desc_t *d, int device, pif_plan_t *out) {
    if (!d || !out) return pif::bad("null plan descriptor");
    *out = nullptr;
    if (d->N < 4 || d->N % 2) return pif::bad("N must be even and >= 4");
    if (!(d->L > 0) || !std::isfinite(d->L)) return pif::bad("invalid L");
    if (d->w < 2 || d->w > pif::kMaxW) return pif::bad("window width out of range");
    if (d->n_up < d->N || d->n_up % 2) return pif::bad("invalid n_up");   // w may exceed n_up
    if ((int64_t)d->n_up * d->n_up * d->n_up >= (int64_t)INT32_MAX)
        return pif::bad("fine grid too large for 32-bit cell keys");
    if (!d->deconv || !d->kvec || !d->shape_cic) return pif::bad("missing host tables");
    pif::DeviceGuard guard(device);
    if (!guard.ok) return pif::fail_cuda(cudaErrorInvalidDevice, "cudaSetDevice");
    pif_plan_s *h = new (std::nothrow) pif_plan_s;
    if (!h) return pif::bad("out of host memory");
    Plan &p = h->p;
    p.N = d->N;
    p.n = d->n_up;
    p.w = d->w;
    p.device = device;
    p.L = d->L;
    p.eps = d->eps;
    p.beta = d->beta;
    p.h = d->L / d->n_up;  // NufftPlan.h (nufft.py:60-63)
    p.inv_L3 = d->inv_L3;
    p.half_L3 = d->half_L3;
    p.n3 = (int64_t)p.n * p.n * p.n;
    p.nhalf = (int64_t)p.n * p.n * (p.n / 2 + 1);
    const int64_t N3 = (int64_t)p.N * p.N * p.N;
    cudaDeviceGetAttribute(&p.sm_count, cudaDevAttrMultiProcessorCount, device);
    p.partial_blocks = p.sm_count * 32;
    pif::build_es_poly(p.w, p.beta, &p.poly, &p.poly_err);
    if (const char *fg = std::getenv("PIF_FORCE_GENERIC")) p.force_generic = std::atoi(fg) != 0;
    if (const char *st = std::getenv("PIF_SEG_TARGET")) p.seg_target = std::max(1, std::atoi(st));
    if (const char *fr = std::getenv("PIF_FORCE_RING")) p.force_ring = std::atoi(fr) != 0;
    if (const char *pa = std::getenv("PIF_PUSH_AGG")) p.push_agg_force = std::atoi(pa) != 0;
    if (const char *rs = std::getenv("PIF_RING_SPREAD_MIN")) p.ring_spread_min = std::atof(rs);
    if (const char *rg = std::getenv("PIF_RING_GATHER_MIN")) p.ring_gather_min = std::atof(rg);
    if (const char *sm = std::getenv("PIF_SPREAD_MERGE")) p.merge_force = std::atoi(sm);
    int rc = PIF_OK;
#define TRY(x)                    \
    do {                          \
        rc = (x);                 \
        if (rc != PIF_OK) goto fail; \
    } while (0)
    TRY(pif::dalloc(p, &p.deconv, p.N));
    TRY(pif::dalloc(p, &p.kvec, p.N));
    TRY(pif::dalloc(p, &p.shape_tab, 2 * p.N));
    TRY(pif::dalloc(p, &p.grid, p.n3));
    TRY(pif::dalloc(p, &p.spec, 3 * p.nhalf));
    TRY(pif::dalloc(p, &p.field, 4 * p.n3));
    TRY(pif::dalloc(p, &p.emodes, 3 * N3));
    TRY(pif::dalloc(p, &p.cell_count, p.n3 + 1));
    TRY(pif::dalloc(p, &p.cell_start, p.n3 + 1));
    TRY(pif::dalloc(p, &p.work, 4));
    p.n_segs = p.n * p.n * ((p.n + p.seg - 1) / p.seg);
    TRY(pif::dalloc(p, &p.seg_parts, p.n_segs + 1));
    TRY(pif::dalloc(p, &p.seg_off, p.n_segs + 1));
    TRY(pif::dalloc(p, &p.max_parts, 1));
    TRY(pif::dalloc(p, &p.partials, (size_t)p.partial_blocks * pif::kDiagSlots));
    TRY(pif::dalloc(p, &p.maxbits, 8));
    {
        cudaError_t e = cudaMemcpy(p.deconv, d->deconv, sizeof(double) * p.N, cudaMemcpyHostToDevice);
        if (e == cudaSuccess)
            e = cudaMemcpy(p.kvec, d->kvec, sizeof(double) * p.N, cudaMemcpyHostToDevice);
        double *ones = new double[p.N];
        for (int i = 0; i < p.N; ++i) ones[i] = 1.0;
        if (e == cudaSuccess)
            e = cudaMemcpy(p.shape_tab, ones, sizeof(double) * p.N, cudaMemcpyHostToDevice);
        delete[] ones;
        if (e == cudaSuccess)
            e = cudaMemcpy(p.shape_tab + p.N, d->shape_cic, sizeof(double) * p.N,
                           cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemset(p.cell_count, 0, sizeof(int32_t) * (p.n3 + 1));
        if (e == cudaSuccess) e = cudaMemset(p.seg_off, 0, sizeof(int) * (p.n_segs + 1));
        if (e == cudaSuccess) e = cudaMemset(p.field, 0, sizeof(double) * 4 * p.n3);
        if (e != cudaSuccess) {
            rc = pif::fail_cuda(e, "plan tables");
            goto fail;
        }
        size_t tmp = 0;
        e = cub::DeviceScan::ExclusiveSum(nullptr, tmp, p.cell_count, p.cell_start,
                                          (int)(p.n3 + 1));
        if (e != cudaSuccess) {
            rc = pif::fail_cuda(e, "scan sizing");
            goto fail;
        }
        p.scan_tmp_bytes = tmp;
        TRY(pif::dalloc(p, reinterpret_cast<char **>(&p.scan_tmp), tmp));
    }
    {
        cufftResult r = cufftPlan3d(&p.d2z, p.n, p.n, p.n, CUFFT_D2Z);
        if (r != CUFFT_SUCCESS) {
            rc = pif::fail_cufft(r, "cufftPlan3d(D2Z)");
            goto fail;
        }
        int dims[3] = {p.n, p.n, p.n};
        int inembed[3] = {p.n, p.n, p.n / 2 + 1};
        int onembed[3] = {p.n, p.n, p.n};
        // Z2D straight into the interleaved (Ex,Ey,Ez,0) grid: ostride 4, odist 1
        r = cufftPlanMany(&p.z2d3, 3, dims, inembed, 1, (int)p.nhalf, onembed, 4, 1, CUFFT_Z2D, 3);
        if (r == CUFFT_SUCCESS) {
            p.z2d_strided = true;
        } else {
            p.z2d3 = 0;
            r = cufftPlanMany(&p.z2d3, 3, dims, inembed, 1, (int)p.nhalf, onembed, 1, (int)p.n3,
                              CUFFT_Z2D, 3);
            if (r != CUFFT_SUCCESS) {
                rc = pif::fail_cufft(r, "cufftPlanMany(Z2D)");
                goto fail;
            }
            TRY(pif::dalloc(p, &p.field3, 3 * p.n3));
        }
    }
#undef TRY
    *out = h;
    return PIF_OK;
fail:
    pif::release(p);
    delete h;
    return rc;
}

int pif_plan_destroy(pif_plan_t plan) {
    if (!plan) return PIF_OK;
    {
        pif::DeviceGuard g(plan->p.device);
        cudaDeviceSynchronize();
        pif::release(plan->p);
    }
    delete plan;
    return PIF_OK;
}

int64_t pif_plan_device_bytes(pif_plan_t plan) { return plan ? plan->p.bytes : 0; }

int pif_debug_phase_cycles(unsigned long long *out) {
    if (!out) return pif::bad("null out");
    return pif::debug_phase_cycles(out);
}

int pif_es_poly_info(int w, double beta, double *max_err, int *exact_mask) {
    if (w < 2 || w > pif::kMaxPolyW || !(beta > 0)) return pif::bad("w must be in [2, 14]");
    pif::EsPolyHost P;
    double e = 0.0;
    pif::build_es_poly(w, beta, &P, &e);
    if (max_err) *max_err = e;
    if (exact_mask) *exact_mask = P.exact_mask;
    return PIF_OK;
}

#define PLAN_CHECK()                                          \
    if (!plan) return pif::bad("null plan");                  \
    Plan &p = plan->p;                                        \
    pif::DeviceGuard guard_(p.device);                        \
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);

int pif_wrap_points(pif_plan_t plan, double *x, double *y, double *z, int64_t M, void *stream) {
    PLAN_CHECK();
    if (M < 0 || (M > 0 && (!x || !y || !z))) return pif::bad("invalid points");
    return pif::launch_wrap(p, x, y, z, M, s);
}

int pif_bin_keys(pif_plan_t plan, const pif_soa_t *src, int32_t *key, int32_t *rank,
                 void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(src, false)) return pif::bad("invalid particle view");
    if (src->count > 0 && (!key || !rank)) return pif::bad("missing key/rank buffers");
    p.agg_check = true;   // a new particle set: re-decide push_agg at its binning
    return pif::launch_bin_keys(p, *src, key, rank, s);
}

int pif_bin_scatter(pif_plan_t plan, const pif_soa_t *src, pif_soa_t *dst, const int32_t *key,
                    const int32_t *rank, int with_velocity, void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(src, with_velocity) || !dst) return pif::bad("invalid particle view");
    pif_soa_t d = *dst;
    d.count = src->count;
    if (!pif::soa_ok(&d, with_velocity)) return pif::bad("invalid destination view");
    int rc = pif::launch_bin_scatter(p, *src, d, key, rank, with_velocity != 0, s);
    dst->count = d.count;
    return rc;
}

int pif_spread_sorted(pif_plan_t plan, const pif_soa_t *sorted, const double *strengths,
                      double q, void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(sorted, false)) return pif::bad("invalid particle view");
    return pif::launch_spread(p, *sorted, nullptr, strengths, q, s);
}

int pif_bin_perm(pif_plan_t plan, const int32_t *key, const int32_t *rank, int64_t M,
                 int32_t *perm, void *stream) {
    PLAN_CHECK();
    if (M < 0 || M >= (int64_t)INT32_MAX || (M > 0 && (!key || !perm)))
        return pif::bad("invalid binning arguments");
    return pif::launch_bin_perm(p, key, rank, M, perm, s);
}

int pif_spread_perm(pif_plan_t plan, const pif_soa_t *parts, const int32_t *perm,
                    const double *strengths, double q, void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(parts, false)) return pif::bad("invalid particle view");
    return pif::launch_spread(p, *parts, perm, strengths, q, s);
}

int pif_interp_push_perm(pif_plan_t plan, const pif_soa_t *src, const int32_t *perm,
                         pif_soa_t *dst, double half, double dt, const double tq[3],
                         const double sq[3], int has_b, int e_kind, int32_t *key, int32_t *rank,
                         double *diag, void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(src, true) || !dst) return pif::bad("invalid particle view");
    pif_soa_t d = *dst;
    d.count = src->count;
    if (!pif::soa_ok(&d, true)) return pif::bad("invalid destination view");
    if (src->count > 0 && (!key || !perm)) return pif::bad("missing key/perm");
    if (!diag) return pif::bad("null diag");
    if (e_kind != PIF_EXT_NONE && e_kind != PIF_EXT_QUADRUPOLE) return pif::bad("unknown e_kind");
    if (!(dt > 0)) return pif::bad("dt must be positive");
    if (d.x == src->x) return pif::bad("dst must not alias src");
    int rc = pif::launch_interp(p, *src, perm, d, true, half, dt, tq, sq, has_b, e_kind, key,
                                rank, diag, nullptr, s);
    dst->count = d.count;
    return rc;
}

int pif_interp_split(pif_plan_t plan, const pif_soa_t *src, const int32_t *perm, int64_t id0,
                     void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(src, false)) return pif::bad("invalid particle view");
    if (src->count > 0 && !perm) return pif::bad("missing perm");
    return pif::launch_interp_split(p, *src, perm, id0, s);
}

int pif_push_ids(pif_plan_t plan, double *x, double *v, int64_t M, int64_t row0, int64_t rows,
                 double half, double dt, const double tq[3], const double sq[3], int has_b,
                 int e_kind, double *diag, void *stream) {
    PLAN_CHECK();
    if (M < 0 || row0 < 0 || rows < 0 || row0 + rows > M) return pif::bad("invalid row range");
    if (M > 0 && (!x || !v)) return pif::bad("null x/v rows");
    if (!diag) return pif::bad("null diag");
    if (e_kind != PIF_EXT_NONE && e_kind != PIF_EXT_QUADRUPOLE) return pif::bad("unknown e_kind");
    if (!(dt > 0)) return pif::bad("dt must be positive");
    return pif::launch_push_ids(p, x, v, M, row0, row0 + rows, half, dt, tq, sq, has_b, e_kind,
                                diag, s);
}

int pif_set_spread_merge(pif_plan_t plan, int c) {
    if (!plan) return pif::bad("null plan");
    if (c != -1 && c != 0 && c != 1 && c != 2 && c != 4)
        return pif::bad("spread merge factor must be -1 (auto), 0/1 (off), 2 or 4");
    plan->p.merge_force = c;
    return PIF_OK;
}

int pif_spread_merge_used(pif_plan_t plan) {
    if (!plan) return pif::bad("null plan");
    return plan->p.merge_used;
}

int pif_split_supported(pif_plan_t plan) {
    if (!plan) return pif::bad("null plan");
    return pif::split_supported(plan->p) ? 1 : 0;
}


int pif_set_deterministic(pif_plan_t plan, int enable) {
    if (!plan) return pif::bad("null plan");
    Plan &p = plan->p;
    if (enable && !pif::det_supported(p))
        return pif::bad("deterministic mode covers the DMMA kernels only: window width w <= 8 "
                        "(eps >= 1e-7)");
    p.det = enable != 0;
    if (p.det) p.wcache_valid = false;
    return PIF_OK;
}

int pif_is_deterministic(pif_plan_t plan) { return plan && plan->p.det ? 1 : 0; }

int pif_push_aggregated(pif_plan_t plan) { return plan && plan->p.push_agg ? 1 : 0; }

int pif_fft_timing(pif_plan_t plan, int slots) {
    if (!plan) return pif::bad("null plan");
    if (slots < 0 || slots > 1 << 16) return pif::bad("slots out of range");
    Plan &p = plan->p;
    pif::DeviceGuard g(p.device);
    if (p.fft_ev) {
        cudaDeviceSynchronize();
        for (int i = 0; i < 4 * p.fft_slots; ++i) cudaEventDestroy(p.fft_ev[i]);
        delete[] p.fft_ev;
        p.fft_ev = nullptr;
    }
    p.fft_slots = p.fft_nd = p.fft_nz = 0;
    if (!slots) return PIF_OK;
    p.fft_ev = new (std::nothrow) cudaEvent_t[4 * slots];
    if (!p.fft_ev) return pif::bad("out of host memory");
    for (int i = 0; i < 4 * slots; ++i) {
        cudaError_t e = cudaEventCreate(&p.fft_ev[i]);
        if (e != cudaSuccess) {
            for (int j = 0; j < i; ++j) cudaEventDestroy(p.fft_ev[j]);
            delete[] p.fft_ev;
            p.fft_ev = nullptr;
            return pif::fail_cuda(e, "cudaEventCreate");
        }
    }
    p.fft_slots = slots;
    return PIF_OK;
}

int pif_fft_times(pif_plan_t plan, double *d2z_ms, double *z2d_ms, int *n_d2z, int *n_z2d) {
    if (!plan || !d2z_ms || !z2d_ms || !n_d2z || !n_z2d) return pif::bad("null argument");
    Plan &p = plan->p;
    pif::DeviceGuard g(p.device);
    double sums[2] = {0.0, 0.0};
    const int counts[2] = {p.fft_nd, p.fft_nz};
    for (int which = 0; which < 2; ++which) {
        for (int k = 0; k < counts[which]; ++k) {
            cudaEvent_t a = p.fft_ev[which * 2 * p.fft_slots + 2 * k];
            cudaEvent_t b = p.fft_ev[which * 2 * p.fft_slots + 2 * k + 1];
            float ms = 0.f;
            cudaError_t e = cudaEventSynchronize(b);
            if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
            if (e != cudaSuccess) return pif::fail_cuda(e, "cudaEventElapsedTime");
            sums[which] += ms;
        }
    }
    *d2z_ms = sums[0];
    *z2d_ms = sums[1];
    *n_d2z = counts[0];
    *n_z2d = counts[1];
    p.fft_nd = p.fft_nz = 0;
    return PIF_OK;
}

int pif_grid_to_modes(pif_plan_t plan, double *modes, void *stream) {
    PLAN_CHECK();
    if (!modes) return pif::bad("null modes");
    return pif::launch_modes_from_spec(p, modes, s);
}

int pif_solve_fields(pif_plan_t plan, const double *raw_modes, int shape, double *rho_out,
                     double *scalars, void *stream) {
    PLAN_CHECK();
    if (!raw_modes || !scalars) return pif::bad("null modes/scalars");
    if (shape != PIF_SHAPE_DELTA && shape != PIF_SHAPE_CIC) return pif::bad("unknown shape");
    return pif::launch_solve_fields(p, raw_modes, shape, rho_out, scalars, true, nullptr, nullptr,
                                    nullptr, s);
}

int pif_fields_from_modes(pif_plan_t plan, const double *ex, const double *ey, const double *ez,
                          int shape, double *scalars, void *stream) {
    PLAN_CHECK();
    if (!ex || !ey || !ez || !scalars) return pif::bad("null E modes/scalars");
    if (shape != PIF_SHAPE_DELTA && shape != PIF_SHAPE_CIC) return pif::bad("unknown shape");
    return pif::launch_solve_fields(p, nullptr, shape, nullptr, scalars, false, ex, ey, ez, s);
}

int pif_field_energy(pif_plan_t plan, const double *rho, double *scalars, void *stream) {
    PLAN_CHECK();
    if (!rho || !scalars) return pif::bad("null rho/scalars");
    return pif::launch_field_energy(p, rho, scalars, s);
}

int pif_poisson(pif_plan_t plan, const double *rho, double *ex, double *ey, double *ez,
                void *stream) {
    PLAN_CHECK();
    if (!rho || !ex || !ey || !ez) return pif::bad("null rho/E");
    return pif::launch_poisson(p, rho, ex, ey, ez, s);
}

int pif_interp_push(pif_plan_t plan, pif_soa_t *sorted, double half, double dt,
                    const double tq[3], const double sq[3], int has_b, int e_kind,
                    int32_t *key, int32_t *rank, double *diag, void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(sorted, true)) return pif::bad("invalid particle view");
    if (sorted->count > 0 && (!key || !rank)) return pif::bad("missing key/rank buffers");
    if (!diag) return pif::bad("null diag");
    if (e_kind != PIF_EXT_NONE && e_kind != PIF_EXT_QUADRUPOLE) return pif::bad("unknown e_kind");
    if (!(dt > 0)) return pif::bad("dt must be positive");
    return pif::launch_interp(p, *sorted, nullptr, *sorted, true, half, dt, tq, sq, has_b, e_kind,
                              key, rank, diag, nullptr, s);
}

int pif_interp_sorted(pif_plan_t plan, const pif_soa_t *sorted, double *E_out, void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(sorted, false)) return pif::bad("invalid particle view");
    if (sorted->count > 0 && !E_out) return pif::bad("null E_out");
    pif_soa_t v = *sorted;
    return pif::launch_interp(p, v, nullptr, v, false, 0.0, 1.0, nullptr, nullptr, 0, PIF_EXT_NONE,
                              nullptr, nullptr, nullptr, E_out, s);
}

int pif_interp_perm(pif_plan_t plan, const pif_soa_t *parts, const int32_t *perm, double *E_out,
                    void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(parts, false)) return pif::bad("invalid particle view");
    if (parts->count > 0 && (!E_out || !perm)) return pif::bad("null E_out/perm");
    pif_soa_t v = *parts;
    return pif::launch_interp(p, v, perm, v, false, 0.0, 1.0, nullptr, nullptr, 0, PIF_EXT_NONE,
                              nullptr, nullptr, nullptr, E_out, s);
}

int pif_soa_to_aos(pif_plan_t plan, const pif_soa_t *parts, int64_t id0, double *x_out,
                   double *v_out, void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(parts, v_out != nullptr) || (parts->count > 0 && !x_out))
        return pif::bad("invalid particle view / output");
    return pif::launch_soa_to_aos(p, *parts, id0, x_out, v_out, s);
}

int pif_set_id_order_output(pif_plan_t plan, double *x_out, double *v_out, int64_t id0) {
    if (!plan) return pif::bad("null plan");
    if ((x_out == nullptr) != (v_out == nullptr)) return pif::bad("x_out and v_out go together");
    plan->p.mirror_x = x_out;
    plan->p.mirror_v = v_out;
    plan->p.mirror_id0 = id0;
    return PIF_OK;
}

int pif_set_weight_cache(pif_plan_t plan, int enable) {
    if (!plan) return pif::bad("null plan");
    pif::Plan &p = plan->p;
    p.wcache_on = enable != 0;
    p.wcache_valid = false;
    if (!p.wcache_on && p.wcache) {
        cudaFree(p.wcache);
        p.wcache = nullptr;
        p.wcache_cap = 0;
    }
    return PIF_OK;
}

int pif_load_aos(pif_plan_t plan, const double *x, const double *v, int64_t id0, pif_soa_t *dst,
                 int32_t *key, int32_t *rank, void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(dst, true)) return pif::bad("invalid destination view");
    if (dst->count > 0 && (!x || !key)) return pif::bad("missing input / key");
    p.agg_check = true;
    return pif::launch_load_aos(p, x, v, id0, *dst, key, rank, s);
}

int pif_permute(pif_plan_t plan, const pif_soa_t *src, int32_t *perm, pif_soa_t *dst, int what,
                void *stream) {
    PLAN_CHECK();
    if (!src || !dst) return pif::bad("invalid particle view");
    const int all = PIF_PERMUTE_POSITIONS | PIF_PERMUTE_VELOCITIES | PIF_PERMUTE_RESET;
    if (what & ~all) return pif::bad("unknown permute flags");
    const bool vel = (what & PIF_PERMUTE_VELOCITIES) != 0;
    if (!pif::soa_ok(src, vel)) return pif::bad("invalid source view");
    pif_soa_t d = *dst;
    d.count = src->count;
    if (!pif::soa_ok(&d, vel)) return pif::bad("invalid destination view");
    if (d.count > 0 && !perm) return pif::bad("missing perm");
    if ((what & PIF_PERMUTE_POSITIONS) && d.x == src->x) return pif::bad("dst must not alias src");
    if (vel && d.vx == src->vx) return pif::bad("dst must not alias src");
    const int rc = pif::launch_permute(p, *src, perm, d, what, s);
    dst->count = d.count;
    return rc;
}

int pif_load_aos_velocities(pif_plan_t plan, const double *v, pif_soa_t *dst, void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(dst, true)) return pif::bad("invalid destination view");
    if (dst->count > 0 && !v) return pif::bad("missing velocities");
    return pif::launch_load_velocities(p, v, *dst, s);
}

int pif_particle_diag(pif_plan_t plan, const pif_soa_t *ps, int e_kind, double *diag,
                      void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(ps, true) || !diag) return pif::bad("invalid particle view");
    return pif::launch_particle_diag(p, *ps, e_kind, diag, s);
}

int pif_type1_complex(pif_plan_t plan, const double *pts, const double *vals, int64_t M,
                      double *modes, void *stream) {
    PLAN_CHECK();
    if (M < 0 || (M > 0 && (!pts || !vals)) || !modes) return pif::bad("invalid type1 arguments");
    return pif::launch_type1_complex(p, pts, vals, M, modes, s);
}

int pif_type2_complex(pif_plan_t plan, const double *modes, const double *pts, int64_t M,
                      double *out, void *stream) {
    PLAN_CHECK();
    if (M < 0 || (M > 0 && (!pts || !out)) || !modes) return pif::bad("invalid type2 arguments");
    return pif::launch_type2_complex(p, modes, pts, M, out, s);
}

int pif_type1_complex_sorted(pif_plan_t plan, const pif_soa_t *sorted, const double *s_re,
                             const double *s_im, double *modes, void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(sorted, false) || !modes) return pif::bad("invalid type1 arguments");
    if (sorted->count > 0 && (!s_re || !s_im)) return pif::bad("missing strengths");
    return pif::launch_type1_complex_sorted(p, *sorted, s_re, s_im, modes, s);
}

int pif_type2_complex_sorted(pif_plan_t plan, const double *modes, const pif_soa_t *sorted,
                             double *E_out, void *stream) {
    PLAN_CHECK();
    if (!pif::soa_ok(sorted, false) || !modes) return pif::bad("invalid type2 arguments");
    if (sorted->count > 0 && !E_out) return pif::bad("null output");
    return pif::launch_type2_complex_sorted(p, modes, *sorted, E_out, s);
}

}  // extern "C"
