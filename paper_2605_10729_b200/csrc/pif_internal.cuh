// Internal declarations shared by the CUDA translation units of libpifb200.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <string>

#include "../../include/pif_b200.h"

// Bounds checks for debug builds (-DPIF_DEBUG_BOUNDS): compute-sanitizer is
// not available on the GPU pool, so the kernels check their own indices.
#ifdef PIF_DEBUG_BOUNDS
#include <cassert>
#define PIF_CHECK(cond) assert(cond)
#else
#define PIF_CHECK(cond) ((void)0)
#endif

namespace pif {

// Fused-kernel specialisations exist for stencil widths up to this value; wider
// windows (eps < 1e-8) take the generic one-thread-per-particle path.
constexpr int kMaxFastW = 8;    // DMMA kernels
constexpr int kMaxPolyW = 14;   // polynomial weights: pair rows a <= 6 (EsPoly)
constexpr int kMaxRingW = 17;   // FMA ring kernels (register ring of w slots per lane pair)
constexpr int kMaxW = 17;          // eps >= 1e-16 (nufft.py:74)
constexpr int kSub = 8;            // particles per warp sub-batch (fast kernels)
constexpr int kWarpsPerBlock = 4;  // fast kernels: one work item per warp
constexpr int kDiagSlots = 6;
constexpr int kItemParticles = 1024;   // max particles per work item
// push_agg from this many parts in the densest segment (A/B: Landau at 64 / 512
// per cell, 2 / 4 parts: per-lane REDs 2% faster; Penning 2^28 on one GPU,
// dozens of parts: aggregated counts 1.7x faster)
constexpr int kPushAggMinParts = 12;
constexpr int kMaxSeg = 127;           // max cells per z-segment work item (DMMA kernels)

// polynomial coefficients for the interior window weights (es_fast.cuh)
constexpr int kEsDegHost = 14;
struct EsPolyHost {
    double c[6][kEsDegHost + 1];
    int exact_mask;
};
void build_es_poly(int w, double beta, EsPolyHost *out, double *max_err);

struct Plan {
    int N = 0, n = 0, w = 0, device = 0;
    double L = 0, eps = 0, beta = 0, h = 0, inv_L3 = 0, half_L3 = 0;
    int64_t n3 = 0, nhalf = 0;     // n^3, n*n*(n/2+1)
    int seg = 8;                   // cells per z-segment work item (set per binning)
    int seg_target = 1024;         // particles per work item the segment length aims at
    double ring_spread_min = 0.1;   // ring kernels from this many particles per stencil cell
    double ring_gather_min = 0.75;  // (PIF_RING_SPREAD_MIN / PIF_RING_GATHER_MIN override, A/B)
    double density = 0.0;          // particles per stencil cell at the last binning
    double *ring_scratch = nullptr;  // E per position for the wide-window gather
    bool wcache_on = false;        // spread keeps its window weights for the next gather
    double *wcache = nullptr;
    int64_t wcache_cap = 0;
    bool wcache_valid = false;     // wcache matches (wcache_x, wcache_perm, wcache_count)
    const double *wcache_x = nullptr;
    const int32_t *wcache_perm = nullptr;
    int64_t wcache_count = 0;
    int64_t ring_scratch_cap = 0;
    double *mirror_x = nullptr;    // id-order (M,3) mirrors written by the push kernels
    double *mirror_v = nullptr;
    long long mirror_id0 = 0;
    // merged-column spread for sparse sets (spread_merged_kernel): C adjacent
    // x columns walked as one super-column in their own cell order
    // (cell_start2 / perm2 / items2, derived from the standard binning at each
    // spread); merge_force -1 auto, 0 or 1 off, 2 / 4 forced
    // (pif_set_spread_merge, PIF_SPREAD_MERGE)
    int merge_force = -1;
    int merge_used = 1;            // C of the last spread (1: standard kernel)
    int32_t *cell_start2 = nullptr;  // 2 (n^3 + 1): merged counts, then their scan
    int32_t *perm2 = nullptr;
    int64_t perm2_cap = 0;
    int2 *items2 = nullptr;
    int64_t items2_cap = 0;
    int *seg_parts2 = nullptr, *seg_off2 = nullptr;
    int64_t segs2_cap = 0;
    // split step (pif_interp_split / pif_push_ids): E rows in id order in
    // ring_scratch, valid for split_count rows; split_parts diagnostic
    // partial blocks used by the row chunks pushed so far
    bool split_valid = false;
    int64_t split_count = 0;
    int split_parts = 0;
    double *deconv = nullptr;      // (N,)
    double *kvec = nullptr;        // (N,) 2 pi m / L
    double *grid = nullptr;        // n^3 real fine grid
    double2 *spec = nullptr;       // 3 * nhalf complex: D2Z output / Z2D inputs
    double *field = nullptr;       // n^3 * 4 interleaved E grid
    double *field3 = nullptr;      // 3 * n^3 separate grids when strided C2R is unavailable
    double2 *emodes = nullptr;     // 3 * N^3 complex: E modes (shape applied) for padding
    double2 *cgrid = nullptr;      // n^3 complex grid (complex API, lazily allocated)
    int32_t *cell_count = nullptr; // n^3 + 1
    int32_t *cell_start = nullptr; // n^3 + 1
    void *scan_tmp = nullptr;
    size_t scan_tmp_bytes = 0;
    unsigned int *work = nullptr;  // work counters for persistent kernels (4)
    // work items = (z-segment, part) with parts of <= kItemParticles particles,
    // rebuilt after every binning (heavy Penning segments split across warps)
    int2 *items = nullptr;
    int64_t items_cap = 0;
    int *seg_parts = nullptr;      // n_segs + 1
    int *seg_off = nullptr;        // n_segs + 1; seg_off[n_segs] = number of items
    int *max_parts = nullptr;      // (1) most parts in one segment (push_agg decision)
    int *max_parts_host = nullptr; // mapped pinned copy of it
    // push_agg: the gather+push kernel counts next-cell keys per run of equal
    // keys in dense segments instead of per particle (heavy cells: per-lane
    // REDs to one counter serialise in L2).  Decided from the parts per
    // segment at the first binning after a load (agg_check; never inside a
    // graph capture); PIF_PUSH_AGG=0/1 forces it.
    bool push_agg = false;
    int64_t aos_id0 = 0;           // id of row 0 of the last pif_load_aos (velocities by id)
    bool agg_check = true;
    int push_agg_force = -1;
    int n_segs = 0;
    double *partials = nullptr;    // per-block diagnostic / reduction partials
    int partial_blocks = 0;
    unsigned long long *maxbits = nullptr;  // atomics for max reductions (8)
    double *shape_tab = nullptr;   // (2, N): delta, cic shape factors
    cufftHandle d2z = 0, z2d3 = 0, z2z = 0;
    bool z2d_strided = false;      // Z2D writes the interleaved grid directly
    bool field_valid = false;
    bool force_generic = false;
    bool force_ring = false;       // PIF_FORCE_RING: w = 8 through the ring kernels (A/B)     // env PIF_FORCE_GENERIC=1: one-thread-per-particle kernels
    int sm_count = 148;
    int64_t bytes = 0;
    // optional cuFFT timing (bench.py): event pairs around each D2Z / Z2D exec,
    // slot k of each ring holds the k-th exec since the last pif_fft_times
    // deterministic mode (pif_set_deterministic): stable binning + fixed-order
    // plane reduction instead of REDG, diagnostics from a fixed-order pass
    bool det = false;
    double *dbuf = nullptr;        // per-item plane slices of the spread
    int64_t dbuf_cap = 0;
    int32_t *det_keys = nullptr, *det_iota = nullptr;
    void *det_tmp = nullptr;
    size_t det_tmp_bytes = 0;
    int64_t det_cap = 0;
    cudaEvent_t *fft_ev = nullptr;  // [d2z begin, d2z end] x slots, then z2d pairs
    int fft_slots = 0, fft_nd = 0, fft_nz = 0;
    EsPolyHost poly{};              // interior weight polynomials for w <= 8
    double poly_err = 0;            // their max abs error (checked at creation)
};

void set_error(const std::string &msg);
int fail_cuda(cudaError_t e, const char *where);
int fail_cufft(cufftResult r, const char *where);
// record the begin (end=false) / end event of a cuFFT exec into the timing ring
// (no-op unless pif_fft_timing enabled it, and never inside a graph capture)
void fft_mark(Plan &p, bool z2d, bool end, cudaStream_t s);

// Kernel launchers (defined in the .cu files); all return PIF_* codes.
int launch_wrap(Plan &p, double *x, double *y, double *z, int64_t M, cudaStream_t s);
int launch_bin_keys(Plan &p, const pif_soa_t &src, int32_t *key, int32_t *rank, cudaStream_t s);
int launch_bin_scatter(Plan &p, const pif_soa_t &src, pif_soa_t &dst, const int32_t *key,
                       const int32_t *rank, bool vel, cudaStream_t s);
int build_items(Plan &p, int64_t M, cudaStream_t s);
bool det_supported(const Plan &p);   // the DMMA (w <= 8) kernels serve this plan
int debug_phase_cycles(unsigned long long *out);
int launch_soa_to_aos(Plan &p, const pif_soa_t &P, int64_t id0, double *ox, double *ov,
                      cudaStream_t s);
int launch_bin_perm(Plan &p, const int32_t *key, const int32_t *rank, int64_t M, int32_t *perm,
                    cudaStream_t s);
int launch_spread(Plan &p, const pif_soa_t &parts, const int32_t *perm, const double *strengths,
                  double q, cudaStream_t s);
int ensure_wcache(Plan &p, int64_t M);
int launch_type1_complex_sorted(Plan &p, const pif_soa_t &sorted, const double *s_re,
                                const double *s_im, double *modes, cudaStream_t s);
int launch_type2_complex_sorted(Plan &p, const double *modes, const pif_soa_t &sorted,
                                double *E_out, cudaStream_t s);
int launch_load_aos(Plan &p, const double *x, const double *v, int64_t id0, pif_soa_t &dst,
                    int32_t *key, int32_t *rank, cudaStream_t s);
int launch_load_velocities(Plan &p, const double *v, pif_soa_t &dst, cudaStream_t s);
int launch_permute(Plan &p, const pif_soa_t &src, int32_t *perm, pif_soa_t &dst, int what,
                   cudaStream_t s);
int launch_interp(Plan &p, const pif_soa_t &src, const int32_t *perm, pif_soa_t &dst, bool push,
                  double half, double dt, const double *tq, const double *sq, int has_b,
                  int e_kind, int32_t *key, int32_t *rank, double *diag, double *E_out,
                  cudaStream_t s);
int launch_interp_split(Plan &p, const pif_soa_t &src, const int32_t *perm, int64_t id0,
                        cudaStream_t s);
int launch_push_ids(Plan &p, double *x, double *v, int64_t M, int64_t r0, int64_t r1,
                    double half, double dt, const double *tq, const double *sq, int has_b,
                    int e_kind, double *diag, cudaStream_t s);
bool split_supported(const Plan &p);
int launch_particle_diag(Plan &p, const pif_soa_t &ps, int e_kind, double *diag, cudaStream_t s);
int launch_modes_from_spec(Plan &p, double *modes, cudaStream_t s);
int launch_solve_fields(Plan &p, const double *raw, int shape, double *rho_out, double *scalars,
                        bool energy, const double *ex, const double *ey, const double *ez,
                        cudaStream_t s);
int launch_field_energy(Plan &p, const double *rho, double *scalars, cudaStream_t s);
int launch_poisson(Plan &p, const double *rho, double *ex, double *ey, double *ez,
                   cudaStream_t s);
int launch_type1_complex(Plan &p, const double *pts, const double *vals, int64_t M,
                         double *modes, cudaStream_t s);
int launch_type2_complex(Plan &p, const double *modes, const double *pts, int64_t M,
                         double *out, cudaStream_t s);

// ----------------------------------------------------------------------------
// Device helpers
// ----------------------------------------------------------------------------

__host__ __device__ inline int pmod(int i, int n) {
    int m = i % n;
    return m < 0 ? m + n : m;
}

// First stencil index and scaled coordinate for one axis, in the reference's
// arithmetic: c = x / h (true division), i0 = ceil(c - w/2) (_kernels.py:19,74).
// c = x / h correctly rounded, as the reference computes it (_kernels.py:41-43):
// q = x * rh, rh = RN(1/h), corrected once by the exact residual x - q h
// (Markstein: with a correctly rounded reciprocal and q within an ulp of x/h,
// RN(q + r rh) = RN(x/h)).  Callers hoist rh = __drcp_rn(h) out of their loops.
__device__ __forceinline__ double axis_coord(double x, double h, double rh) {
    const double q = x * rh;
    return fma(fma(-q, h, x), rh, q);
}
__device__ __forceinline__ double stencil_start(double c, int w) {
    return ceil(__dsub_rn(c, 0.5 * w));
}

// Exponential-of-semicircle weight of grid point i0d + a for coordinate c:
// t = (c - i) * 2/w, u = max(1 - t^2, 0), exp(beta (sqrt(u) - 1))
// (_kernels.py:21-26), without FMA contraction so it rounds like the reference.
__device__ __forceinline__ double es_weight(double c, double i, double inv_half, double beta) {
    double t = __dmul_rn(__dsub_rn(c, i), inv_half);
    double u = __dsub_rn(1.0, __dmul_rn(t, t));
    u = u < 0.0 ? 0.0 : u;
    return exp(__dmul_rn(beta, __dsub_rn(sqrt(u), 1.0)));
}

__device__ __forceinline__ double wrap_coord(double x, double L) {
    // numpy float mod (sign follows the divisor) then the x == L guard
    // (particles.py:65-70).  For x in [-L, 2L) np.mod is x, x - L (exact,
    // Sterbenz) or x + L; anything farther takes the fmod route.
    double r;
    if (x >= 0.0 && x < L) return x;
    if (x >= L && x < L + L) {
        r = x - L;
    } else if (x < 0.0 && x >= -L) {
        r = x + L;
    } else {
        r = fmod(x, L);
        if (r != 0.0 && r < 0.0) r += L;
    }
    if (r >= L) r -= L;
    return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace pif
