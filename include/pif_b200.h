/*
 * pif_b200.h — C ABI of the B200-native particle-decomposition PIF step.
 *
 * Plain C: device pointers, sizes and a cudaStream_t passed as void*.  No torch
 * or C++ types cross this boundary.  Every entry point returns PIF_OK or an
 * error code; pif_last_error() gives the message of the calling thread's last
 * failure.  All launches are asynchronous on the given stream; nothing here
 * synchronises the device except pif_plan_create/pif_plan_destroy.
 *
 * Each group cites the reference interface it replaces
 * (/root/reference/pkg/src/pifsim/...; the "FFI" of the reference is its numba
 * kernels in _kernels.py, called from nufft.py / pif.py / strategies.py).
 *
 * Layouts:
 *   particles   structure of arrays (pif_soa_t), fp64, in HBM; id = int64
 *   fine grid   n^3 fp64, flat index (ix*n + iy)*n + iz      (_kernels.py:48-54)
 *   modes       (N,N,N) complex128 interleaved re/im, C order, m = index - N/2
 *               (spectral.py:1-6)
 *   field grid  n^3 x 4 fp64 interleaved (Ex, Ey, Ez, 0), plan-owned
 */
#ifndef PIF_B200_H
#define PIF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PIF_OK 0
#define PIF_ERR_VALUE 1       /* invalid argument: maps to ValueError          */
#define PIF_ERR_CUDA 2        /* CUDA / cuFFT / allocation failure: RuntimeError */
#define PIF_ERR_STATE 3       /* call out of order (e.g. no field solved yet)  */

#define PIF_SHAPE_DELTA 0     /* pif.py:77-78 */
#define PIF_SHAPE_CIC 1       /* pif.py:79-85 */
#define PIF_EXT_NONE 0        /* pif.py:50-51 */
#define PIF_EXT_QUADRUPOLE 1  /* pif.py:52-57 */
#define PIF_PERMUTE_POSITIONS 1   /* pif_permute: x, y, z, id           */
#define PIF_PERMUTE_VELOCITIES 2  /* pif_permute: vx, vy, vz              */
#define PIF_PERMUTE_RESET 4       /* pif_permute: then perm[i] = i        */

typedef struct pif_plan_s *pif_plan_t;

/* Particle view (structure of arrays, device memory, `count` particles). */
typedef struct {
    double *x, *y, *z;
    double *vx, *vy, *vz;
    int64_t *id;
    int64_t count;
} pif_soa_t;

const char *pif_last_error(void);
int pif_abi_version(void);

/* ---- plan: replaces nufft.make_plan / NufftPlan (nufft.py:43-84) ----------
 * All scalars and (N,) tables are computed on the host by the caller exactly
 * as the reference computes them (numpy), so the device sees identical
 * constants; the plan owns the cuFFT plans, the fine
 * grid, spectra, the interleaved field grid and the cell tables on `device`.
 * A plan carries the state of one particle set between calls (cell table,
 * field grid): use one plan per particle set / stream, not concurrently. */
typedef struct {
    int N;                   /* modes per dimension (even, >= 4)               */
    double L;                /* periodic box length                            */
    double eps;              /* NUFFT tolerance                                */
    int w;                   /* window width  ceil(|log10 eps|) + 1 (nufft.py:79) */
    double beta;             /* 2.30 w (nufft.py:81)                           */
    int n_up;                /* fine grid per dimension (nufft.py:82-83)        */
    const double *deconv;    /* host (N,) 1/psi_hat (nufft.py:57, 87-102)      */
    const double *kvec;      /* host (N,) 2 pi/L * m (spectral.py:57-60)       */
    const double *shape_cic; /* host (N,) cloud-in-cell S_k (pif.py:79-85)     */
    double inv_L3;           /* 1.0 / L**3 (pif.py:101)                        */
    double half_L3;          /* 0.5 * L**3 (spectral.py:91)                    */
} pif_plan_desc_t;

int pif_plan_create(const pif_plan_desc_t *desc, int device, pif_plan_t *out);
int pif_plan_destroy(pif_plan_t plan);
/* Bytes of device memory owned by the plan. */
int64_t pif_plan_device_bytes(pif_plan_t plan);
/* Host-only: the interior ES-weight polynomials a plan builds for window w
 * (es_fast.cuh): max abs error vs the exact window on 4001 points, and the mask
 * of weights that fall back to the exact formula.  w in [2, 8]. */
int pif_es_poly_info(int w, double beta, double *max_err, int *exact_mask);

/* ---- binning (new; the reference spreads in particle order, _kernels.py:73) -
 * pif_bin_keys: per-particle ES-stencil cell key ((i0x*n + i0y)*n + i0z, each
 * i0 = ceil(x/h - w/2) mod n as in _kernels.py:19) plus its rank inside the
 * cell; counts accumulate in the plan's cell table.  Positions must already
 * lie in [0, L) (pif_wrap_points does that, nufft.py:105-113).
 * pif_bin_scatter: exclusive scan of the counts, then scatter src -> dst in
 * cell order; dst is what the *_sorted kernels read.  Resets the counts. */
int pif_wrap_points(pif_plan_t plan, double *x, double *y, double *z, int64_t M, void *stream);
int pif_bin_keys(pif_plan_t plan, const pif_soa_t *src, int32_t *key, int32_t *rank,
                 void *stream);
int pif_bin_scatter(pif_plan_t plan, const pif_soa_t *src, pif_soa_t *dst, const int32_t *key,
                    const int32_t *rank, int with_velocity, void *stream);

/* pif_bin_perm: exclusive scan of the counts, then perm[start[key[j]] + rank[j]] = j,
 * the cell-ordered view of a particle set that is NOT moved (12 B/particle
 * instead of the 120 B of pif_bin_scatter).  Resets the counts.  The hot PD
 * loop uses this: the gather+push kernel then reads through perm and writes
 * the particles out in cell order (pif_interp_push_perm). */
int pif_bin_perm(pif_plan_t plan, const int32_t *key, const int32_t *rank, int64_t M,
                 int32_t *perm, void *stream);
/* rank may be NULL: each particle then takes the next free slot of its cell
 * from a per-cell cursor (warp-aggregated atomics), so producers of keys (the
 * push kernels) only count and never wait on a returning atomic. */

/* ---- type-1 spreading: replaces _kernels.spread_r (_kernels.py:57-96) ------
 * Reads cell-sorted particles (dst of pif_bin_scatter).  strengths == NULL
 * means the uniform charge q (strategies.py:160-161); otherwise strengths is
 * indexed by particle id.  Overwrites the plan's fine grid. */
int pif_spread_sorted(pif_plan_t plan, const pif_soa_t *sorted, const double *strengths,
                      double q, void *stream);
/* Same, reading the particles through perm (pif_bin_perm) instead of in place. */
int pif_spread_perm(pif_plan_t plan, const pif_soa_t *parts, const int32_t *perm,
                    const double *strengths, double q, void *stream);

/* ---- uniform FFT + truncate/deconvolve: replaces nufft.py:140-145 ----------
 * D2Z of the plan's fine grid (cuFFT), then modes = F[m mod n] * d(mx)d(my)d(mz) / n^3
 * into `modes` (complex N^3, caller-owned, e.g. the allreduce buffer). */
int pif_grid_to_modes(pif_plan_t plan, double *modes, void *stream);

/* ---- field solve: replaces pif.finish_deposit (pif.py:95-105),
 * spectral.poisson_efield (spectral.py:63-82), field_energy (spectral.py:85-91),
 * the Hermitian guard (pif.py:128-133, spectral.py:94-101) and
 * nufft._padded_spectrum + 3x ifftn (nufft.py:148-156, 182-185).
 * Input: the allreduced raw type-1 modes.  Output: rho (optional, complex N^3),
 * the plan's interleaved field grid, and scalars[0..2] (device) =
 * {field energy W, max Hermitian mismatch over Ex,Ey,Ez relative to each scale,
 *  unused}.  shape is PIF_SHAPE_*. */
int pif_solve_fields(pif_plan_t plan, const double *raw_modes, int shape, double *rho_out,
                     double *scalars, void *stream);
/* Same, from caller-supplied E modes (gather_efield API, pif.py:115-137):
 * guard value into scalars[1], no energy. */
int pif_fields_from_modes(pif_plan_t plan, const double *ex, const double *ey, const double *ez,
                          int shape, double *scalars, void *stream);
/* Field energy only (spectral.field_energy of poisson_efield(rho)) for a
 * finished rho: scalars[0] = W. */
int pif_field_energy(pif_plan_t plan, const double *rho, double *scalars, void *stream);
/* Poisson solve only (spectral.poisson_efield): rho -> Ex, Ey, Ez (complex N^3). */
int pif_poisson(pif_plan_t plan, const double *rho, double *ex, double *ey, double *ez,
                void *stream);

/* ---- type-2 gather fused with the Boris push: replaces _kernels.interp_r3
 * (_kernels.py:125-183) + pif.boris_push (pif.py:140-158) +
 * pif.external_field_eval (pif.py:43-57) + particles.wrap_positions.
 * Updates the sorted particles in place, emits the next cell key and rank
 * (pif_bin_keys semantics) and writes diag[0..5] = {sum v.v, sum vx, sum vy,
 * sum vz, sum phi_ext(x), 0} over the updated particles (device, overwritten;
 * the caller scales by m/2, m, q as pif.py:60-68, 240-245 do).
 * half = 0.5*dt*qm and the Boris constants (tq = half*B, sq = 2 tq/(1+tq.tq))
 * are computed by the caller exactly as pif.py:146-153 does; has_b == 0 skips
 * the rotation. */
int pif_interp_push(pif_plan_t plan, pif_soa_t *sorted, double half, double dt,
                    const double tq[3], const double sq[3], int has_b, int e_kind,
                    int32_t *key, int32_t *rank, double *diag, void *stream);
/* Same, reading src through perm and writing the updated particles (and ids)
 * to dst in that order (dst must not alias src); key/rank refer to dst.  rank
 * may be NULL (then only the cell counts are incremented; pif_bin_perm with a
 * NULL rank assigns the slots). */
int pif_interp_push_perm(pif_plan_t plan, const pif_soa_t *src, const int32_t *perm,
                         pif_soa_t *dst, double half, double dt, const double tq[3],
                         const double sq[3], int has_b, int e_kind, int32_t *key, int32_t *rank,
                         double *diag, void *stream);
/* The same step in two parts, for host-streamed stepping (the gather only
 * needs positions; the push needs the velocities, which may still be on the
 * way from the host):
 * pif_interp_split: gather E (interp_r3, _kernels.py:125-183) at every
 *   particle of src (read through perm) into a plan-owned (M,3) array, row
 *   id - id0 (src holds ids id0 .. id0+M-1);
 * pif_push_ids: Boris push (pif.py:140-158; E_ext pif.py:43-57; wrap
 *   particles.py:65-70) of rows [row0, row0+rows) of device (M,3) x, v in id
 *   order (the host ParticleEnsemble layout) in place with those E rows.
 *   Chunks may be pushed in any number of calls in increasing row order; the
 *   call that reaches row M writes diag ({sum v.v, sum vx, sum vy, sum vz,
 *   sum phi_ext, 0}, like pif_interp_push_perm).  No cell keys are written:
 *   the caller rebins from the pushed rows (pif_load_aos).
 * DMMA kernels only (w <= 8): pif_split_supported returns 1 / 0. */
int pif_interp_split(pif_plan_t plan, const pif_soa_t *src, const int32_t *perm, int64_t id0,
                     void *stream);
int pif_push_ids(pif_plan_t plan, double *x, double *v, int64_t M, int64_t row0, int64_t rows,
                 double half, double dt, const double tq[3], const double sq[3], int has_b,
                 int e_kind, double *diag, void *stream);
int pif_split_supported(pif_plan_t plan);
/* Sparse sets (a few particles per stencil cell): the DMMA spread can walk C
 * x-adjacent columns as one super-column (fewer plane flushes and REDs, fuller
 * k-steps, (C+7)/8 of the DMMAs per k-step; spread_r, _kernels.py:57-96, same
 * sums).  c = -1: by density (default; env PIF_SPREAD_MERGE overrides at plan
 * creation), 0 or 1: never, 2 or 4: always (w = 6..8, n >= 32, not in the
 * deterministic mode).  pif_spread_merge_used: the C of the last spread. */
int pif_set_spread_merge(pif_plan_t plan, int c);
int pif_spread_merge_used(pif_plan_t plan);
/* Gather only (gather_efield): E at the sorted particles written to
 * E_out[3*id + d] (AoS, particle id order). */
int pif_interp_sorted(pif_plan_t plan, const pif_soa_t *sorted, double *E_out, void *stream);
/* Same, reading the particles through perm (pif_bin_perm). */
int pif_interp_perm(pif_plan_t plan, const pif_soa_t *parts, const int32_t *perm, double *E_out,
                    void *stream);
/* Particles back to id order (ParticleEnsemble layout, particles.py:10-62):
 * x_out/v_out are (M,3) AoS, row id - id0 (ids of the set must be
 * id0 .. id0+M-1); v_out may be NULL. */
int pif_soa_to_aos(pif_plan_t plan, const pif_soa_t *parts, int64_t id0, double *x_out,
                   double *v_out, void *stream);
/* Complex type 1 / type 2 on the binned fast kernels (cell-sorted points from
 * pif_bin_scatter, strengths / outputs indexed by point id):
 * pif_type1_complex_sorted: modes = type1 of s_re + i s_im (two production
 * spreads, one C2C FFT; replaces spread_c, _kernels.py:31-54, nufft.py:132-145).
 * pif_type2_complex_sorted: E_out[3 id + {0, 1}] = (Re, Im) of the type-2 value
 * at point id (C2C inverse FFT, production gather; replaces interp_c,
 * _kernels.py:99-122, nufft.py:159-172).  Both overwrite the plan's grids. */
int pif_type1_complex_sorted(pif_plan_t plan, const pif_soa_t *sorted, const double *s_re,
                             const double *s_im, double *modes, void *stream);
int pif_type2_complex_sorted(pif_plan_t plan, const double *modes, const pif_soa_t *sorted,
                             double *E_out, void *stream);

/* Spread -> gather weight cache.  The gather of a PD step runs at the positions
 * the previous step's deposit spread (strategies.py:290-300: solve(x_n+1), then
 * gather(x_n+1)), in the same perm order and chunking.  When enabled, the
 * w <= 8 spread also stores its 3w window weights per particle (192 B each at
 * w = 8, allocated on first use; if that fails the plan runs without) and the
 * next gather over the same particle view and perm loads them instead of
 * recomputing them.  Anything that moves or re-bins the particles invalidates
 * the cache.  Default off; the Python engine enables it when HBM allows. */
int pif_set_weight_cache(pif_plan_t plan, int enable);

/* Host-layout (ParticleEnsemble, particles.py:10-62) streaming, used when the
 * caller keeps the particles in host memory between steps (pif_step,
 * pif.py:178-190):
 * pif_load_aos: (M,3) AoS x, v rows of ids id0 .. id0+M-1 (device copies of the
 * host arrays) -> wrapped SoA store dst (dst->count = M) with ids, cell keys and
 * ranks in one pass (= upload + pif_wrap_points + pif_bin_keys); follow with
 * pif_bin_perm.
 * pif_set_id_order_output: while x_out/v_out are set, every pif_interp_push*
 * launch also writes each pushed particle's x, v to row id - id0 of these (M,3)
 * arrays (a fused pif_soa_to_aos); NULL, NULL clears.  Plan state: set it only
 * around the pushes that should mirror. */
int pif_load_aos(pif_plan_t plan, const double *x, const double *v, int64_t id0, pif_soa_t *dst,
                 int32_t *key, int32_t *rank, void *stream);
/* pif_load_aos with v == NULL loads positions (and keys) only, so binning and
 * the deposit can start while the velocities are still on the way;
 * pif_load_aos_velocities then fills dst's velocities from the (M,3) rows
 * (same set, before any push): slot i takes row dst->id[i] - id0, so it also
 * works after pif_permute.  rank may be NULL (pif_bin_perm with NULL rank
 * assigns the in-cell slots). */
int pif_load_aos_velocities(pif_plan_t plan, const double *v, pif_soa_t *dst, void *stream);
/* dst[i] = src[perm[i]] for the fields `what` selects (PIF_PERMUTE_*), i <
 * src->count; PIF_PERMUTE_RESET afterwards sets perm to the identity.  No
 * reference counterpart (its particles are never reordered): the data
 * movement step of a host-streamed step (PifEngine.run_host), where the set
 * arrives in id order (spatially random) and is put into the cell order of
 * pif_bin_perm once, so the spread and the gather read it coalesced.  dst
 * must not alias src. */
int pif_permute(pif_plan_t plan, const pif_soa_t *src, int32_t *perm, pif_soa_t *dst, int what,
                void *stream);
int pif_set_id_order_output(pif_plan_t plan, double *x_out, double *v_out, int64_t id0);
/* Diagnostic sums of a particle set (Recorder.record, strategies.py:96-106). */
int pif_particle_diag(pif_plan_t plan, const pif_soa_t *p, int e_kind, double *diag,
                      void *stream);

/* ---- complex variants for the type1/type2 API (_kernels.py:31-54, 99-122) --
 * pts are AoS (M,3) device doubles already wrapped into [0,L). */
int pif_type1_complex(pif_plan_t plan, const double *pts, const double *vals, int64_t M,
                      double *modes, void *stream);
int pif_type2_complex(pif_plan_t plan, const double *modes, const double *pts, int64_t M,
                      double *out, void *stream);

/* ---- measurement ------------------------------------------------------------
 * FP64 DFMA throughput probe (the roofline denominator; MEASURED_PEAKS.json has
 * no FP64 figure).  Launches blocks x threads threads, each running `iters`
 * iterations of 8 independent FMAs; *flops_out = flops issued. */
int pif_probe_fp64(double *scratch, int blocks, int threads, int iters, void *stream,
                   double *flops_out);
/* ---- deterministic mode: the reference is bit-reproducible by construction
 * (serial numba kernels _kernels.py:1-5, fixed-order tree sums comm.py:329-339;
 * its tests test_strategies.py:57-62, 405-409 compare runs with array_equal).
 * When enabled, binning is a stable sort of the cell keys (particles of a cell
 * keep their buffer order instead of atomic arrival order) and the spread
 * writes each work item's planes to its own buffer slice, summed per grid point
 * in a fixed order (det_reduce_kernel) instead of REDG.ADD.F64.  The caller
 * takes the step's diagnostic sums from pif_particle_diag (fixed-order) after
 * the push.  Same results to rounding as the default mode, identical bits run
 * to run.  Only for the DMMA kernels (w <= 8); PIF_ERR_VALUE otherwise. */
int pif_set_deterministic(pif_plan_t plan, int enable);
int pif_is_deterministic(pif_plan_t plan);

/* 1 if the gather+push counts next-cell keys per run of equal keys in dense
 * segments (sets with heavy cells, e.g. a Penning cloud at 2^28 on one GPU),
 * 0 for per-particle counts.  Decided at the first binning after each
 * pif_bin_keys / pif_load_aos from the most particles any z-segment holds
 * (>= 12 work items); PIF_PUSH_AGG=0/1 in the environment forces it.  Same
 * counts either way: a performance switch only. */
int pif_push_aggregated(pif_plan_t plan);

/* ---- in-process communicators: replaces comm.allreduce_sum's fixed-order
 * tree over rank threads (comm.py:329-339, 391-408) for spawn_spmd's thread
 * ranks (comm.py:483-528), one GPU per rank.
 * pif_comm_init_all: ncclCommInitAll over `devices` (distinct; one rank per
 * device), comms_out[r] = rank r's communicator.  pif_allreduce_f64: in-place
 * sum of `count` doubles on `stream` (device memory of the comm's device);
 * every rank must call it, each from its own thread.  libnccl.so.2 is opened at
 * run time (the instance torch loaded, if any); pif_nccl_version reports it. */
typedef struct pif_comm_s *pif_comm_t;
int pif_nccl_version(int *version);
int pif_comm_init_all(int ndev, const int *devices, pif_comm_t *comms_out);
int pif_allreduce_f64(pif_comm_t comm, double *buf, int64_t count, void *stream);
int pif_comm_destroy(pif_comm_t comm);

/* cuFFT stage timing (the north star's "cuFFT call timed separately";
 * the reference times its fftn/ifftn inside Scatter/Gather, strategies.py:158-170).
 * pif_fft_timing(plan, slots): record CUDA events around each of the next
 * `slots` D2Z execs (pif_grid_to_modes) and Z2D execs (pif_solve_fields /
 * pif_fields_from_modes, incl. the interleave when the strided C2R is absent);
 * 0 disables.  Never records inside a stream capture.
 * pif_fft_times: waits for the recorded events, returns the summed milliseconds
 * and counts since the last call, and restarts the rings. */
int pif_fft_timing(pif_plan_t plan, int slots);
int pif_fft_times(pif_plan_t plan, double *d2z_ms, double *z2d_ms, int *n_d2z, int *n_z2d);
/* ---- device samplers (reference bench.py:67-122) -----
 * One numpy Philox4x64-10 stream per (seed, attribute): counter[4] / key[2] as
 * numpy's Philox(SeedSequence((seed, attr))).state holds them; uint64 number j
 * of the stream is drawn for global index j.  Output element i goes to
 * out[i * stride] (stride 3 writes one column of an (M, 3) array).  *status is
 * OR-ed with 1 (CDF inversion failed) / 2 (rejection budget exhausted).
 *
 * Landau positions of ids [lo, lo + count): Newton inversion of
 * (x + (alpha/k) sin kx)/L = u_id with bisection rescue, then wrapped
 * (replaces _invert_landau_cdf + wrap_positions, bench.py:80-110,151-154). */
int pif_sample_landau_axis(const uint64_t *counter, const uint64_t *key, int64_t lo,
                           int64_t count, double alpha, double k, double L, double *out,
                           int64_t stride, int *status, void *stream);
/* Normals of ids [lo, lo + count) out of n_total: budget == 0 gives
 * _standard_normal (Box-Muller of rows 0 / 1 of a (2, n_total) draw,
 * bench.py:71-77); budget > 0 gives _rejection_normal_in_box, the first of
 * mean + std * normal over rows r / budget + r (r < budget) inside [0, L)
 * (bench.py:113-122). */
int pif_sample_normal(const uint64_t *counter, const uint64_t *key, int64_t n_total, int64_t lo,
                      int64_t count, double mean, double std_dev, int budget, double L,
                      double *out, int64_t stride, int *status, void *stream);
/* Profiling builds only (-DPIF_PHASE_TIMING): per-phase SM cycles of the
 * gather+push kernel summed over warps since the last call, out[0..4] =
 * {weights, DMMA gather, push, chunks, particles}; PIF_ERR_STATE otherwise. */
int pif_debug_phase_cycles(unsigned long long *out);

#ifdef __cplusplus
}
#endif
#endif /* PIF_B200_H */
