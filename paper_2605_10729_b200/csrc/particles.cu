// Particle-side kernels of the PD-PIF step on sm_100a:
//   binning (ES-stencil cell keys, cell-order permutation, work items),
//   type-1 spreading (replaces _kernels.spread_r, _kernels.py:57-96),
//   type-2 gather fused with the Boris push (replaces _kernels.interp_r3,
//   _kernels.py:125-183, and pif.boris_push, pif.py:140-158),
//   diagnostics sums (strategies.py:96-106), FMA "ring" kernels for wide
//   windows (w = 9..14), one-thread-per-particle kernels for the rest, the
//   complex-strength variants and the host-layout (AoS) load / id-order output.
//
// Fast kernels (w <= 8): particles are binned by their ES-stencil start cell
// (i0x, i0y, i0z), so every particle of a cell shares one w^3 footprint.  One
// warp owns a work item = a z-segment of one (i0x, i0y) column of cells and
// keeps the 8 x 8 x 8 footprint block in DMMA (fp64 mma.sync m8n8k4) fragments:
// spreading accumulates it, gathering contracts it; the z-slot of a plane is
// its index mod 8, so stepping to the next cell in z flushes (spread) or loads
// (gather) exactly one plane.  Window weights come from es_fast.cuh.
#include <cub/cub.cuh>

#include <cstring>

#include "pif_internal.cuh"
#include "es_fast.cuh"

namespace pif {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int cell_index_of(double c, int w, int n) {
    return pmod((int)stencil_start(c, w), n);
}

__device__ __forceinline__ int cell_key(double x, double y, double z, double h, double rh, int w,
                                        int n) {
    int kx = cell_index_of(axis_coord(x, h, rh), w, n);
    int ky = cell_index_of(axis_coord(y, h, rh), w, n);
    int kz = cell_index_of(axis_coord(z, h, rh), w, n);
    return (kx * n + ky) * n + kz;
}

// ----------------------------------------------------------------------------
// binning
// ----------------------------------------------------------------------------

__global__ void wrap_kernel(double *x, double *y, double *z, int64_t M, double L) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        x[i] = wrap_coord(x[i], L);
        y[i] = wrap_coord(y[i], L);
        z[i] = wrap_coord(z[i], L);
    }
}

__global__ void bin_keys_kernel(const double *__restrict__ x, const double *__restrict__ y,
                                const double *__restrict__ z, int64_t M, double h, int w, int n,
                                int32_t *__restrict__ key, int32_t *__restrict__ rank,
                                int32_t *__restrict__ count) {
    const double rh = __drcp_rn(h);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        int k = cell_key(x[i], y[i], z[i], h, rh, w, n);
        key[i] = k;
        rank[i] = atomicAdd(&count[k], 1);
    }
}

__global__ void bin_scatter_kernel(pif_soa_t src, pif_soa_t dst, const int32_t *__restrict__ key,
                                   const int32_t *__restrict__ rank,
                                   const int32_t *__restrict__ start, int vel) {
    const int64_t M = src.count;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t d = (int64_t)start[key[i]] + rank[i];
        PIF_CHECK(d >= 0 && d < M);
        dst.x[d] = src.x[i];
        dst.y[d] = src.y[i];
        dst.z[d] = src.z[i];
        if (vel) {
            dst.vx[d] = src.vx[i];
            dst.vy[d] = src.vy[i];
            dst.vz[d] = src.vz[i];
        }
        dst.id[d] = src.id[i];
    }
}

// particles back to id order as AoS (M,3) x and v: out[(id - id0)] = particle
__global__ void soa_to_aos_by_id_kernel(pif_soa_t P, int64_t id0, double *__restrict__ ox,
                                        double *__restrict__ ov) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P.count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = 3 * (P.id[i] - id0);
        PIF_CHECK(o >= 0 && o < 3 * P.count);
        ox[o] = P.x[i];
        ox[o + 1] = P.y[i];
        ox[o + 2] = P.z[i];
        if (ov) {
            ov[o] = P.vx[i];
            ov[o + 1] = P.vy[i];
            ov[o + 2] = P.vz[i];
        }
    }
}

// Host-layout upload in one pass (replaces upload + pif_wrap_points +
// pif_bin_keys for ParticleEnsemble-shaped input): AoS (M,3) x, v rows in id
// order -> wrapped SoA store, ids id0 + i, cell keys and ranks.
__global__ void load_aos_kernel(const double *__restrict__ xa, const double *__restrict__ va,
                                int64_t id0, int64_t M, pif_soa_t dst, double L, double h,
                                int w, int n, int32_t *__restrict__ key,
                                int32_t *__restrict__ rank, int32_t *__restrict__ count) {
    const double rh = __drcp_rn(h);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = wrap_coord(xa[3 * i], L), y = wrap_coord(xa[3 * i + 1], L),
                     z = wrap_coord(xa[3 * i + 2], L);
        dst.x[i] = x;
        dst.y[i] = y;
        dst.z[i] = z;
        if (va) {
            dst.vx[i] = va[3 * i];
            dst.vy[i] = va[3 * i + 1];
            dst.vz[i] = va[3 * i + 2];
        }
        dst.id[i] = id0 + i;
        const int k = cell_key(x, y, z, h, rh, w, n);
        key[i] = k;
        if (rank) rank[i] = atomicAdd(&count[k], 1);
        else atomicAdd(&count[k], 1);
    }
}

// the velocities of a set loaded with load_aos_kernel(va = NULL): AoS rows of
// ids id0 .. id0+M-1 -> SoA slots i (the load left particle i in slot i)
// slot i takes the row of its own id (i itself right after the load; any
// slot after pif_permute)
__global__ void load_vel_kernel(const double *__restrict__ va, int64_t id0, int64_t M,
                                pif_soa_t dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = dst.id[i] - id0;
        PIF_CHECK(r >= 0 && r < M);
        dst.vx[i] = va[3 * r];
        dst.vy[i] = va[3 * r + 1];
        dst.vz[i] = va[3 * r + 2];
    }
}

// perm[start[key[j]] + rank[j]] = j: the cell-ordered view of a particle set
__global__ void bin_perm_kernel(const int32_t *__restrict__ key, const int32_t *__restrict__ rank,
                                const int32_t *__restrict__ start, int64_t M,
                                int32_t *__restrict__ perm) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M;
         j += (int64_t)gridDim.x * blockDim.x) {
        PIF_CHECK(start[key[j]] + rank[j] >= 0 && start[key[j]] + rank[j] < M);
        perm[start[key[j]] + rank[j]] = (int32_t)j;
    }
}

// rank-free variant: the in-cell slot comes from a cursor per cell (the count
// table, zeroed after the scan); lanes of a warp holding the same key take
// consecutive slots with one atomic (consecutive particles mostly share a
// cell: they were written in cell order by the previous push).  Each warp
// takes kPermUnroll x 32 consecutive particles per pass so that many cursor
// atomics are in flight at once (the pass is bound by their round trips).
constexpr int kPermUnroll = 4;
__global__ void bin_perm_cursor_kernel(const int32_t *__restrict__ key, int32_t *__restrict__ cursor,
                                       const int32_t *__restrict__ start, int64_t M,
                                       int32_t *__restrict__ perm) {
    const int lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    const int64_t sweep = (int64_t)gridDim.x * blockDim.x * kPermUnroll;
    for (int64_t b0 = ((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * kPermUnroll;
         b0 < M; b0 += sweep) {
        int k[kPermUnroll], base[kPermUnroll];
        unsigned peers[kPermUnroll];
#pragma unroll
        for (int u = 0; u < kPermUnroll; ++u) {
            const int64_t j = b0 + u * 32 + lane;
            k[u] = j < M ? key[j] : -1;
        }
#pragma unroll
        for (int u = 0; u < kPermUnroll; ++u) peers[u] = __match_any_sync(0xffffffffu, k[u]);
#pragma unroll
        for (int u = 0; u < kPermUnroll; ++u) {
            base[u] = 0;
            if (k[u] >= 0 && lane == __ffs(peers[u]) - 1)
                base[u] = atomicAdd(&cursor[k[u]], __popc(peers[u]));
        }
#pragma unroll
        for (int u = 0; u < kPermUnroll; ++u) {
            base[u] = __shfl_sync(peers[u], base[u], __ffs(peers[u]) - 1);
            if (k[u] >= 0) {
                const int64_t j = b0 + u * 32 + lane;
                const int slot = start[k[u]] + base[u] + __popc(peers[u] & below);
                PIF_CHECK(slot >= 0 && slot < M);
                perm[slot] = (int32_t)j;
            }
        }
    }
}

// work items: parts of <= kItemParticles particles of each non-empty z-segment
__global__ void seg_parts_kernel(const int32_t *__restrict__ cell_start, int n, int seg, int nseg,
                                 int nsegs, int *__restrict__ parts) {
    for (int sidx = blockIdx.x * blockDim.x + threadIdx.x; sidx <= nsegs;
         sidx += gridDim.x * blockDim.x) {
        if (sidx == nsegs) {
            parts[sidx] = 0;
            continue;
        }
        const int col = sidx / nseg, sg = sidx - col * nseg;
        const int base = col * n, k0 = sg * seg, k1 = min(k0 + seg, n);
        const int c = cell_start[base + k1] - cell_start[base + k0];
        parts[sidx] = (c + kItemParticles - 1) / kItemParticles;
    }
}

__global__ void seg_items_kernel(const int *__restrict__ parts, const int *__restrict__ off,
                                 int nsegs, int2 *__restrict__ items) {
    for (int sidx = blockIdx.x * blockDim.x + threadIdx.x; sidx < nsegs;
         sidx += gridDim.x * blockDim.x) {
        const int o = off[sidx];
        for (int j = 0; j < parts[sidx]; ++j) items[o + j] = make_int2(sidx, j);
    }
}

__global__ void publish_int_kernel(const int *__restrict__ src, volatile int *dst) { *dst = *src; }

__global__ void max_parts_kernel(const int *__restrict__ parts, int nsegs, int *out) {
    int m = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nsegs; i += gridDim.x * blockDim.x)
        m = max(m, parts[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(out, m);
}

// ----------------------------------------------------------------------------
// DMMA building blocks
// ----------------------------------------------------------------------------

// D(8x8) += A(8x4) B(4x8), fp64 tensor-core MMA (SASS DMMA.8x8x4).  Fragments:
// A[row = lane>>2][col = lane&3], B[row = lane&3][col = lane>>2],
// D[row = lane>>2][col = 2*(lane&3) + {0,1}] (checked by tools/dmma_probe.cu).
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Per-warp staging of one chunk of up to kChunk consecutive (cell-sorted)
// particles of a work item; chunks run across cell boundaries.  Lane j owns
// particle j of the chunk: it loads it, computes its 3 x w window weights and
// (gather) pushes it.  Weights are padded to 8 with zeros (entries a >= w are
// never written) and laid out so the DMMA fragment loads are conflict-free or
// 2-way (row strides 33 and 9 doubles).
constexpr int kChunk = 32;
// accumulator chains per gather sub-batch: 3 (one per component; default,
// gather 17.38 -> 17.17 ms at 2^27) or 6 (per half-slot and component, merged
// by 6 DADDs per sub-batch)
#ifndef PIF_GATHER_CHAINS
#define PIF_GATHER_CHAINS 3
#endif

// Layouts chosen so the hot shared-memory accesses are bank-conflict free
// (64-bit words, 16 per half-warp phase): wz is [c][p] with row stride 36
// (= 4 mod 16): the DMMA loops read (c = slot of lane column, p = row lane)
// and the weight phase writes (p = lane) without conflicts.
constexpr int kWzStride = kChunk + 4;
struct WarpChunk {
    double wx[8][kChunk + 1];   // [a][p]  x weights (spreading: times the strength)
    double wy[kChunk][9];       // [p][b]
    double wz[8][kWzStride];    // [c][p]
    double E[3][kChunk];        // gathered field (gather+push)
};

// gather: per-particle partial sums over (a, c) for each y offset b, reduced
// against wy in the push phase instead of a shuffle tree per sub-batch;
// [b][p] with row stride 34 (= 2 mod 16): the sub-batch stores (b = 2 c4 + j,
// p = row lane) and the per-particle reads (p = lane) are conflict free
constexpr int kDStride = kChunk + 2;
struct GatherPartials {
    double D[3][8][kDStride];   // [component][b][p]
};

__device__ __forceinline__ void chunk_zero(WarpChunk &st, int lane) {
    double *w = &st.wx[0][0];
    const int nw = 8 * (kChunk + 1) + 2 * kChunk * 9;
    for (int i = lane; i < nw; i += 32) w[i] = 0.0;
    __syncwarp();
}

// Window weights of this lane's particle (lane < cnt): c = x/h and the w
// weights per axis (_kernels.py:11-28; interior ones by polynomial,
// es_fast.cuh), x row scaled by the strength s.
// XYZ: advance the three axes' polynomial chains together (more ILP, more
// registers) — used by the low-occupancy gather kernel; the spread kernel runs
// enough warps to hide the per-axis chains and keeps its registers low.
template <int W, bool XYZ>
__device__ __forceinline__ void chunk_weights(WarpChunk &st, const double *tab, const EsPoly &P,
                                              int lane, int cnt, double x, double y, double z,
                                              double s, bool scale, double h, double rh,
                                              double beta, double *wc = nullptr,
                                              int64_t wstride = 0, int64_t wpos = 0) {
    if (lane < cnt) {
        if (XYZ) {
            const double c[3] = {axis_coord(x, h, rh), axis_coord(y, h, rh), axis_coord(z, h, rh)};
            double wt[3][W];
            es_xyz_weights<W>(c, beta, P, tab, wt);
#pragma unroll
            for (int a = 0; a < W; ++a) {
                st.wx[a][lane] = scale ? __dmul_rn(s, wt[0][a]) : wt[0][a];
                st.wy[lane][a] = wt[1][a];
                st.wz[a][lane] = wt[2][a];
                if (wc) {
                    wc[a * wstride + wpos] = wt[0][a];
                    wc[(8 + a) * wstride + wpos] = wt[1][a];
                    wc[(16 + a) * wstride + wpos] = wt[2][a];
                }
            }
        } else {
            // wc: also keep the (unscaled) weights for the next gather at these
            // positions, row 8 * axis + a of a [24][wstride] array, column wpos
            double wt[W];
            es_axis_weights<W>(axis_coord(x, h, rh), beta, P, tab, wt);
#pragma unroll
            for (int a = 0; a < W; ++a) {
                st.wx[a][lane] = scale ? __dmul_rn(s, wt[a]) : wt[a];
                if (wc) wc[a * wstride + wpos] = wt[a];
            }
            es_axis_weights<W>(axis_coord(y, h, rh), beta, P, tab, wt);
#pragma unroll
            for (int a = 0; a < W; ++a) {
                st.wy[lane][a] = wt[a];
                if (wc) wc[(8 + a) * wstride + wpos] = wt[a];
            }
            es_axis_weights<W>(axis_coord(z, h, rh), beta, P, tab, wt);
#pragma unroll
            for (int a = 0; a < W; ++a) {
                st.wz[a][lane] = wt[a];
                if (wc) wc[(16 + a) * wstride + wpos] = wt[a];
            }
        }
    }
    __syncwarp();
}

// The gather's window weights from the cache the preceding spread wrote
// (same particles, same perm, same chunking): lane l copies its particle's
// 3 x w weights into the stage with cp.async (one commit group per chunk).
template <int W>
__device__ __forceinline__ void chunk_weights_async(WarpChunk &st, const double *wc,
                                                    int64_t wstride, int64_t wpos, int lane,
                                                    int cnt) {
    if (lane < cnt) {
#pragma unroll
        for (int a = 0; a < W; ++a) {
            const unsigned dx = (unsigned)__cvta_generic_to_shared(&st.wx[a][lane]);
            const unsigned dy = (unsigned)__cvta_generic_to_shared(&st.wy[lane][a]);
            const unsigned dz = (unsigned)__cvta_generic_to_shared(&st.wz[a][lane]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dx),
                         "l"(wc + a * wstride + wpos));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dy),
                         "l"(wc + (8 + a) * wstride + wpos));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dz),
                         "l"(wc + (16 + a) * wstride + wpos));
        }
    }
    asm volatile("cp.async.commit_group;");
}

// ----------------------------------------------------------------------------
// spreading (w <= 8) on the fp64 tensor cores
//
// Warp = one work item (z-segment of an (i0x, i0y) column of stencil cells).
// For each stencil-x offset a, the 8 x 8 block G_a[b][z-slot] of the current
// cell's footprint is one DMMA accumulator: G_a += A_a B over k-steps of 4
// particles of that cell, with
//   A_a[b][p] = (s_p wx_p[a]) wy_p[b]      (8 rows b  x 4 particles)
//   B[p][s]   = wz_p[(s - k) mod 8]        (4 particles x 8 z-slots)
// z-slot s holds plane z == s (mod 8): leaving cell k completes plane k
// (slot k&7), which is flushed with REDG.ADD.F64 and reused for plane k+8.
// ----------------------------------------------------------------------------

// Deterministic mode (pif_set_deterministic): instead of REDG into the grid,
// plane k of the item goes to its own slice of the plane buffer,
// dbuf[((item * 64 + a * 8 + b) * dstride) + (k - k0)], and det_reduce_kernel
// sums the slices of every grid point in a fixed order.
struct DetOut {
    double *buf = nullptr;   // null: atomics into the grid
    int64_t stride = 0;      // planes per (item, a, b) row: seg + 7
};

template <int W, bool DET>
__device__ __forceinline__ void spread_flush_plane(double (&acc)[8][2], int k, int c4, int ix,
                                                   int64_t yrow, int n, double *grid,
                                                   const DetOut &det, int64_t drow, int k0) {
    const int s = k & 7;
    if (c4 == (s >> 1)) {
        const int j = s & 1;
        if (DET) {
            // drow = (item * 64 + r) * stride: this lane's b = r rows, a-major
#pragma unroll
            for (int a = 0; a < W; ++a)
                det.buf[drow + (int64_t)a * 8 * det.stride + (k - k0)] = j ? acc[a][1] : acc[a][0];
        } else {
            const int z = k;   // cells of an item never wrap: k < n
            const int64_t nn = (int64_t)n * n;
            int64_t off = ((int64_t)ix * n + yrow) * n + z;
#pragma unroll
            for (int a = 0; a < W; ++a) {
                const double v = j ? acc[a][1] : acc[a][0];
                PIF_CHECK(off == ((int64_t)((ix + a) % n) * n + yrow) * n + z);
                if (v != 0.0) atomicAdd(grid + off, v);
                off += (ix + a + 1 == n) ? nn - (int64_t)n * nn : nn;   // x wraps once (w <= n)
            }
        }
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            if (j) acc[a][1] = 0.0;
            else acc[a][0] = 0.0;
        }
    }
}

// k-steps unrolled in the spread's DMMA loop (4: 9.24 -> 9.16 ms at 2^27
// against 2, profiles/round2/spread_knobs_ab.txt)
#ifndef PIF_SPREAD_UNROLL
#define PIF_SPREAD_UNROLL 4
#endif
constexpr int kSpreadUnroll = PIF_SPREAD_UNROLL;
#ifndef PIF_SPREAD_MINB
#define PIF_SPREAD_MINB 4
#endif
// 1: the spread evaluates the three axes' weight polynomials interleaved (more
// ILP, more registers); A/B knob, see DESIGN.md §4
#ifndef PIF_SPREAD_XYZ
#define PIF_SPREAD_XYZ 1
#endif

template <int W, bool DET>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, PIF_SPREAD_MINB)
spread_mma_kernel(const double *__restrict__ px, const double *__restrict__ py,
                  const double *__restrict__ pz, const int64_t *__restrict__ pid,
                  const int32_t *__restrict__ perm, const double *__restrict__ strengths, double q,
                  const int32_t *__restrict__ cell_start, double *__restrict__ grid, int n,
                  int seg, int nseg, double h, double beta, const EsPoly poly, unsigned int *work,
                  const int2 *__restrict__ items, const int *__restrict__ n_items,
                  double *__restrict__ wc, int64_t wstride, const DetOut det) {
    const int nitems = *n_items;
    const double rh = __drcp_rn(h);
    __shared__ WarpChunk stage[kWarpsPerBlock];
    __shared__ double tab[32];
    // the item's cell boundaries, loaded once per item (a per-cell global load
    // shares a scoreboard with the chunk prefetch and stalls on it)
    __shared__ int seg_cells[kWarpsPerBlock][kMaxSeg + 1];
    if (threadIdx.x < 32) tab[threadIdx.x] = kExp2Table[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    WarpChunk &st = stage[threadIdx.x >> 5];
    int *cbt = seg_cells[threadIdx.x >> 5];
    chunk_zero(st, lane);
    const int r = lane >> 2, c4 = lane & 3;

    for (;;) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(work, 1u);
        item = __shfl_sync(kFull, item, 0);
        if (item >= nitems) break;
        const int2 it = items[item];
        const int col = it.x / nseg, sg = it.x - col * nseg;
        const int ix = col / n, iy = col - ix * n;
        const int k0 = sg * seg, k1 = min(k0 + seg, n);
        const int base = col * n;
        __syncwarp();   // the previous item is done with the cell table
        for (int c = lane; c <= k1 - k0; c += 32) cbt[c] = cell_start[base + k0 + c];
        __syncwarp();
        const int pbeg = cbt[0] + it.y * kItemParticles;
        const int pend = min(pbeg + kItemParticles, cbt[k1 - k0]);
        const int64_t yrow = (iy + r) % n;   // this lane's footprint row b = r
        const int64_t drow = DET ? ((int64_t)item * 64 + r) * det.stride : 0;

        double acc[8][2];
#pragma unroll
        for (int a = 0; a < 8; ++a) acc[a][0] = acc[a][1] = 0.0;
        int k = k0;
        int cell_end = cbt[1];
        while (cell_end <= pbeg) cell_end = cbt[(++k) - k0 + 1];   // first cell

        double nx = 0.0, ny = 0.0, nz = 0.0, ns = q;
        if (pbeg + lane < pend) {
            const int i = perm ? perm[pbeg + lane] : pbeg + lane;
            nx = px[i];
            ny = py[i];
            nz = pz[i];
            if (strengths) ns = strengths[pid[i]];
        }
        int npi = -1;   // perm entry one chunk ahead of the particle prefetch
        if (pbeg + kChunk + lane < pend) npi = perm ? perm[pbeg + kChunk + lane] : pbeg + kChunk + lane;
        for (int pos = pbeg; pos < pend; pos += kChunk) {
            const int cnt = min(kChunk, pend - pos);
            const double cx = nx, cy = ny, cz = nz, cs = ns;
            if (npi >= 0) {   // prefetch the next chunk
                const int i = npi;
                nx = px[i];
                ny = py[i];
                nz = pz[i];
                if (strengths) ns = strengths[pid[i]];
            }
            npi = -1;
            if (pos + 2 * kChunk + lane < pend)
                npi = perm ? perm[pos + 2 * kChunk + lane] : pos + 2 * kChunk + lane;
            chunk_weights<W, (bool)PIF_SPREAD_XYZ>(st, tab, poly, lane, cnt, cx, cy, cz, cs, true, h,
                                                  rh, beta, wc,
                                    wstride, pos + lane);
            int j = 0;
            while (j < cnt) {
                if (pos + j >= cell_end) {
                    spread_flush_plane<W, DET>(acc, k, c4, ix, yrow, n, grid, det, drow, k0);
                    ++k;
                    cell_end = cbt[k - k0 + 1];
                    continue;
                }
                const int jend = min(cnt, cell_end - pos);   // this cell's part of the chunk
                const int zs = (r - k) & 7;
                PIF_CHECK(jend <= kChunk && k >= k0 && k < k1);
                // full k-steps of 4 particles: no masking, unrolled so the next
                // step's shared-memory loads overlap this step's DMMAs
#pragma unroll kSpreadUnroll
                for (; j + 4 <= jend; j += 4) {
                    const int pj = j + c4;
                    const double wyb = st.wy[pj][r];
                    const double bz = st.wz[zs][pj];
#pragma unroll
                    for (int a = 0; a < 8; ++a)
                        dmma884(acc[a][0], acc[a][1], st.wx[a][pj] * wyb, bz);
                }
                if (j < jend) {   // ragged tail of the cell
                    const bool ok = c4 < jend - j;
                    const int pj = ok ? j + c4 : j;
                    const double wyb = ok ? st.wy[pj][r] : 0.0;
                    const double bz = st.wz[zs][pj];
#pragma unroll
                    for (int a = 0; a < 8; ++a)
                        dmma884(acc[a][0], acc[a][1], st.wx[a][pj] * wyb, bz);
                    j = jend;
                }
            }
            __syncwarp();
        }
        for (; k < k1; ++k) spread_flush_plane<W, DET>(acc, k, c4, ix, yrow, n, grid, det, drow, k0);
        // pending planes k1 .. k1+6
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int s = 2 * c4 + j;
            const int dz = (s - k1) & 7;   // dz == 7: plane k1 + 7, flushed with cell k1 - 1
            const int z = (k1 + dz) % n;
#pragma unroll
            for (int a = 0; a < W; ++a) {
                const double v = acc[a][j];
                if (DET) {
                    if (dz < 7)
                        det.buf[drow + (int64_t)a * 8 * det.stride + (k1 + dz - k0)] = v;
                } else if (v != 0.0) {
                    atomicAdd(grid + ((int64_t)((ix + a) % n) * n + yrow) * n + z, v);
                }
            }
        }
    }
}

// ----------------------------------------------------------------------------
// merged-column spreading for sparse sets
//
// At a few particles per stencil cell the column kernel above pays per cell
// step, not per particle: every cell step flushes a full 8 x 8 plane (so the
// grid receives 64 REDs per point and step whatever the density) and most
// k-steps of 4 particles are ragged.  Walking C x-adjacent columns as one
// super-column divides the cell steps and plane flushes by C, the REDs per
// grid point by 64 C / (8 (C + 7)) and the ragged steps by about C, for
// (C + 7) / 8 times the DMMAs per k-step: a particle of sub-column
// q = i0x - ix0 occupies union rows a' = q .. q + 7, i.e. its (strength-scaled)
// wx row is shifted by q and zero elsewhere, so one k-step mixes sub-columns.
// The super-columns have their own cell order,
//   mk = (((kx / C) n + ky) n + kz) C + kx mod C,
// in which a super-column's C cells of level kz are consecutive; cell_start2,
// perm2 and the work items are derived from the standard binning before each
// merged spread (merged_counts / scan / merged_perm / merged_seg_parts).
// ----------------------------------------------------------------------------

// count2[mk] = size of the standard cell behind merged cell mk; count2[n^3] = 0
__global__ void merged_counts_kernel(const int32_t *__restrict__ cell_start, int n, int C,
                                     int32_t *__restrict__ count2) {
    const int64_t n3 = (int64_t)n * n * n;
    for (int64_t mk = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; mk <= n3;
         mk += (int64_t)gridDim.x * blockDim.x) {
        if (mk == n3) {
            count2[mk] = 0;
            continue;
        }
        const int q = (int)(mk % C);
        int64_t t = mk / C;
        const int kz = (int)(t % n);
        t /= n;
        const int ky = (int)(t % n);
        const int mx = (int)(t / n);
        const int64_t k = ((int64_t)(mx * C + q) * n + ky) * n + kz;
        count2[mk] = cell_start[k + 1] - cell_start[k];
    }
}

// perm2: each merged cell mk copies the perm run of its standard cell k (same
// particles, same order): one lane per merged cell for the first 16 entries,
// the whole warp for the rest of heavy cells (a Penning core cell holds
// thousands), so perm2 is written nearly in order and only the two cell
// tables and perm are read
__global__ void merged_perm_kernel(const int32_t *__restrict__ perm,
                                   const int32_t *__restrict__ cell_start,
                                   const int32_t *__restrict__ cell_start2, int n, int C,
                                   int32_t *__restrict__ perm2) {
    constexpr int kLight = 16;
    const int64_t n3 = (int64_t)n * n * n;
    const int lane = threadIdx.x & 31;
    const int64_t sweep = (int64_t)gridDim.x * blockDim.x;
    for (int64_t w0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); w0 < n3;
         w0 += sweep) {   // warp-uniform trip count
        const int64_t mk = w0 + lane;
        int src = 0, cnt = 0, dst = 0;
        if (mk < n3) {
            const int q = (int)(mk % C);
            int64_t t = mk / C;
            const int kz = (int)(t % n);
            t /= n;
            const int ky = (int)(t % n);
            const int mx = (int)(t / n);
            const int64_t k = ((int64_t)(mx * C + q) * n + ky) * n + kz;
            src = cell_start[k];
            cnt = cell_start[k + 1] - src;
            dst = cell_start2[mk];
        }
        for (int i = 0; i < min(cnt, kLight); ++i) perm2[dst + i] = perm ? perm[src + i] : src + i;
        unsigned heavy = __ballot_sync(0xffffffffu, cnt > kLight);
        while (heavy) {
            const int h = __ffs(heavy) - 1;
            heavy &= heavy - 1u;
            const int hs = __shfl_sync(0xffffffffu, src, h), hc = __shfl_sync(0xffffffffu, cnt, h),
                      hd = __shfl_sync(0xffffffffu, dst, h);
            for (int i = kLight + lane; i < hc; i += 32)
                perm2[hd + i] = perm ? perm[hs + i] : hs + i;
        }
    }
}

// parts of <= kItemParticles particles of each non-empty segment of seg levels
// of a super-column (C n consecutive merged cells)
__global__ void merged_seg_parts_kernel(const int32_t *__restrict__ cell_start2, int n, int C,
                                        int seg, int nseg, int nsegs, int *__restrict__ parts) {
    for (int sidx = blockIdx.x * blockDim.x + threadIdx.x; sidx <= nsegs;
         sidx += gridDim.x * blockDim.x) {
        if (sidx == nsegs) {
            parts[sidx] = 0;
            continue;
        }
        const int col = sidx / nseg, sg = sidx - col * nseg;
        const int64_t base = (int64_t)col * C * n;
        const int k0 = sg * seg, k1 = min(k0 + seg, n);
        const int c = cell_start2[base + (int64_t)k1 * C] - cell_start2[base + (int64_t)k0 * C];
        parts[sidx] = (c + kItemParticles - 1) / kItemParticles;
    }
}

template <int NA>
struct MergedChunk {
    double wx[NA][kChunk + 1];   // union x rows a' (times the strength)
    double wy[kChunk][9];        // [p][b]
    double wz[8][kWzStride];     // [c][p]
};

// this lane's particle: per-axis weights (es_fast.cuh), the x row shifted to
// the particle's sub-column q = i0x - ix0
template <int W, int NA>
__device__ __forceinline__ void merged_weights(MergedChunk<NA> &st, const double *tab,
                                               const EsPoly &P, int lane, int cnt, double x,
                                               double y, double z, double s, double h, double rh,
                                               double beta, int ix0, int n) {
    if (lane < cnt) {
        const double cx = axis_coord(x, h, rh);
        const int q = cell_index_of(cx, W, n) - ix0;
        PIF_CHECK(q >= 0 && q + 8 <= NA);
        double wt[W];
        es_axis_weights<W>(cx, beta, P, tab, wt);
#pragma unroll
        for (int a = 0; a < NA; ++a) st.wx[a][lane] = 0.0;
#pragma unroll
        for (int a = 0; a < W; ++a) st.wx[a + q][lane] = __dmul_rn(s, wt[a]);
        es_axis_weights<W>(axis_coord(y, h, rh), beta, P, tab, wt);
#pragma unroll
        for (int a = 0; a < W; ++a) st.wy[lane][a] = wt[a];
        es_axis_weights<W>(axis_coord(z, h, rh), beta, P, tab, wt);
#pragma unroll
        for (int a = 0; a < W; ++a) st.wz[a][lane] = wt[a];
    }
    __syncwarp();
}

template <int NA>
__device__ __forceinline__ void merged_flush_plane(double (&acc)[NA][2], int k, int c4, int ix0,
                                                   int64_t yrow, int n, double *grid) {
    const int s = k & 7;
    if (c4 == (s >> 1)) {
        const int j = s & 1;
#pragma unroll
        for (int a = 0; a < NA; ++a) {
            const double v = j ? acc[a][1] : acc[a][0];
            int xa = ix0 + a;
            xa = xa >= n ? xa - n : xa;   // n >= 32 > NA (merged_factor)
            if (v != 0.0) atomicAdd(grid + ((int64_t)xa * n + yrow) * n + k, v);
            if (j) acc[a][1] = 0.0;
            else acc[a][0] = 0.0;
        }
    }
}

// spread_mma_kernel over super-columns (same chunks, k-steps, z-slot planes
// and flush order per plane), NA = C + 7 union x rows per k-step
template <int W, int C>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, PIF_SPREAD_MINB)
spread_merged_kernel(const double *__restrict__ px, const double *__restrict__ py,
                     const double *__restrict__ pz, const int64_t *__restrict__ pid,
                     const int32_t *__restrict__ perm2, const double *__restrict__ strengths,
                     double q, const int32_t *__restrict__ cell_start2, double *__restrict__ grid,
                     int n, int seg, int nseg, double h, double beta, const EsPoly poly,
                     unsigned int *work, const int2 *__restrict__ items,
                     const int *__restrict__ n_items) {
    constexpr int NA = C + 7;
    const int nitems = *n_items;
    const double rh = __drcp_rn(h);
    __shared__ MergedChunk<NA> stage[kWarpsPerBlock];
    __shared__ double tab[32];
    __shared__ int seg_cells[kWarpsPerBlock][kMaxSeg + 1];
    if (threadIdx.x < 32) tab[threadIdx.x] = kExp2Table[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    MergedChunk<NA> &st = stage[threadIdx.x >> 5];
    int *cbt = seg_cells[threadIdx.x >> 5];
    {
        double *wp = &st.wx[0][0];
        const int nw = (int)(sizeof(MergedChunk<NA>) / sizeof(double));
        for (int i = lane; i < nw; i += 32) wp[i] = 0.0;
        __syncwarp();
    }
    const int r = lane >> 2, c4 = lane & 3;

    for (;;) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(work, 1u);
        item = __shfl_sync(kFull, item, 0);
        if (item >= nitems) break;
        const int2 it = items[item];
        const int col = it.x / nseg, sg = it.x - col * nseg;
        const int mx = col / n, iy = col - mx * n;
        const int ix0 = mx * C;
        const int k0 = sg * seg, k1 = min(k0 + seg, n);
        const int64_t base = (int64_t)col * C * n;
        __syncwarp();   // the previous item is done with the level table
        for (int c = lane; c <= k1 - k0; c += 32) cbt[c] = cell_start2[base + (int64_t)(k0 + c) * C];
        __syncwarp();
        const int pbeg = cbt[0] + it.y * kItemParticles;
        const int pend = min(pbeg + kItemParticles, cbt[k1 - k0]);
        const int64_t yrow = (iy + r) % n;

        double acc[NA][2];
#pragma unroll
        for (int a = 0; a < NA; ++a) acc[a][0] = acc[a][1] = 0.0;
        int k = k0;
        int cell_end = cbt[1];
        while (cell_end <= pbeg) cell_end = cbt[(++k) - k0 + 1];

        double nx = 0.0, ny = 0.0, nz = 0.0, ns = q;
        if (pbeg + lane < pend) {
            const int i = perm2[pbeg + lane];
            nx = px[i];
            ny = py[i];
            nz = pz[i];
            if (strengths) ns = strengths[pid[i]];
        }
        int npi = -1;
        if (pbeg + kChunk + lane < pend) npi = perm2[pbeg + kChunk + lane];
        for (int pos = pbeg; pos < pend; pos += kChunk) {
            const int cnt = min(kChunk, pend - pos);
            const double cx = nx, cy = ny, cz = nz, cs = ns;
            if (npi >= 0) {
                nx = px[npi];
                ny = py[npi];
                nz = pz[npi];
                if (strengths) ns = strengths[pid[npi]];
            }
            npi = -1;
            if (pos + 2 * kChunk + lane < pend) npi = perm2[pos + 2 * kChunk + lane];
            merged_weights<W, NA>(st, tab, poly, lane, cnt, cx, cy, cz, cs, h, rh, beta, ix0, n);
            int j = 0;
            while (j < cnt) {
                if (pos + j >= cell_end) {
                    merged_flush_plane<NA>(acc, k, c4, ix0, yrow, n, grid);
                    ++k;
                    cell_end = cbt[k - k0 + 1];
                    continue;
                }
                const int jend = min(cnt, cell_end - pos);
                const int zs = (r - k) & 7;
                PIF_CHECK(jend <= kChunk && k >= k0 && k < k1);
#pragma unroll kSpreadUnroll
                for (; j + 4 <= jend; j += 4) {
                    const int pj = j + c4;
                    const double wyb = st.wy[pj][r];
                    const double bz = st.wz[zs][pj];
#pragma unroll
                    for (int a = 0; a < NA; ++a)
                        dmma884(acc[a][0], acc[a][1], st.wx[a][pj] * wyb, bz);
                }
                if (j < jend) {
                    const bool ok = c4 < jend - j;
                    const int pj = ok ? j + c4 : j;
                    const double wyb = ok ? st.wy[pj][r] : 0.0;
                    const double bz = st.wz[zs][pj];
#pragma unroll
                    for (int a = 0; a < NA; ++a)
                        dmma884(acc[a][0], acc[a][1], st.wx[a][pj] * wyb, bz);
                    j = jend;
                }
            }
            __syncwarp();
        }
        for (; k < k1; ++k) merged_flush_plane<NA>(acc, k, c4, ix0, yrow, n, grid);
        // pending planes k1 .. k1+6
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int sl = 2 * c4 + jj;
            const int dz = (sl - k1) & 7;   // dz == 7: plane k1 + 7, flushed with cell k1 - 1
            const int z = (k1 + dz) % n;
#pragma unroll
            for (int a = 0; a < NA; ++a) {
                const double v = acc[a][jj];
                int xa = ix0 + a;
                xa = xa >= n ? xa - n : xa;
                if (v != 0.0) atomicAdd(grid + ((int64_t)xa * n + yrow) * n + z, v);
            }
        }
    }
}

// Deterministic plane reduction: grid point (X, Y, Z) = sum over the footprint
// rows (a, b) of column (X - a, Y - b), over the z-segments of that column
// whose footprint [k0, k1 + 7) covers Z (cyclically), over each segment's
// parts in order.
// Fixed order, so the grid is the same bits on every run.
__global__ void det_reduce_kernel(const double *__restrict__ dbuf, int64_t stride,
                                  const int *__restrict__ seg_off, const int *__restrict__ seg_parts,
                                  int n, int seg, int nseg, int w, double *__restrict__ grid) {
    const int64_t n3 = (int64_t)n * n * n;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n3;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int Z = (int)(idx % n), Y = (int)((idx / n) % n), X = (int)(idx / ((int64_t)n * n));
        // the segment holding Z and the ones before it (cyclically) whose 7-plane
        // tails may reach Z: a short last segment (n % seg < 7) lets the tail
        // of the one before it wrap past it, so walk back up to 8 segments
        const int s0 = Z / seg, nback = min(nseg, 8);
        double acc = 0.0;
        for (int a = 0; a < w; ++a) {
            const int ix = (X - a + n) % n;
            for (int b = 0; b < w; ++b) {
                const int col = ix * n + (Y - b + n) % n;
                for (int t = 0; t < nback; ++t) {
                    const int sg = (s0 - t + nseg) % nseg;
                    const int k0 = sg * seg, len = min(k0 + seg, n) - k0;
                    const int sidx = col * nseg + sg;
                    const int first = seg_off[sidx], cnt = seg_parts[sidx];
                    for (int pz = (Z - k0 + n) % n; pz < len + 7; pz += n)
                        for (int j = 0; j < cnt; ++j)
                            acc += dbuf[((int64_t)(first + j) * 64 + a * 8 + b) * stride + pz];
                }
            }
        }
        grid[idx] = acc;
    }
}

// ----------------------------------------------------------------------------
// gather (+ Boris push) (w <= 8) on the fp64 tensor cores
//
// The field window of the current cell (8 a x 8 b x 8 z-slots x 3 components)
// lives in registers as DMMA A fragments: A_{a,h,d}[b][c'] = E_d(a, b, slot
// c' + 4h).  For a sub-batch of up to 8 particles of the cell,
// B_{a,h}[c'][p] = wx_p[a] wz_p[(c' + 4h - k) mod 8], so 16 DMMAs per component
// accumulate D_d[b][p] = sum_{a,c} E_d(a,b,c) wx_p[a] wz_p[c]; the remaining
// wy_p[b] contraction is 6 products and a 3-level butterfly over the b lanes.
// Gathered fields go to shared memory; then every lane pushes one particle of
// the chunk (coalesced loads/stores).
// ----------------------------------------------------------------------------

struct PushParams {
    double half, dt, L, h, rh;
    double ext_c, ext_xy, ext_z, pot_xy, pot_z;   // L/2, -15/L, 30/L, 7.5/L, 15/L
    double tq[3], sq[3];
    int has_b, e_kind, n, w;
    double *mx, *mv;      // id-order mirror (pif_set_id_order_output) or null
    long long mid0;
    double *eslot;        // gather only: E rows id - mid0 of an (M,3) array (pif_interp_split)
};

// pushed particle also written to row id - mid0 of the (M,3) mirrors
__device__ __forceinline__ void mirror_store(const PushParams &pp, int64_t id, double x, double y,
                                             double z, double vx, double vy, double vz) {
    if (pp.mx) {
        const int64_t o = 3 * (id - pp.mid0);
        pp.mx[o] = x;
        pp.mx[o + 1] = y;
        pp.mx[o + 2] = z;
        pp.mv[o] = vx;
        pp.mv[o + 1] = vy;
        pp.mv[o + 2] = vz;
    }
}

// Boris push of one particle (pif.py:146-157), external quadrupole
// (pif.py:52-57), periodic wrap (particles.py:65-70); no FMA contraction so the
// update rounds like numpy.  Accumulates diagnostics of the updated particle.
__device__ __forceinline__ void boris_one(const PushParams &pp, double E0, double E1, double E2,
                                          double &x, double &y, double &z, double &vx,
                                          double &vy, double &vz, double *dg) {
    double et0 = E0, et1 = E1, et2 = E2;
    const double L = pp.L;
    if (pp.e_kind == PIF_EXT_QUADRUPOLE) {
        const double c = pp.ext_c;
        et0 = __dadd_rn(et0, __dmul_rn(pp.ext_xy, __dsub_rn(x, c)));
        et1 = __dadd_rn(et1, __dmul_rn(pp.ext_xy, __dsub_rn(y, c)));
        et2 = __dadd_rn(et2, __dmul_rn(pp.ext_z, __dsub_rn(z, c)));
    }
    const double hf = pp.half;
    double m0 = __dadd_rn(vx, __dmul_rn(hf, et0));
    double m1 = __dadd_rn(vy, __dmul_rn(hf, et1));
    double m2 = __dadd_rn(vz, __dmul_rn(hf, et2));
    if (pp.has_b) {
        const double *t = pp.tq, *s = pp.sq;
        // vp = vm + vm x t ; vm = vm + vp x s  (pif.py:154-155)
        double p0 = __dadd_rn(m0, __dsub_rn(__dmul_rn(m1, t[2]), __dmul_rn(m2, t[1])));
        double p1 = __dadd_rn(m1, __dsub_rn(__dmul_rn(m2, t[0]), __dmul_rn(m0, t[2])));
        double p2 = __dadd_rn(m2, __dsub_rn(__dmul_rn(m0, t[1]), __dmul_rn(m1, t[0])));
        double n0 = __dadd_rn(m0, __dsub_rn(__dmul_rn(p1, s[2]), __dmul_rn(p2, s[1])));
        double n1 = __dadd_rn(m1, __dsub_rn(__dmul_rn(p2, s[0]), __dmul_rn(p0, s[2])));
        double n2 = __dadd_rn(m2, __dsub_rn(__dmul_rn(p0, s[1]), __dmul_rn(p1, s[0])));
        m0 = n0;
        m1 = n1;
        m2 = n2;
    }
    vx = __dadd_rn(m0, __dmul_rn(hf, et0));
    vy = __dadd_rn(m1, __dmul_rn(hf, et1));
    vz = __dadd_rn(m2, __dmul_rn(hf, et2));
    x = wrap_coord(__dadd_rn(x, __dmul_rn(pp.dt, vx)), L);
    y = wrap_coord(__dadd_rn(y, __dmul_rn(pp.dt, vy)), L);
    z = wrap_coord(__dadd_rn(z, __dmul_rn(pp.dt, vz)), L);
    dg[0] += vx * vx + vy * vy + vz * vz;
    dg[1] += vx;
    dg[2] += vy;
    dg[3] += vz;
    if (pp.e_kind == PIF_EXT_QUADRUPOLE) {
        const double c = pp.ext_c;
        const double dx = x - c, dy = y - c, dz = z - c;
        dg[4] += pp.pot_xy * (dx * dx + dy * dy) - pp.pot_z * (dz * dz);
    }
}

__device__ __forceinline__ void block_diag_store(double *dg, double *partials) {
    __shared__ double red[32][5];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int d = 0; d < 5; ++d) dg[d] = warp_sum(dg[d]);
    if (lane == 0)
        for (int d = 0; d < 5; ++d) red[wid][d] = dg[d];
    __syncthreads();
    if (threadIdx.x < 5) {
        double s = 0.0;
        for (int i = 0; i < nw; ++i) s += red[i][threadIdx.x];
        partials[blockIdx.x * kDiagSlots + threadIdx.x] = s;
    }
}

__device__ __forceinline__ void load_plane(double (&g)[8][2][3], int hh, const double4 *field,
                                           int ix, int64_t yrow, int n, int64_t z) {
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        int xa = ix + a;
        xa = xa >= n ? xa - n : xa;
        PIF_CHECK(xa >= 0 && xa < n && yrow >= 0 && yrow < n && z >= 0 && z < n);
        const double4 f = field[((int64_t)xa * n + yrow) * n + z];
        g[a][hh][0] = f.x;
        g[a][hh][1] = f.y;
        g[a][hh][2] = f.z;
    }
}

// One sub-batch of up to m particles (<= 8) of cell k starting at chunk slot j.
// DMMA with the particle weights as the A operand and the register window as
// the B operand (the A and B fragment layouts are transposes of each other, so
// lane (r, c4) holding E(a, b=r, slot c4+4h) is a valid B fragment):
//   A_{a,h}[p][c'] = wx_p[a] wz_p[(c' + 4h - k) mod 8]    (p = r)
//   D_d[p][b]     += A_{a,h} x B_{a,h,d}[c'][b]           (16 DMMAs per component)
// The 8 x 8 result D_d[p][b] of the sub-batch goes to shared memory;
// E_d(p) = sum_b wy_p[b] D_d[p][b] is formed later by lane p (gather_reduce),
// off the DMMA loop's critical path.
__device__ __forceinline__ void gather_sub_d(WarpChunk &st, GatherPartials &gp,
                                             const double (&g)[8][2][3], int j, int m, int k,
                                             int r, int c4) {
    const int pb = r < m ? j + r : j;
    const double sc = r < m ? 1.0 : 0.0;
    const double bz0 = sc * st.wz[(c4 - k) & 7][pb];
    const double bz1 = sc * st.wz[(c4 + 4 - k) & 7][pb];
    double A[8][2];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const double wxa = st.wx[a][pb];
        A[a][0] = wxa * bz0;
        A[a][1] = wxa * bz1;
    }
#if PIF_GATHER_CHAINS == 3
    // one accumulator chain per component (16 DMMAs each, interleaved: a
    // chain's next DMMA issues 3 DMMAs = 48 clk later, past the ~29 clk DMMA
    // latency), so no per-sub-batch merge adds
    double D[3][2];
#pragma unroll
    for (int d = 0; d < 3; ++d) D[d][0] = D[d][1] = 0.0;
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int d = 0; d < 3; ++d) dmma884(D[d][0], D[d][1], A[a][hh], g[a][hh][d]);
    if (r < m) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            gp.D[d][2 * c4][j + r] = D[d][0];
            gp.D[d][2 * c4 + 1][j + r] = D[d][1];
        }
    }
#else
    double Dh[2][3][2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int d = 0; d < 3; ++d) Dh[hh][d][0] = Dh[hh][d][1] = 0.0;
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int d = 0; d < 3; ++d)
                dmma884(Dh[hh][d][0], Dh[hh][d][1], A[a][hh], g[a][hh][d]);
    if (r < m) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            gp.D[d][2 * c4][j + r] = Dh[0][d][0] + Dh[1][d][0];
            gp.D[d][2 * c4 + 1][j + r] = Dh[0][d][1] + Dh[1][d][1];
        }
    }
#endif
}

// A sub-batch of m < 8 particles without the tensor cores: lane (r, c4) adds
// its window entries (b = r, slots c4 and c4 + 4) weighted by wx and wz for each
// particle and the 4 lanes of row r reduce, giving the same D_d[p][b] as
// gather_sub_d.  Pipe cost ~54 FMAs per particle against 48 DMMAs per
// sub-batch, so partial sub-batches (cell tails, sparse cells) run here.
template <bool PAIRS>
__device__ __forceinline__ void gather_sub_fma(WarpChunk &st, GatherPartials &gp,
                                               const double (&g)[8][2][3], int j, int m, int k,
                                               int r, int c4) {
    const int s0 = (c4 - k) & 7, s1 = (c4 + 4 - k) & 7;
    int q = j;
    // PAIRS (sparse sets, which run almost all their particles here): two
    // particles at a time, 12 independent FMA chains and 6 shuffle reductions
    // in flight instead of 6 and 3; each particle's arithmetic is unchanged
    // (256^3 / 1.25 per cell: gather -1.5%; dense sets: +1%, so not there)
    for (; PAIRS && q + 2 <= j + m; q += 2) {
        double h0[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
        double h1[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const double xa = st.wx[a][q], xb = st.wx[a][q + 1];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                h0[0][d] = fma(g[a][0][d], xa, h0[0][d]);
                h1[0][d] = fma(g[a][1][d], xa, h1[0][d]);
                h0[1][d] = fma(g[a][0][d], xb, h0[1][d]);
                h1[1][d] = fma(g[a][1][d], xb, h1[1][d]);
            }
        }
        double e[2][3];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const double z0 = st.wz[s0][q + u], z1 = st.wz[s1][q + u];
#pragma unroll
            for (int d = 0; d < 3; ++d) e[u][d] = fma(h1[u][d], z1, h0[u][d] * z0);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int d = 0; d < 3; ++d) e[u][d] += __shfl_xor_sync(kFull, e[u][d], 1);
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int d = 0; d < 3; ++d) e[u][d] += __shfl_xor_sync(kFull, e[u][d], 2);
        if (c4 == 0) {
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int d = 0; d < 3; ++d) gp.D[d][r][q + u] = e[u][d];
        }
    }
    for (; q < j + m; ++q) {
        double h0[3] = {0.0, 0.0, 0.0}, h1[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const double xa = st.wx[a][q];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                h0[d] = fma(g[a][0][d], xa, h0[d]);
                h1[d] = fma(g[a][1][d], xa, h1[d]);
            }
        }
        const double z0 = st.wz[s0][q], z1 = st.wz[s1][q];
        double e[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            e[d] = fma(h1[d], z1, h0[d] * z0);
            e[d] += __shfl_xor_sync(kFull, e[d], 1);
            e[d] += __shfl_xor_sync(kFull, e[d], 2);
        }
        if (c4 == 0) {
#pragma unroll
            for (int d = 0; d < 3; ++d) gp.D[d][r][q] = e[d];
        }
    }
}

// E of this lane's particle p from its partial sums (same pairing as the
// pairwise tree ((b0 b1 + b2 b3) + (b4 b5 + b6 b7)))
__device__ __forceinline__ void gather_reduce(const WarpChunk &st, const GatherPartials &gp, int p,
                                              double (&E)[3]) {
    double wy[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) wy[b] = st.wy[p][b];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double e[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            e[q] = fma(wy[2 * q + 1], gp.D[d][2 * q + 1][p], wy[2 * q] * gp.D[d][2 * q][p]);
        E[d] = (e[0] + e[1]) + (e[2] + e[3]);
    }
}

// Next-plane prefetch: all 32 lanes copy the 8 x 8 double4 block of plane z
// into shared memory with cp.async (LDGSTS) one cell ahead of its use.
__device__ __forceinline__ void prefetch_plane(double4 (*pf)[8], const double4 *field, int ix,
                                               int iy, int n, int64_t z, int lane) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int q = lane + 32 * t;              // 16-byte chunk: (a, b, half)
        const int a = q >> 4, b = (q >> 1) & 7, hf = q & 1;
        int xa = ix + a;
        xa = xa >= n ? xa - n : xa;
        int yb = iy + b;
        yb = yb >= n ? yb - n : yb;
        const char *src = reinterpret_cast<const char *>(field + ((int64_t)xa * n + yb) * n + z) +
                          16 * hf;
        const unsigned dst =
            (unsigned)__cvta_generic_to_shared(reinterpret_cast<char *>(&pf[a][b]) + 16 * hf);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
    }
    asm volatile("cp.async.commit_group;");
}

__device__ __forceinline__ void prefetch_wait() {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
}

__device__ __forceinline__ void plane_from_smem(double (&g)[8][2][3], int hh, double4 (*pf)[8],
                                                int r) {
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const double4 f = pf[a][r];
        g[a][hh][0] = f.x;
        g[a][hh][1] = f.y;
        g[a][hh][2] = f.z;
    }
}

#ifdef PIF_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[8];
#define PHASE_MARK(v) long long v = clock64()
#define PHASE_ADD(slot, a, b) ph[slot] += (unsigned long long)((b) - (a))
#else
#define PHASE_MARK(v)
#define PHASE_ADD(slot, a, b)
#endif

#ifndef PIF_INTERP_MINB
#define PIF_INTERP_MINB 2
#endif
#ifndef PIF_INTERP_MINB_WC
#define PIF_INTERP_MINB_WC 2
#endif
// sub-batches of at most this many particles take the FMA path
#ifndef PIF_GATHER_FMA_MAX
#define PIF_GATHER_FMA_MAX 3
#endif
constexpr int kGatherFmaMax = PIF_GATHER_FMA_MAX;

#ifndef PIF_GATHER_WARPS
#define PIF_GATHER_WARPS 4
#endif
constexpr int kGatherWarps = PIF_GATHER_WARPS;   // warps per gather block

// WC: the window weights come from the spread's cache (pif_set_weight_cache)
// instead of being evaluated here; a separate instantiation so the polynomial
// code and its registers are not carried when unused.  AGG (Plan::push_agg,
// sets with heavy cells): dense segments count next-cell keys per run of
// equal keys; its own instantiation for the same reason (+9 registers, 2%
// slower where per-lane REDs do not collide).
template <int W, bool PUSH, bool LONGSEG, bool WC, bool AGG>
__global__ void __launch_bounds__(kGatherWarps * 32, WC ? PIF_INTERP_MINB_WC : PIF_INTERP_MINB)
interp_mma_kernel(pif_soa_t P, const int32_t *__restrict__ perm, pif_soa_t Q,
                  const int32_t *__restrict__ cell_start,
                  const double4 *__restrict__ field, int seg, int nseg, double beta,
                  const EsPoly poly, PushParams pp, int32_t *__restrict__ key,
                  int32_t *__restrict__ rank, int32_t *__restrict__ count,
                  double *__restrict__ partials, double *__restrict__ E_out, unsigned int *work,
                  const int2 *__restrict__ items, const int *__restrict__ n_items,
                  const double *__restrict__ wc, int64_t wstride) {
    const int nitems = *n_items;
    __shared__ WarpChunk stage[kGatherWarps];
    __shared__ double4 planes[kGatherWarps][8][8];
    __shared__ double tab[32];
    // this item's cell boundaries: one per lane in a register (segments of
    // <= 31 cells), or a per-warp shared table (LONGSEG: up to kMaxSeg cells)
    __shared__ int seg_cells[LONGSEG ? kGatherWarps : 1][LONGSEG ? kMaxSeg + 1 : 1];
    extern __shared__ double4 dyn_smem[];
    GatherPartials &gpart = reinterpret_cast<GatherPartials *>(dyn_smem)[threadIdx.x >> 5];
    int *cbt = seg_cells[LONGSEG ? (threadIdx.x >> 5) : 0];
    WarpChunk *stage2 = reinterpret_cast<WarpChunk *>(
        reinterpret_cast<GatherPartials *>(dyn_smem) + kGatherWarps);
    if (threadIdx.x < 32) tab[threadIdx.x] = kExp2Table[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    WarpChunk &st0 = stage[threadIdx.x >> 5];
    // with the weight cache, chunks alternate between two stages (the next
    // chunk's weights land by cp.async while this one is gathered)
    WarpChunk &st1 = WC ? stage2[threadIdx.x >> 5] : st0;
    double4 (*pf)[8] = planes[threadIdx.x >> 5];
    chunk_zero(st0, lane);
    if (WC) chunk_zero(st1, lane);
    int wb = 0;            // stage of the current chunk
    bool wnewest = false;  // the newest cp.async group holds weights (not a plane)
    const int n = pp.n;
    const double h = pp.h;
    const int r = lane >> 2, c4 = lane & 3;
    double dg[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    // rank of the previous chunk's particle: stored one chunk later so the
    // atomic's round trip overlaps the next chunk's work
    int64_t rank_idx = -1;
    int rank_val = 0;
#ifdef PIF_PHASE_TIMING
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif

    for (;;) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(work, 1u);
        item = __shfl_sync(kFull, item, 0);
        if (item >= nitems) break;
        const int2 it = items[item];
        const int col = it.x / nseg, sg = it.x - col * nseg;
        const int ix = col / n, iy = col - ix * n;
        const int k0 = sg * seg, k1 = min(k0 + seg, n);
        const int base = col * n;
        int cb = 0;
        if (LONGSEG) {
            __syncwarp();   // the previous item is done with the cell table
            for (int c = lane; c <= k1 - k0; c += 32) cbt[c] = cell_start[base + k0 + c];
            __syncwarp();
        } else {
            cb = cell_start[base + k0 + min(lane, k1 - k0)];
        }
        // boundary t of the item's cells (warp-uniform t)
        auto bound = [&](int t) { return LONGSEG ? cbt[t] : __shfl_sync(kFull, cb, t); };
        const int pbeg = bound(0) + it.y * kItemParticles;
        const int pend = min(pbeg + kItemParticles, bound(k1 - k0));
        // dense segment (> 3 parts, so several warps push into the same few
        // cells at once): one count RED per run of equal next-cell keys in
        // lane order instead of one per particle.  Per-lane REDs to one
        // address serialise in L2 (Penning 2^28 per GPU: gather 57.6 ->
        // 34.3 ms); at 64 per cell they are cheaper than the warp exchange.
        const bool agg = AGG && PUSH && !rank && bound(k1 - k0) - bound(0) > 3 * kItemParticles;
        int kf = k0;   // cell holding the item's first particle
        while (bound(kf - k0 + 1) <= pbeg) ++kf;
        const int64_t yrow = (iy + r) % n;

        // prefetch the first chunk (positions, velocities, id) before the window;
        // the perm entries run one chunk further ahead than the particle data,
        // so a chunk's data loads never wait on their own perm load
        double nx = 0.0, ny = 0.0, nz = 0.0, nvx = 0.0, nvy = 0.0, nvz = 0.0;
        int64_t nid = 0;
        if (pbeg + lane < pend) {
            const int i = perm ? perm[pbeg + lane] : pbeg + lane;
            nx = P.x[i]; ny = P.y[i]; nz = P.z[i];
            if (PUSH) { nvx = P.vx[i]; nvy = P.vy[i]; nvz = P.vz[i]; }
            if (perm || !PUSH || pp.mx) nid = P.id[i];
        }
        int npi = -1;   // perm entry of this lane's particle in the next chunk
        if (pbeg + kChunk + lane < pend)
            npi = perm ? perm[pbeg + kChunk + lane] : pbeg + kChunk + lane;
        // window: slot s = c4 + 4h holds plane z == s (mod 8) of [kf, kf+8)
        double g[8][2][3];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int s = c4 + 4 * hh;
            load_plane(g, hh, field, ix, yrow, n, (kf + ((s - kf) & 7)) % n);
        }
        int k = kf;
        int cell_end = bound(kf - k0 + 1);
        prefetch_wait();   // previous item's outstanding prefetch
        if (WC) {          // first chunk's cached weights
            chunk_weights_async<W>(wb ? st1 : st0, wc, wstride, pbeg + lane, lane,
                                   min(kChunk, pend - pbeg));
        }
        prefetch_plane(pf, field, ix, iy, n, (kf + 8) % n, lane);
        wnewest = false;

        for (int pos = pbeg; pos < pend; pos += kChunk) {
            const int cnt = min(kChunk, pend - pos);
            const double x0 = nx, y0 = ny, z0 = nz, vx0 = nvx, vy0 = nvy, vz0 = nvz;
            const int64_t id0 = nid;
            if (PUSH && rank_idx >= 0) {
                rank[rank_idx] = rank_val;
                rank_idx = -1;
            }
            if (npi >= 0) {   // prefetch the next chunk (its perm entry is already here)
                const int i = npi;
                nx = P.x[i]; ny = P.y[i]; nz = P.z[i];
                if (PUSH) { nvx = P.vx[i]; nvy = P.vy[i]; nvz = P.vz[i]; }
                if (perm || !PUSH || pp.mx) nid = P.id[i];
            }
            npi = -1;         // and the perm entry of the chunk after it
            if (pos + 2 * kChunk + lane < pend)
                npi = perm ? perm[pos + 2 * kChunk + lane] : pos + 2 * kChunk + lane;
            PHASE_MARK(t0);
            WarpChunk &st = wb ? st1 : st0;
            if (WC) {
                if (pos + kChunk < pend) {   // next chunk's weights into the other stage
                    chunk_weights_async<W>(wb ? st0 : st1, wc, wstride, pos + kChunk + lane,
                                           lane, min(kChunk, pend - pos - kChunk));
                    asm volatile("cp.async.wait_group 1;" ::: "memory");
                    wnewest = true;
                } else {
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                    wnewest = false;
                }
                __syncwarp();
            } else {
                chunk_weights<W, true>(st, tab, poly, lane, cnt, x0, y0, z0, 1.0, false, h, pp.rh,
                                       beta);
            }
            PHASE_MARK(t1);
            PHASE_ADD(0, t0, t1);
            int j = 0;
            while (j < cnt) {
                const int gp = pos + j;
                if (gp >= cell_end) {   // next cell: plane k leaves slot k&7, plane k+8 enters
                    const int s = k & 7;
                    if (wnewest) {   // the plane group is older than the weights group
                        asm volatile("cp.async.wait_group 1;" ::: "memory");
                        __syncwarp();
                    } else {
                        prefetch_wait();
                    }
                    if (c4 == (s & 3)) {
                        if (s >> 2) plane_from_smem(g, 1, pf, r);
                        else plane_from_smem(g, 0, pf, r);
                    }
                    __syncwarp();
                    ++k;
                    prefetch_plane(pf, field, ix, iy, n, (k + 8) % n, lane);
                    wnewest = false;
                    cell_end = bound(k - k0 + 1);
                    continue;
                }
                const int m = min(8, min(pos + cnt, cell_end) - gp);
                PIF_CHECK(m > 0 && j + m <= kChunk && k >= k0 && k < k1);
                if (m <= kGatherFmaMax) gather_sub_fma<LONGSEG>(st, gpart, g, j, m, k, r, c4);
                else gather_sub_d(st, gpart, g, j, m, k, r, c4);
                j += m;
            }
            __syncwarp();
            PHASE_MARK(t2);
            PHASE_ADD(1, t1, t2);
            int ckey = -1;   // next cell key to count (dense segments)
            if (lane < cnt) {
                const int64_t i = pos + lane;
                double Eg[3];
                gather_reduce(st, gpart, lane, Eg);
                const double E0 = Eg[0], E1 = Eg[1], E2 = Eg[2];
                if (PUSH) {
                    double x = x0, y = y0, z = z0;
                    double vx = vx0, vy = vy0, vz = vz0;
                    boris_one(pp, E0, E1, E2, x, y, z, vx, vy, vz, dg);
                    Q.x[i] = x; Q.y[i] = y; Q.z[i] = z;
                    Q.vx[i] = vx; Q.vy[i] = vy; Q.vz[i] = vz;
                    if (perm) Q.id[i] = id0;
                    mirror_store(pp, id0, x, y, z, vx, vy, vz);
                    const int kk = cell_key(x, y, z, h, pp.rh, pp.w, n);
                    PIF_CHECK(kk >= 0 && kk < n * n * n && i < P.count);
                    key[i] = kk;
                    if (rank) {
                        rank_val = atomicAdd(&count[kk], 1);
                        rank_idx = i;
                    } else {
                        // count only (RED, nothing returns): pif_bin_perm
                        // assigns the in-cell slots, so no atomic round trip
                        // sits on this warp's scoreboards.  Dense segments
                        // count per run of equal keys after the lane branch.
                        if (agg) ckey = kk;
                        else atomicAdd(&count[kk], 1);
                    }
                } else if (pp.eslot) {   // row id - mid0, for pif_push_ids
                    const int64_t o = 3 * (id0 - pp.mid0);
                    pp.eslot[o] = E0;
                    pp.eslot[o + 1] = E1;
                    pp.eslot[o + 2] = E2;
                } else {
                    const int64_t o = 3 * id0;
                    E_out[o] = E0;
                    E_out[o + 1] = E1;
                    E_out[o + 2] = E2;
                }
            }
            if (AGG && PUSH && agg) {
                const int prev_k = __shfl_up_sync(kFull, ckey, 1);
                const bool head = ckey >= 0 && (lane == 0 || prev_k != ckey);
                const unsigned heads = __ballot_sync(kFull, lane == 0 || prev_k != ckey);
                if (head) {
                    const unsigned later = heads & ~((2u << lane) - 1u);
                    const int end = later ? __ffs(later) - 1 : cnt;
                    atomicAdd(&count[ckey], end - lane);
                }
            }
            __syncwarp();
            PHASE_MARK(t3);
            PHASE_ADD(2, t2, t3);
#ifdef PIF_PHASE_TIMING
            ph[3] += 1;
            ph[4] += (unsigned long long)cnt;
#endif
            if (WC) wb ^= 1;
        }
    }
#ifdef PIF_PHASE_TIMING
    if (lane == 0)
        for (int i = 0; i < 5; ++i) atomicAdd(&g_phase_cycles[i], ph[i]);
#endif
    prefetch_wait();
    if (PUSH && rank_idx >= 0) rank[rank_idx] = rank_val;
    if (PUSH) block_diag_store(dg, partials);
}

// ----------------------------------------------------------------------------
// wide windows (9 <= w <= 17): FMA "ring" kernels
//
// Same work items, chunks and cell order as the DMMA kernels, but the w x w
// (a, b) pairs of the footprint are dealt to the lanes and each lane keeps,
// per pair, a ring of w z-slots in registers (slot s holds plane z == s mod w
// of the current cell's footprint).  Per particle of a chunk, lane-owned pairs
// do acc[t][s] += (s wx[a] wy[b]) wz[s]: w FMAs per pair, all lanes busy, no
// atomics until a plane leaves the ring.  The particle's z weights are stored
// rotated into slot order by the lane that computes them, so the inner loop has
// compile-time register indices.  From w = 13 (eps <= 1e-12) one warp does
// not hold w^2 rings without spilling (w = 13 / 14 unsplit: 200-600 B of
// spills; split vs unsplit A/B in profiles/round2/ring_split_ab.txt), from
// w = 15 not at all: the pair set is split over G warps ("sub-warps", each
// claiming (item, part) of the work list), <= 4 pairs per lane; the spread's
// sub-warps flush their own pairs, the gather's add their partial sums into
// the per-position scratch and a separate pass pushes.
// ----------------------------------------------------------------------------

// from this width on the pair set is split over sub-warps (<= 4 pairs per lane)
#ifndef PIF_RING_SPLIT_W
#define PIF_RING_SPLIT_W 13
#endif
template <int W>
struct RingSplit {
    static constexpr int G = W < PIF_RING_SPLIT_W ? 1 : (W * W + 127) / 128;   // sub-warps per item
    static constexpr int NP = (W * W + 32 * G - 1) / (32 * G);               // pairs per lane
};

template <int W>
struct RingStage {
    double wx[kChunk][W + 1];   // [p][a] (spreading: times the strength)
    double wy[kChunk][W + 1];   // [p][b]
    double wz[kChunk][W + 1];   // [p][slot]: wz[c] at slot (k_p + c) mod W
};

// the w window weights of one axis: interior ones by polynomial up to
// kMaxPolyW, the exact formula (es_weight_fast) for wider windows
template <int W>
__device__ __forceinline__ void ring_axis_weights(double c, double beta, const EsPoly &P,
                                                  const double *tab, double (&wt)[W]) {
    if (W <= kMaxPolyW) {
        es_axis_weights<W>(c, beta, P, tab, wt);
    } else {
        constexpr double inv_half = 2.0 / W;
        const double i0 = stencil_start(c, W);
#pragma unroll
        for (int a = 0; a < W; ++a) wt[a] = es_weight_fast(c, i0 + (double)a, inv_half, beta, tab);
    }
}

// lane p: window weights of its particle into the stage (z rotated by its cell)
template <int W>
__device__ __forceinline__ void ring_weights(RingStage<W> &st, const double *tab, const EsPoly &P,
                                             int lane, int cnt, double x, double y, double z,
                                             double sc, double h, double rh, double beta, int n) {
    if (lane < cnt) {
        // one axis at a time: the ring accumulators stay live across this phase
        double wt[W];
        ring_axis_weights<W>(axis_coord(x, h, rh), beta, P, tab, wt);
#pragma unroll
        for (int a = 0; a < W; ++a) st.wx[lane][a] = __dmul_rn(sc, wt[a]);
        ring_axis_weights<W>(axis_coord(y, h, rh), beta, P, tab, wt);
#pragma unroll
        for (int a = 0; a < W; ++a) st.wy[lane][a] = wt[a];
        const double cz = axis_coord(z, h, rh);
        ring_axis_weights<W>(cz, beta, P, tab, wt);
        const int r0 = pmod((int)stencil_start(cz, W), n) % W;
#pragma unroll
        for (int a = 0; a < W; ++a) {
            const int sl = r0 + a >= W ? r0 + a - W : r0 + a;
            st.wz[lane][sl] = wt[a];
        }
    }
    __syncwarp();
}

// plane z (ring slot `slot`) leaves the ring: lane-owned pairs (qbase + lane +
// 32 t) add their value at (ix + a, iy + b, z) and clear the slot
template <int W>
__device__ __forceinline__ void ring_flush_slot(double (&acc)[RingSplit<W>::NP][W], int slot,
                                                int lane, int qbase, int ix, int iy, int n,
                                                int64_t z, double *grid) {
    constexpr int NP = RingSplit<W>::NP;
#pragma unroll
    for (int s = 0; s < W; ++s) {
        if (s == slot) {
#pragma unroll
            for (int t = 0; t < NP; ++t) {
                const int qq = qbase + lane + 32 * t;
                const double v = acc[t][s];
                if (qq < W * W && v != 0.0) {
                    const int a = qq / W, b = qq - (qq / W) * W;
                    const int xa = (ix + a) % n, yb = (iy + b) % n;   // w may exceed n
                    atomicAdd(grid + ((int64_t)xa * n + yb) * n + z, v);
                }
                acc[t][s] = 0.0;
            }
        }
    }
}

template <int W>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
spread_ring_kernel(const double *__restrict__ px, const double *__restrict__ py,
                   const double *__restrict__ pz, const int64_t *__restrict__ pid,
                   const int32_t *__restrict__ perm, const double *__restrict__ strengths, double q,
                   const int32_t *__restrict__ cell_start, double *__restrict__ grid, int n,
                   int seg, int nseg, double h, double beta, const EsPoly poly, unsigned int *work,
                   const int2 *__restrict__ items, const int *__restrict__ n_items) {
    constexpr int NP = RingSplit<W>::NP, G = RingSplit<W>::G;
    const int nunits = *n_items * G;
    const double rh = __drcp_rn(h);
    extern __shared__ double4 ring_spread_smem[];   // RingStage<W> per warp
    __shared__ double tab[32];
    __shared__ int seg_cells[kWarpsPerBlock][kMaxSeg + 1];   // the item's cell boundaries
    if (threadIdx.x < 32) tab[threadIdx.x] = kExp2Table[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    RingStage<W> &st = reinterpret_cast<RingStage<W> *>(ring_spread_smem)[threadIdx.x >> 5];
    int *cbt = seg_cells[threadIdx.x >> 5];

    for (;;) {
        int unit = 0;
        if (lane == 0) unit = (int)atomicAdd(work, 1u);
        unit = __shfl_sync(kFull, unit, 0);
        if (unit >= nunits) break;
        const int item = unit / G, qbase = (unit - item * G) * 32 * NP;
        int pa[NP], pb[NP];
#pragma unroll
        for (int t = 0; t < NP; ++t) {
            const int qq = qbase + lane + 32 * t;
            pa[t] = qq < W * W ? qq / W : 0;
            pb[t] = qq < W * W ? qq % W : 0;
        }
        const int2 it = items[item];
        const int col = it.x / nseg, sg = it.x - col * nseg;
        const int ix = col / n, iy = col - ix * n;
        const int k0 = sg * seg, k1 = min(k0 + seg, n);
        const int base = col * n;
        __syncwarp();   // the previous item is done with the cell table
        for (int c = lane; c <= k1 - k0; c += 32) cbt[c] = cell_start[base + k0 + c];
        __syncwarp();
        const int pbeg = cbt[0] + it.y * kItemParticles;
        const int pend = min(pbeg + kItemParticles, cbt[k1 - k0]);
        double acc[NP][W];
#pragma unroll
        for (int t = 0; t < NP; ++t)
#pragma unroll
            for (int s = 0; s < W; ++s) acc[t][s] = 0.0;
        int k = k0;
        int cell_end = cbt[1];
        while (cell_end <= pbeg) cell_end = cbt[(++k) - k0 + 1];

        double nx = 0.0, ny = 0.0, nz = 0.0, ns = q;
        if (pbeg + lane < pend) {
            const int i = perm ? perm[pbeg + lane] : pbeg + lane;
            nx = px[i];
            ny = py[i];
            nz = pz[i];
            if (strengths) ns = strengths[pid[i]];
        }
        for (int pos = pbeg; pos < pend; pos += kChunk) {
            const int cnt = min(kChunk, pend - pos);
            const double cx = nx, cy = ny, cz = nz, cs = ns;
            if (pos + kChunk + lane < pend) {
                const int i = perm ? perm[pos + kChunk + lane] : pos + kChunk + lane;
                nx = px[i];
                ny = py[i];
                nz = pz[i];
                if (strengths) ns = strengths[pid[i]];
            }
            ring_weights<W>(st, tab, poly, lane, cnt, cx, cy, cz, cs, h, rh, beta, n);
            int j = 0;
            while (j < cnt) {
                if (pos + j >= cell_end) {   // plane k leaves the ring
                    ring_flush_slot<W>(acc, k % W, lane, qbase, ix, iy, n, k % n, grid);
                    ++k;
                    cell_end = cbt[k - k0 + 1];
                    continue;
                }
                const int jend = min(cnt, cell_end - pos);
                for (; j < jend; ++j) {
                    double f[NP];
#pragma unroll
                    for (int t = 0; t < NP; ++t) f[t] = st.wx[j][pa[t]] * st.wy[j][pb[t]];
#pragma unroll
                    for (int s = 0; s < W; ++s) {
                        const double zw = st.wz[j][s];
#pragma unroll
                        for (int t = 0; t < NP; ++t) acc[t][s] = fma(f[t], zw, acc[t][s]);
                    }
                }
            }
            __syncwarp();
        }
        for (; k < k1; ++k) ring_flush_slot<W>(acc, k % W, lane, qbase, ix, iy, n, k % n, grid);
        // planes k1 .. k1 + W - 2 are still in the ring
        for (int pl = k1; pl < k1 + W - 1; ++pl)
            ring_flush_slot<W>(acc, pl % W, lane, qbase, ix, iy, n, pl % n, grid);
    }
}

// Gather (+ push) for wide windows.  A warp walks its work item once per
// field component d: the lane-owned (a, b) pairs hold a ring of w z-slots of
// E_d in registers for the whole item (loaded for the first cell, one plane
// swapped per cell step); per particle a lane forms
// sum_t wx[a_t] wy[b_t] sum_s E_d[t][s] wz[s], the 32 lane partials are reduced
// per particle through shared memory and E_d goes to a per-position scratch
// (L2-resident; added to by each sub-warp when G > 1).  A last walk pushes every
// particle exactly as interp_mma_kernel does (for G > 1 in ring_push_kernel,
// after all sub-warps are done).  Window weights are recomputed per component walk.
template <int W>
struct RingGather {
    double red[kChunk][kChunk + 1];   // [particle][lane] partial sums
};

template <int W>
__device__ __forceinline__ void ring_load_plane(double (&g)[RingSplit<W>::NP][W], int slot,
                                                const double4 *field, int comp, int lane,
                                                int qbase, int ix, int iy, int n, int64_t z) {
    constexpr int NP = RingSplit<W>::NP;
#pragma unroll
    for (int s = 0; s < W; ++s) {
        if (s == slot) {
#pragma unroll
            for (int t = 0; t < NP; ++t) {
                const int qq = qbase + lane + 32 * t;
                double v = 0.0;
                if (qq < W * W) {
                    const int a = qq / W, b = qq - (qq / W) * W;
                    const double *f = reinterpret_cast<const double *>(
                        field + ((int64_t)((ix + a) % n) * n + (iy + b) % n) * n + z);
                    v = __ldg(f + comp);
                }
                g[t][s] = v;
            }
        }
    }
}

// push of the particle at cell-order position pos with its gathered E
template <bool PUSH>
__device__ __forceinline__ void ring_push_one(const pif_soa_t &P, const int32_t *perm,
                                              const pif_soa_t &Q, const PushParams &pp, int64_t pos,
                                              double E0, double E1, double E2, int32_t *key,
                                              int32_t *rank, int32_t *count, double *E_out,
                                              double (&dg)[5]) {
    const int64_t i = perm ? perm[pos] : pos;
    if (PUSH) {
        double x = P.x[i], y = P.y[i], z = P.z[i];
        double vx = P.vx[i], vy = P.vy[i], vz = P.vz[i];
        const int64_t id = P.id[i];
        boris_one(pp, E0, E1, E2, x, y, z, vx, vy, vz, dg);
        Q.x[pos] = x; Q.y[pos] = y; Q.z[pos] = z;
        Q.vx[pos] = vx; Q.vy[pos] = vy; Q.vz[pos] = vz;
        Q.id[pos] = id;
        mirror_store(pp, id, x, y, z, vx, vy, vz);
        const int kk = cell_key(x, y, z, pp.h, pp.rh, pp.w, pp.n);
        key[pos] = kk;
        if (rank) rank[pos] = atomicAdd(&count[kk], 1);
        else atomicAdd(&count[kk], 1);
    } else {
        const int64_t o = 3 * P.id[i];
        E_out[o] = E0;
        E_out[o + 1] = E1;
        E_out[o + 2] = E2;
    }
}

template <int W, bool PUSH>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
interp_ring_kernel(pif_soa_t P, const int32_t *__restrict__ perm, pif_soa_t Q,
                   const int32_t *__restrict__ cell_start, const double4 *__restrict__ field,
                   int seg, int nseg, double beta, const EsPoly poly, PushParams pp,
                   int32_t *__restrict__ key, int32_t *__restrict__ rank,
                   int32_t *__restrict__ count, double *__restrict__ partials,
                   double *__restrict__ E_out, double *__restrict__ scratch, unsigned int *work,
                   const int2 *__restrict__ items, const int *__restrict__ n_items) {
    constexpr int NP = RingSplit<W>::NP, G = RingSplit<W>::G;
    const int nunits = *n_items * G;
    extern __shared__ double4 ring_smem[];
    RingStage<W> *stages = reinterpret_cast<RingStage<W> *>(ring_smem);
    RingGather<W> *gathers = reinterpret_cast<RingGather<W> *>(stages + kWarpsPerBlock);
    __shared__ double tab[32];
    __shared__ int seg_cells[kWarpsPerBlock][kMaxSeg + 1];   // the item's cell boundaries
    if (threadIdx.x < 32) tab[threadIdx.x] = kExp2Table[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    RingStage<W> &st = stages[threadIdx.x >> 5];
    RingGather<W> &rg = gathers[threadIdx.x >> 5];
    int *cbt = seg_cells[threadIdx.x >> 5];
    const int n = pp.n;
    const double h = pp.h;
    const int64_t M = P.count;
    double dg[5] = {0.0, 0.0, 0.0, 0.0, 0.0};

    for (;;) {
        int unit = 0;
        if (lane == 0) unit = (int)atomicAdd(work, 1u);
        unit = __shfl_sync(kFull, unit, 0);
        if (unit >= nunits) break;
        const int item = unit / G, qbase = (unit - item * G) * 32 * NP;
        int pa[NP], pb[NP];
#pragma unroll
        for (int t = 0; t < NP; ++t) {
            const int qq = qbase + lane + 32 * t;
            pa[t] = qq < W * W ? qq / W : 0;
            pb[t] = qq < W * W ? qq % W : 0;
        }
        const int2 it = items[item];
        const int col = it.x / nseg, sg = it.x - col * nseg;
        const int ix = col / n, iy = col - ix * n;
        const int k0 = sg * seg, k1 = min(k0 + seg, n);
        const int base = col * n;
        __syncwarp();   // the previous item is done with the cell table
        for (int c = lane; c <= k1 - k0; c += 32) cbt[c] = cell_start[base + k0 + c];
        __syncwarp();
        const int pbeg = cbt[0] + it.y * kItemParticles;
        const int pend = min(pbeg + kItemParticles, cbt[k1 - k0]);
        int kf = k0;
        while (cbt[kf - k0 + 1] <= pbeg) ++kf;

#pragma unroll 1
        for (int d = 0; d < 3; ++d) {
            double g[NP][W];
            int k = kf;
#pragma unroll
            for (int s = 0; s < W; ++s) {   // planes k .. k + W - 1 of the first cell
                const int pl = k + ((s - k % W + W) % W);
                ring_load_plane<W>(g, s, field, d, lane, qbase, ix, iy, n, pl % n);
            }
            int cell_end = cbt[k - k0 + 1];
            double nx = 0.0, ny = 0.0, nz = 0.0;
            if (pbeg + lane < pend) {
                const int i = perm ? perm[pbeg + lane] : pbeg + lane;
                nx = P.x[i]; ny = P.y[i]; nz = P.z[i];
            }
            for (int pos = pbeg; pos < pend; pos += kChunk) {
                const int cnt = min(kChunk, pend - pos);
                const double x0 = nx, y0 = ny, z0 = nz;
                if (pos + kChunk + lane < pend) {
                    const int i = perm ? perm[pos + kChunk + lane] : pos + kChunk + lane;
                    nx = P.x[i]; ny = P.y[i]; nz = P.z[i];
                }
                ring_weights<W>(st, tab, poly, lane, cnt, x0, y0, z0, 1.0, h, pp.rh, beta, n);
                for (int j = 0; j < cnt; ++j) {
                    while (pos + j >= cell_end) {   // next cell: plane k leaves, k + W enters
                        ring_load_plane<W>(g, k % W, field, d, lane, qbase, ix, iy, n,
                                           (k + W) % n);
                        ++k;
                        cell_end = cbt[k - k0 + 1];
                    }
                    double part = 0.0;
#pragma unroll
                    for (int t = 0; t < NP; ++t) {
                        double inner = 0.0;
#pragma unroll
                        for (int s = 0; s < W; ++s) inner = fma(g[t][s], st.wz[j][s], inner);
                        part = fma(st.wx[j][pa[t]] * st.wy[j][pb[t]], inner, part);
                    }
                    rg.red[j][lane] = part;
                }
                __syncwarp();
                if (lane < cnt) {
                    double e = 0.0;
#pragma unroll 8
                    for (int l = 0; l < 32; ++l) e += rg.red[lane][l];
                    if (G == 1) scratch[d * M + pos + lane] = e;
                    else atomicAdd(&scratch[d * M + pos + lane], e);   // two or three adds
                }
                __syncwarp();
            }
        }
        if (G == 1) {   // push walk (the lane reads back its own scratch entries)
            for (int pos = pbeg + lane; pos < pend; pos += 32)
                ring_push_one<PUSH>(P, perm, Q, pp, pos, scratch[pos], scratch[M + pos],
                                    scratch[2 * M + pos], key, rank, count, E_out, dg);
            __syncwarp();
        }
    }
    if (PUSH && G == 1) block_diag_store(dg, partials);
}

// push (or E output) of every position after a split (G > 1) ring gather
template <bool PUSH>
__global__ void ring_push_kernel(pif_soa_t P, const int32_t *__restrict__ perm, pif_soa_t Q,
                                 PushParams pp, int32_t *__restrict__ key,
                                 int32_t *__restrict__ rank, int32_t *__restrict__ count,
                                 double *__restrict__ partials, double *__restrict__ E_out,
                                 const double *__restrict__ scratch) {
    const int64_t M = P.count;
    double dg[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < M;
         pos += (int64_t)gridDim.x * blockDim.x)
        ring_push_one<PUSH>(P, perm, Q, pp, pos, scratch[pos], scratch[M + pos],
                            scratch[2 * M + pos], key, rank, count, E_out, dg);
    if (PUSH) block_diag_store(dg, partials);
}

// Boris push of id-ordered (M,3) host-layout rows in place, with the E rows a
// split gather wrote (pif_interp_split): the push phase of
// interp_mma_kernel<PUSH> (same boris_one, same wrap of the loaded positions
// as load_aos_kernel) as a coalesced streaming pass over rows [r0, r1), for
// host-streamed stepping (PifEngine.run_host): the next step rebins from the
// downloaded rows, so no cell keys, counts or SoA copy are written, and each
// chunk of rows can be downloaded as soon as its launch ends.
__global__ void __launch_bounds__(256)
push_ids_kernel(double *__restrict__ xa, double *__restrict__ va,
                const double *__restrict__ Ea, int64_t r0, int64_t r1, PushParams pp,
                double *__restrict__ partials) {
    double dg[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    const double L = pp.L;
    for (int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r1;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = 3 * r;
        double x = wrap_coord(xa[o], L), y = wrap_coord(xa[o + 1], L),
               z = wrap_coord(xa[o + 2], L);
        double vx = va[o], vy = va[o + 1], vz = va[o + 2];
        boris_one(pp, Ea[o], Ea[o + 1], Ea[o + 2], x, y, z, vx, vy, vz, dg);
        xa[o] = x; xa[o + 1] = y; xa[o + 2] = z;
        va[o] = vx; va[o + 1] = vy; va[o + 2] = vz;
    }
    block_diag_store(dg, partials);
}

// ----------------------------------------------------------------------------
// generic one-thread-per-particle kernels (any w <= kMaxW)
// ----------------------------------------------------------------------------

__device__ __forceinline__ int axis_stencil(double xv, double h, int w, double beta, int n,
                                            double *wt, int *idx) {
    const double c = axis_coord(xv, h, __drcp_rn(h));
    const double i0 = stencil_start(c, w);
    const double inv_half = 2.0 / w;
    for (int a = 0; a < w; ++a) {
        wt[a] = es_weight(c, i0 + a, inv_half, beta);
        idx[a] = pmod((int)i0 + a, n);
    }
    return (int)i0;
}

__global__ void spread_generic_kernel(pif_soa_t P, const double *__restrict__ strengths, double q,
                                      double *__restrict__ grid, int n, int w, double h,
                                      double beta) {
    double wx[kMaxW], wy[kMaxW], wz[kMaxW];
    int ixs[kMaxW], iys[kMaxW], izs[kMaxW];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P.count;
         i += (int64_t)gridDim.x * blockDim.x) {
        axis_stencil(P.x[i], h, w, beta, n, wx, ixs);
        axis_stencil(P.y[i], h, w, beta, n, wy, iys);
        axis_stencil(P.z[i], h, w, beta, n, wz, izs);
        const double s = strengths ? strengths[P.id[i]] : q;
        for (int a = 0; a < w; ++a) {
            const double sa = __dmul_rn(s, wx[a]);
            for (int b = 0; b < w; ++b) {
                const double sab = __dmul_rn(sa, wy[b]);
                double *row = grid + ((int64_t)ixs[a] * n + iys[b]) * n;
                for (int c = 0; c < w; ++c) atomicAdd(row + izs[c], __dmul_rn(sab, wz[c]));
            }
        }
    }
}

__global__ void interp_generic_kernel(pif_soa_t P, const int32_t *__restrict__ perm, pif_soa_t Q,
                                      const double4 *__restrict__ field, double beta,
                                      PushParams pp, int push, int32_t *__restrict__ key,
                                      int32_t *__restrict__ rank, int32_t *__restrict__ count,
                                      double *__restrict__ partials, double *__restrict__ E_out) {
    double wx[kMaxW], wy[kMaxW], wz[kMaxW];
    int ixs[kMaxW], iys[kMaxW], izs[kMaxW];
    const int n = pp.n, w = pp.w;
    double dg[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P.count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src = perm ? perm[i] : i;   // read in cell order, write at i
        axis_stencil(P.x[src], pp.h, w, beta, n, wx, ixs);
        axis_stencil(P.y[src], pp.h, w, beta, n, wy, iys);
        axis_stencil(P.z[src], pp.h, w, beta, n, wz, izs);
        double l0[kMaxW], l1[kMaxW], l2[kMaxW];
        for (int c = 0; c < w; ++c) l0[c] = l1[c] = l2[c] = 0.0;
        for (int a = 0; a < w; ++a)
            for (int b = 0; b < w; ++b) {
                const double wab = __dmul_rn(wx[a], wy[b]);
                const double4 *row = field + ((int64_t)ixs[a] * n + iys[b]) * n;
                for (int c = 0; c < w; ++c) {
                    const double4 g = row[izs[c]];
                    l0[c] = __dadd_rn(l0[c], __dmul_rn(g.x, wab));
                    l1[c] = __dadd_rn(l1[c], __dmul_rn(g.y, wab));
                    l2[c] = __dadd_rn(l2[c], __dmul_rn(g.z, wab));
                }
            }
        double e0 = 0.0, e1 = 0.0, e2 = 0.0;
        for (int c = 0; c < w; ++c) {
            e0 = __dadd_rn(e0, __dmul_rn(l0[c], wz[c]));
            e1 = __dadd_rn(e1, __dmul_rn(l1[c], wz[c]));
            e2 = __dadd_rn(e2, __dmul_rn(l2[c], wz[c]));
        }
        if (push) {
            double x = P.x[src], y = P.y[src], z = P.z[src];
            double vx = P.vx[src], vy = P.vy[src], vz = P.vz[src];
            const int64_t id = P.id[src];
            boris_one(pp, e0, e1, e2, x, y, z, vx, vy, vz, dg);
            Q.x[i] = x; Q.y[i] = y; Q.z[i] = z;
            Q.vx[i] = vx; Q.vy[i] = vy; Q.vz[i] = vz;
            Q.id[i] = id;
            mirror_store(pp, id, x, y, z, vx, vy, vz);
            const int kk = cell_key(x, y, z, pp.h, pp.rh, w, n);
            key[i] = kk;
            if (rank) rank[i] = atomicAdd(&count[kk], 1);
            else atomicAdd(&count[kk], 1);
        } else {
            const int64_t o = 3 * P.id[src];
            E_out[o] = e0;
            E_out[o + 1] = e1;
            E_out[o + 2] = e2;
        }
    }
    if (push) block_diag_store(dg, partials);
}

__global__ void particle_diag_kernel(pif_soa_t P, double L, int e_kind,
                                     double *__restrict__ partials) {
    double dg[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P.count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double vx = P.vx[i], vy = P.vy[i], vz = P.vz[i];
        dg[0] += vx * vx + vy * vy + vz * vz;
        dg[1] += vx;
        dg[2] += vy;
        dg[3] += vz;
        if (e_kind == PIF_EXT_QUADRUPOLE) {
            const double c = L / 2.0;
            const double dx = P.x[i] - c, dy = P.y[i] - c, dz = P.z[i] - c;
            dg[4] += (7.5 / L) * (dx * dx + dy * dy) - (15.0 / L) * (dz * dz);
        }
    }
    block_diag_store(dg, partials);
}

__global__ void finish_diag_kernel(const double *__restrict__ partials, int nblocks,
                                   double *__restrict__ diag) {
    // fixed-order reduction of the per-block sums: one warp per slot
    const int lane = threadIdx.x & 31, slot = threadIdx.x >> 5;
    if (slot >= kDiagSlots) return;
    double s = 0.0;
    if (slot < 5)
        for (int b = lane; b < nblocks; b += 32) s += partials[b * kDiagSlots + slot];
    s = warp_sum(s);
    if (lane == 0) diag[slot] = s;
}

// complex API: spreading / gather on a complex n^3 grid, one thread per point
__global__ void spread_complex_kernel(const double *__restrict__ pts,
                                      const double2 *__restrict__ vals, int64_t M,
                                      double2 *__restrict__ grid, int n, int w, double h,
                                      double beta) {
    double wx[kMaxW], wy[kMaxW], wz[kMaxW];
    int ixs[kMaxW], iys[kMaxW], izs[kMaxW];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        axis_stencil(pts[3 * i], h, w, beta, n, wx, ixs);
        axis_stencil(pts[3 * i + 1], h, w, beta, n, wy, iys);
        axis_stencil(pts[3 * i + 2], h, w, beta, n, wz, izs);
        const double2 s = vals[i];
        for (int a = 0; a < w; ++a) {
            const double ar = __dmul_rn(s.x, wx[a]), ai = __dmul_rn(s.y, wx[a]);
            for (int b = 0; b < w; ++b) {
                const double br = __dmul_rn(ar, wy[b]), bi = __dmul_rn(ai, wy[b]);
                double *row = reinterpret_cast<double *>(grid + ((int64_t)ixs[a] * n + iys[b]) * n);
                for (int c = 0; c < w; ++c) {
                    atomicAdd(row + 2 * izs[c], __dmul_rn(br, wz[c]));
                    atomicAdd(row + 2 * izs[c] + 1, __dmul_rn(bi, wz[c]));
                }
            }
        }
    }
}

__global__ void interp_complex_kernel(const double2 *__restrict__ grid,
                                      const double *__restrict__ pts, int64_t M,
                                      double2 *__restrict__ out, int n, int w, double h,
                                      double beta) {
    double wx[kMaxW], wy[kMaxW], wz[kMaxW];
    int ixs[kMaxW], iys[kMaxW], izs[kMaxW];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        axis_stencil(pts[3 * i], h, w, beta, n, wx, ixs);
        axis_stencil(pts[3 * i + 1], h, w, beta, n, wy, iys);
        axis_stencil(pts[3 * i + 2], h, w, beta, n, wz, izs);
        double ar = 0.0, ai = 0.0;
        for (int a = 0; a < w; ++a)
            for (int b = 0; b < w; ++b) {
                const double wab = __dmul_rn(wx[a], wy[b]);
                const double2 *row = grid + ((int64_t)ixs[a] * n + iys[b]) * n;
                for (int c = 0; c < w; ++c) {
                    const double k = __dmul_rn(wab, wz[c]);
                    const double2 g = row[izs[c]];
                    ar = __dadd_rn(ar, __dmul_rn(g.x, k));
                    ai = __dadd_rn(ai, __dmul_rn(g.y, k));
                }
            }
        out[i] = make_double2(ar, ai);
    }
}

int grid_for(int64_t work, int threads, int sm_count) {
    int64_t b = (work + threads - 1) / threads;
    int64_t cap = (int64_t)sm_count * 32;
    if (b > cap) b = cap;
    return (int)(b < 1 ? 1 : b);
}

template <typename K>
int persistent_blocks(K kernel, int threads, size_t smem, int sm_count) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) !=
            cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    return per_sm * sm_count;
}

// Wide windows (9..14; 8 only when forced, for comparison) take the FMA ring
// kernels: polynomial weights only, so the plan's polynomials must all be valid.
// per-position E scratch of the ring gather (3 x M doubles), grown on demand
int ensure_ring_scratch(Plan &p, int64_t M) {
    if (3 * M <= p.ring_scratch_cap) return PIF_OK;
    if (p.ring_scratch) cudaFree(p.ring_scratch);
    p.ring_scratch = nullptr;
    p.ring_scratch_cap = 0;
    cudaError_t e = cudaMalloc(&p.ring_scratch, sizeof(double) * 3 * M);
    if (e != cudaSuccess) return fail_cuda(e, "ring gather scratch");
    p.ring_scratch_cap = 3 * M;
    return PIF_OK;
}

// Density thresholds of the ring kernels (Plan::ring_spread_min = 0.1,
// ring_gather_min = 0.75 particles per stencil cell).  With segments of up to
// 127 cells and zero planes skipped, the ring spreader beats the
// one-thread-per-particle atomics down to ~0.1 per cell (0.125 per cell:
// 2.3x / 1.9x at w = 13 / 10; at 0.06 and 0.008 per cell walking the empty
// cells makes it 2.4x / 3.1x slower); the ring gather, which reloads a plane per cell
// step, wins from ~1 per cell (1.5x / 2.5x) and loses below (0.5 per cell:
// -6% / -45% at w = 13 / 16; 0.125: -90% / -40% at w = 13 / 10).
// profiles/round2/ring_density_ab.txt

bool ring_path_ok(const Plan &p) {
    if (p.force_generic) return false;
    // w <= kMaxPolyW evaluates interior weights by polynomial (all must pass
    // the plan's accuracy check); wider windows use the exact formula
    if (p.w <= kMaxPolyW && p.poly.exact_mask != 0) return false;
    return (p.w >= 9 && p.w <= kMaxRingW) || (p.force_ring && p.w == 8);
}

// The DMMA kernels cover w <= 8; for w >= kPolyOnlyW they are compiled without
// the exact-weight fallback, so a plan whose polynomials missed the bound there
// (not the case for the reference's beta = 2.30 w) takes the generic kernels.
bool fast_path_ok(const Plan &p) {
    if (p.w > kMaxFastW || p.force_generic || p.force_ring) return false;
    return p.w < kPolyOnlyW || p.poly.exact_mask == 0;
}

PushParams make_push(const Plan &p, double half, double dt, const double *tq, const double *sq,
                     int has_b, int e_kind) {
    PushParams pp;
    pp.half = half;
    pp.dt = dt;
    pp.L = p.L;
    pp.h = p.h;
    pp.rh = 1.0 / p.h;
    pp.ext_c = p.L / 2.0;       // the reference's constants (pif.py:52-57, 66-67)
    pp.ext_xy = -15.0 / p.L;
    pp.ext_z = 30.0 / p.L;
    pp.pot_xy = 7.5 / p.L;
    pp.pot_z = 15.0 / p.L;
    for (int d = 0; d < 3; ++d) {
        pp.tq[d] = tq ? tq[d] : 0.0;
        pp.sq[d] = sq ? sq[d] : 0.0;
    }
    pp.has_b = has_b;
    pp.e_kind = e_kind;
    pp.n = p.n;
    pp.w = p.w;
    pp.mx = p.mirror_x;
    pp.mv = p.mirror_v;
    pp.mid0 = p.mirror_id0;
    pp.eslot = nullptr;
    return pp;
}

}  // namespace

// ============================================================================
// launchers
// ============================================================================

bool det_supported(const Plan &p) { return fast_path_ok(p); }

int launch_wrap(Plan &p, double *x, double *y, double *z, int64_t M, cudaStream_t s) {
    p.wcache_valid = false;
    if (M == 0) return PIF_OK;
    wrap_kernel<<<grid_for(M, 256, p.sm_count), 256, 0, s>>>(x, y, z, M, p.L);
    return fail_cuda(cudaGetLastError(), "wrap_kernel");
}

int launch_bin_keys(Plan &p, const pif_soa_t &src, int32_t *key, int32_t *rank, cudaStream_t s) {
    if (src.count == 0) return PIF_OK;
    bin_keys_kernel<<<grid_for(src.count, 256, p.sm_count), 256, 0, s>>>(
        src.x, src.y, src.z, src.count, p.h, p.w, p.n, key, rank, p.cell_count);
    return fail_cuda(cudaGetLastError(), "bin_keys_kernel");
}

int launch_bin_scatter(Plan &p, const pif_soa_t &src, pif_soa_t &dst, const int32_t *key,
                       const int32_t *rank, bool vel, cudaStream_t s) {
    p.wcache_valid = false;
    size_t tmp = p.scan_tmp_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(p.scan_tmp, tmp, p.cell_count, p.cell_start,
                                                  (int)(p.n3 + 1), s);
    if (e != cudaSuccess) return fail_cuda(e, "cell scan");
    if (src.count > 0) {
        bin_scatter_kernel<<<grid_for(src.count, 256, p.sm_count), 256, 0, s>>>(
            src, dst, key, rank, p.cell_start, vel ? 1 : 0);
        e = cudaGetLastError();
        if (e != cudaSuccess) return fail_cuda(e, "bin_scatter_kernel");
    }
    dst.count = src.count;
    const int rc = build_items(p, src.count, s);
    if (rc != PIF_OK) return rc;
    return fail_cuda(cudaMemsetAsync(p.cell_count, 0, sizeof(int32_t) * (p.n3 + 1), s),
                     "reset cell counts");
}

static EsPoly device_poly(const Plan &p) {
    static_assert(sizeof(EsPoly) == sizeof(EsPolyHost), "EsPoly layout");
    static_assert(kEsDeg == kEsDegHost, "EsPoly degree");
    EsPoly e;
    std::memcpy(&e, &p.poly, sizeof(e));
    return e;
}

// Cells per z-segment work item: 16 at the benchmark density (64 particles per
// stencil cell); sparser sets get longer segments (up to kMaxSeg; the gathers
// keep an item's cell boundaries in shared memory) so an item still holds
// ~seg_target particles and the per-item window / first-chunk loads stay
// amortised.
int segment_cells(const Plan &p, int64_t M) {
    const double per_cell = (double)M / (double)p.n3;
    const double want = (double)p.seg_target / (per_cell > 1.0 ? per_cell : 1.0);
    const int seg = (int)std::ceil(want);
    return seg < 8 ? 8 : (seg > kMaxSeg ? kMaxSeg : seg);
}

int build_items(Plan &p, int64_t M, cudaStream_t s) {
    p.density = (double)M / (double)p.n3;
    p.seg = segment_cells(p, M);
    p.n_segs = p.n * p.n * ((p.n + p.seg - 1) / p.seg);
    const int64_t need = p.n_segs + M / kItemParticles + 1;
    if (need > p.items_cap) {
        if (p.items) cudaFree(p.items);
        p.items = nullptr;
        cudaError_t e = cudaMalloc(&p.items, sizeof(int2) * need);
        if (e != cudaSuccess) return fail_cuda(e, "work item table");
        p.items_cap = need;
    }
    const int nseg = (p.n + p.seg - 1) / p.seg;
    seg_parts_kernel<<<grid_for(p.n_segs + 1, 256, p.sm_count), 256, 0, s>>>(
        p.cell_start, p.n, p.seg, nseg, p.n_segs, p.seg_parts);
    size_t tmp = p.scan_tmp_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(p.scan_tmp, tmp, p.seg_parts, p.seg_off,
                                                  p.n_segs + 1, s);
    if (e != cudaSuccess) return fail_cuda(e, "segment scan");
    seg_items_kernel<<<grid_for(p.n_segs, 256, p.sm_count), 256, 0, s>>>(p.seg_parts, p.seg_off,
                                                                         p.n_segs, p.items);
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail_cuda(e, "work item kernels");
    if (p.push_agg_force >= 0) {
        p.push_agg = p.push_agg_force != 0;
    } else if (p.agg_check) {
        // once per particle set, outside graph capture: the most parts any
        // segment holds (Landau 64^3 / 2^27: 2; Penning 2^28 on one GPU: dozens)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        e = cudaStreamIsCapturing(s, &cs);
        if (e != cudaSuccess) return fail_cuda(e, "capture status");
        if (cs == cudaStreamCaptureStatusNone) {
            // the value reaches the host through mapped pinned memory (a
            // kernel store), not a D2H copy: a copy would queue behind
            // whatever the copy engine is streaming (run_host: the previous
            // step's velocities, ~55 ms)
            if (!p.max_parts_host) {
                e = cudaHostAlloc(reinterpret_cast<void **>(&p.max_parts_host), sizeof(int),
                                  cudaHostAllocMapped);
                if (e != cudaSuccess) return fail_cuda(e, "mapped host word");
            }
            int *mapped = nullptr;
            e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&mapped), p.max_parts_host, 0);
            if (e == cudaSuccess) e = cudaMemsetAsync(p.max_parts, 0, sizeof(int), s);
            if (e == cudaSuccess) {
                max_parts_kernel<<<grid_for(p.n_segs, 256, p.sm_count), 256, 0, s>>>(
                    p.seg_parts, p.n_segs, p.max_parts);
                publish_int_kernel<<<1, 1, 0, s>>>(p.max_parts, mapped);
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) return fail_cuda(e, "max parts per segment");
            p.push_agg = *reinterpret_cast<volatile int *>(p.max_parts_host) >= kPushAggMinParts;
            p.agg_check = false;
        }
    }
    return PIF_OK;
}

// dst[slot] = src[perm[slot]] (what: PIF_PERMUTE_POSITIONS x, y, z, id;
// PIF_PERMUTE_VELOCITIES vx, vy, vz; PIF_PERMUTE_RESET then perm[slot] = slot).
// A set loaded in id order from host memory is spatially random, and the
// kernels reading it through perm would gather 8-byte words at random with
// few warps in flight; one streaming pass with full occupancy puts it in
// cell order instead (random reads, coalesced writes).
__global__ void permute_kernel(pif_soa_t src, int32_t *__restrict__ perm, pif_soa_t dst, int what) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dst.count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = perm[i];
        if (what & PIF_PERMUTE_POSITIONS) {
            const double x = src.x[j], y = src.y[j], z = src.z[j];
            const int64_t id = src.id[j];
            dst.x[i] = x;
            dst.y[i] = y;
            dst.z[i] = z;
            dst.id[i] = id;
        }
        if (what & PIF_PERMUTE_VELOCITIES) {
            const double vx = src.vx[j], vy = src.vy[j], vz = src.vz[j];
            dst.vx[i] = vx;
            dst.vy[i] = vy;
            dst.vz[i] = vz;
        }
        if (what & PIF_PERMUTE_RESET) perm[i] = (int32_t)i;
    }
}

int launch_permute(Plan &p, const pif_soa_t &src, int32_t *perm, pif_soa_t &dst, int what,
                   cudaStream_t s) {
    if (dst.count == 0) return PIF_OK;
    permute_kernel<<<grid_for(dst.count, 256, p.sm_count), 256, 0, s>>>(src, perm, dst, what);
    return fail_cuda(cudaGetLastError(), "permute_kernel");
}

int launch_soa_to_aos(Plan &p, const pif_soa_t &P, int64_t id0, double *ox, double *ov,
                      cudaStream_t s) {
    if (P.count == 0) return PIF_OK;
    soa_to_aos_by_id_kernel<<<grid_for(P.count, 256, p.sm_count), 256, 0, s>>>(P, id0, ox, ov);
    return fail_cuda(cudaGetLastError(), "soa_to_aos_by_id_kernel");
}

int debug_phase_cycles(unsigned long long *out) {
#ifdef PIF_PHASE_TIMING
    cudaError_t e = cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 8);
    if (e == cudaSuccess) {
        unsigned long long z[8] = {0};
        e = cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
    }
    return fail_cuda(e, "phase counters");
#else
    (void)out;
    set_error("built without PIF_PHASE_TIMING");
    return PIF_ERR_STATE;
#endif
}

int launch_load_velocities(Plan &p, const double *v, pif_soa_t &dst, cudaStream_t s) {
    if (dst.count == 0) return PIF_OK;
    load_vel_kernel<<<grid_for(dst.count, 256, p.sm_count), 256, 0, s>>>(v, p.aos_id0, dst.count,
                                                                        dst);
    return fail_cuda(cudaGetLastError(), "load_vel_kernel");
}

int launch_load_aos(Plan &p, const double *x, const double *v, int64_t id0, pif_soa_t &dst,
                    int32_t *key, int32_t *rank, cudaStream_t s) {
    p.wcache_valid = false;
    p.aos_id0 = id0;
    if (dst.count == 0) return PIF_OK;
    load_aos_kernel<<<grid_for(dst.count, 256, p.sm_count), 256, 0, s>>>(
        x, v, id0, dst.count, dst, p.L, p.h, p.w, p.n, key, rank, p.cell_count);
    return fail_cuda(cudaGetLastError(), "load_aos_kernel");
}

__global__ void iota_kernel(int32_t *out, int64_t M) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)i;
}

// perm = stable argsort of the cell keys (CUB LSD radix sort is stable)
int det_sort_perm(Plan &p, const int32_t *key, int64_t M, int32_t *perm, cudaStream_t s) {
    int bits = 1;
    while ((int64_t(1) << bits) < p.n3) ++bits;
    size_t tmp = 0;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, p.det_keys, p.det_iota, perm,
                                                    (int)M, 0, bits, s);
    if (e != cudaSuccess) return fail_cuda(e, "radix sort size");
    if (M > p.det_cap || tmp > p.det_tmp_bytes) {
        cudaFree(p.det_keys);
        cudaFree(p.det_iota);
        cudaFree(p.det_tmp);
        p.det_keys = nullptr;
        p.det_iota = nullptr;
        p.det_tmp = nullptr;
        p.det_cap = 0;
        p.det_tmp_bytes = 0;
        e = cudaMalloc(&p.det_keys, sizeof(int32_t) * M);
        if (e == cudaSuccess) e = cudaMalloc(&p.det_iota, sizeof(int32_t) * M);
        if (e == cudaSuccess) e = cudaMalloc(&p.det_tmp, tmp);
        if (e != cudaSuccess) return fail_cuda(e, "deterministic binning scratch");
        p.det_cap = M;
        p.det_tmp_bytes = tmp;
    }
    iota_kernel<<<grid_for(M, 256, p.sm_count), 256, 0, s>>>(p.det_iota, M);
    tmp = p.det_tmp_bytes;
    e = cub::DeviceRadixSort::SortPairs(p.det_tmp, tmp, key, p.det_keys, p.det_iota, perm, (int)M,
                                        0, bits, s);
    return fail_cuda(e, "radix sort");
}

int launch_bin_perm(Plan &p, const int32_t *key, const int32_t *rank, int64_t M, int32_t *perm,
                    cudaStream_t s) {
    p.wcache_valid = false;
    size_t tmp = p.scan_tmp_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(p.scan_tmp, tmp, p.cell_count, p.cell_start,
                                                  (int)(p.n3 + 1), s);
    if (e != cudaSuccess) return fail_cuda(e, "cell scan");
    if (M > 0 && p.det) {
        // stable binning: perm = indices sorted by key, ties in index order
        // (the atomic ranks would order a cell's particles by arrival)
        const int rc = det_sort_perm(p, key, M, perm, s);
        if (rc != PIF_OK) return rc;
    } else if (M > 0 && rank) {
        bin_perm_kernel<<<grid_for(M, 256, p.sm_count), 256, 0, s>>>(key, rank, p.cell_start, M,
                                                                      perm);
        e = cudaGetLastError();
        if (e != cudaSuccess) return fail_cuda(e, "bin_perm_kernel");
    } else if (M > 0) {
        e = cudaMemsetAsync(p.cell_count, 0, sizeof(int32_t) * (p.n3 + 1), s);
        if (e != cudaSuccess) return fail_cuda(e, "reset cell cursors");
        bin_perm_cursor_kernel<<<grid_for((M + kPermUnroll - 1) / kPermUnroll, 256, p.sm_count),
                                 256, 0, s>>>(
            key, p.cell_count, p.cell_start, M, perm);
        e = cudaGetLastError();
        if (e != cudaSuccess) return fail_cuda(e, "bin_perm_cursor_kernel");
    }
    const int rc = build_items(p, M, s);
    if (rc != PIF_OK) return rc;
    return fail_cuda(cudaMemsetAsync(p.cell_count, 0, sizeof(int32_t) * (p.n3 + 1), s),
                     "reset cell counts");
}

// Merged-column spread (spread_merged_kernel) below these densities
// (particles per stencil cell) when the weight cache is off: C = 4, then
// C = 2; above, the column kernel (256^3 / 1.25 per cell: spread 59.4 ms ->
// 43.1 (C = 2) -> 33.6 (C = 4); profiles/round2/spread_merge_ab.txt).
#ifndef PIF_MERGE4_BELOW
#define PIF_MERGE4_BELOW 3.0
#endif
#ifndef PIF_MERGE2_BELOW
#define PIF_MERGE2_BELOW 12.0
#endif

int merged_factor(const Plan &p) {
    if (p.det || p.n < 32 || p.w < 6 || !fast_path_ok(p)) return 1;
    if (p.merge_force >= 0) return p.merge_force >= 2 ? p.merge_force : 1;
    // the merged order cannot feed the gather's weight cache (its slots are in
    // the column order), and from 4 per cell the cache is worth more (128^3 /
    // 8 per cell: spread -1.0 ms merged, gather +1.9 ms without the cache)
    if (p.wcache_on) return 1;
    // heavy cells (the push_agg decision: some segment holds >= 12 work
    // items): the merged walk only adds DMMAs there (clustered 64^3 / 2^24:
    // 1.21 -> 1.87 ms merged; profiles/round2/microbench_merge_ab.md)
    if (p.push_agg) return 1;
    if (p.density < PIF_MERGE4_BELOW) return 4;
    if (p.density < PIF_MERGE2_BELOW) return 2;
    return 1;
}

template <typename T>
int grow(T **ptr, int64_t &cap, int64_t need, const char *what) {
    if (need <= cap) return PIF_OK;
    if (*ptr) cudaFree(*ptr);
    *ptr = nullptr;
    cap = 0;
    const cudaError_t e = cudaMalloc(reinterpret_cast<void **>(ptr), sizeof(T) * need);
    if (e != cudaSuccess) return fail_cuda(e, what);
    cap = need;
    return PIF_OK;
}

// super-column cell order, perm and work items from the standard binning
// (p.cell_start of perm); returns the merged segment length / count
int build_merged(Plan &p, const pif_soa_t &P, const int32_t *perm, int C, int &seg, int &nseg,
                 int &nsegs, cudaStream_t s) {
    const int64_t n3 = p.n3, M = P.count;
    if (!p.cell_start2) {
        const cudaError_t e =
            cudaMalloc(reinterpret_cast<void **>(&p.cell_start2), sizeof(int32_t) * 2 * (n3 + 1));
        if (e != cudaSuccess) return fail_cuda(e, "merged cell table");
    }
    int32_t *count2 = p.cell_start2, *cs2 = p.cell_start2 + (n3 + 1);
    if (grow(&p.perm2, p.perm2_cap, M, "merged perm") != PIF_OK) return PIF_ERR_CUDA;
    merged_counts_kernel<<<grid_for(n3 + 1, 256, p.sm_count), 256, 0, s>>>(p.cell_start, p.n, C,
                                                                           count2);
    size_t tmp = p.scan_tmp_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(p.scan_tmp, tmp, count2, cs2, (int)(n3 + 1), s);
    if (e != cudaSuccess) return fail_cuda(e, "merged cell scan");
    merged_perm_kernel<<<grid_for(n3, 256, p.sm_count), 256, 0, s>>>(perm, p.cell_start, cs2, p.n,
                                                                    C, p.perm2);
    // segments of seg levels holding ~seg_target particles, as segment_cells
    const double per_level = p.density * C;
    seg = (int)std::ceil((double)p.seg_target / (per_level > 1.0 ? per_level : 1.0));
    seg = seg < 8 ? 8 : (seg > kMaxSeg ? kMaxSeg : seg);
    nseg = (p.n + seg - 1) / seg;
    nsegs = (p.n / C) * p.n * nseg;
    if (p.segs2_cap < (int64_t)nsegs + 1) {
        if (p.seg_parts2) cudaFree(p.seg_parts2);
        if (p.seg_off2) cudaFree(p.seg_off2);
        p.seg_parts2 = p.seg_off2 = nullptr;
        p.segs2_cap = 0;
        e = cudaMalloc(reinterpret_cast<void **>(&p.seg_parts2), sizeof(int) * (nsegs + 1));
        if (e == cudaSuccess)
            e = cudaMalloc(reinterpret_cast<void **>(&p.seg_off2), sizeof(int) * (nsegs + 1));
        if (e != cudaSuccess) return fail_cuda(e, "merged segment tables");
        p.segs2_cap = nsegs + 1;
    }
    if (grow(&p.items2, p.items2_cap, (int64_t)nsegs + M / kItemParticles + 1,
             "merged work items") != PIF_OK)
        return PIF_ERR_CUDA;
    merged_seg_parts_kernel<<<grid_for(nsegs + 1, 256, p.sm_count), 256, 0, s>>>(
        cs2, p.n, C, seg, nseg, nsegs, p.seg_parts2);
    tmp = p.scan_tmp_bytes;
    e = cub::DeviceScan::ExclusiveSum(p.scan_tmp, tmp, p.seg_parts2, p.seg_off2, nsegs + 1, s);
    if (e != cudaSuccess) return fail_cuda(e, "merged segment scan");
    seg_items_kernel<<<grid_for(nsegs, 256, p.sm_count), 256, 0, s>>>(p.seg_parts2, p.seg_off2,
                                                                      nsegs, p.items2);
    return fail_cuda(cudaGetLastError(), "merged binning kernels");
}

int launch_spread_merged(Plan &p, const pif_soa_t &P, const int32_t *perm,
                         const double *strengths, double q, int C, cudaStream_t s) {
    int seg = 0, nseg = 0, nsegs = 0;
    int rc = build_merged(p, P, perm, C, seg, nseg, nsegs, s);
    if (rc != PIF_OK) return rc;
    cudaError_t e = cudaMemsetAsync(p.work, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess) return fail_cuda(e, "zero work counter");
    const EsPoly poly = device_poly(p);
    const int threads = kWarpsPerBlock * 32;
    const int32_t *cs2 = p.cell_start2 + (p.n3 + 1);
    const int *nitems = p.seg_off2 + nsegs;
#define PIF_MERGED_CASE(W, CC)                                                                 \
    if (p.w == W && C == CC) {                                                                 \
        auto k = spread_merged_kernel<W, CC>;                                                  \
        const int blocks = persistent_blocks(k, threads, 0, p.sm_count);                      \
        k<<<blocks, threads, 0, s>>>(P.x, P.y, P.z, P.id, p.perm2, strengths, q, cs2, p.grid,  \
                                     p.n, seg, nseg, p.h, p.beta, poly, p.work, p.items2,     \
                                     nitems);                                                  \
        return fail_cuda(cudaGetLastError(), "spread_merged_kernel");                          \
    }
    PIF_MERGED_CASE(8, 2)
    PIF_MERGED_CASE(8, 4)
    PIF_MERGED_CASE(7, 2)
    PIF_MERGED_CASE(7, 4)
    PIF_MERGED_CASE(6, 2)
    PIF_MERGED_CASE(6, 4)
#undef PIF_MERGED_CASE
    set_error("merged spread: w = 6..8 and C = 2 or 4 only");
    return PIF_ERR_STATE;
}

int launch_spread(Plan &p, const pif_soa_t &P, const int32_t *perm, const double *strengths,
                  double q, cudaStream_t s) {
    const EsPoly poly = device_poly(p);
    cudaError_t e = cudaMemsetAsync(p.grid, 0, sizeof(double) * p.n3, s);
    if (e != cudaSuccess) return fail_cuda(e, "zero grid");
    if (P.count == 0) return PIF_OK;
    p.wcache_valid = false;
    p.merge_used = 1;
    if (fast_path_ok(p)) {
        const int C = merged_factor(p);
        if (C > 1) {
            p.merge_used = C;
            return launch_spread_merged(p, P, perm, strengths, q, C, s);
        }
        const int nseg = (p.n + p.seg - 1) / p.seg;
        const int *nitems = p.seg_off + p.n_segs;
        e = cudaMemsetAsync(p.work, 0, sizeof(unsigned int), s);
        if (e != cudaSuccess) return fail_cuda(e, "zero work counter");
        const int threads = kWarpsPerBlock * 32;
        // keep this spread's window weights for the gather at the same positions
        double *wc = (!p.det && p.wcache_on && ensure_wcache(p, P.count) == PIF_OK) ? p.wcache
                                                                                : nullptr;
        if (wc) {
            p.wcache_valid = true;
            p.wcache_x = P.x;
            p.wcache_perm = perm;
            p.wcache_count = P.count;
        }
        DetOut det;
        if (p.det) {
            // one slice of (seg + 7) planes x 64 rows per work item, zeroed (an
            // item flushes only the planes from its first non-empty cell on)
            det.stride = p.seg + 7;
            const int64_t need = p.items_cap * 64 * det.stride;
            if (need > p.dbuf_cap) {
                if (p.dbuf) cudaFree(p.dbuf);
                p.dbuf = nullptr;
                p.dbuf_cap = 0;
                e = cudaMalloc(&p.dbuf, sizeof(double) * need);
                if (e != cudaSuccess) return fail_cuda(e, "deterministic plane buffer");
                p.dbuf_cap = need;
            }
            e = cudaMemsetAsync(p.dbuf, 0, sizeof(double) * need, s);
            if (e != cudaSuccess) return fail_cuda(e, "zero plane buffer");
            det.buf = p.dbuf;
            wc = nullptr;
            p.wcache_valid = false;
        }
#define PIF_SPREAD_CASE(W)                                                                   \
    case W: {                                                                                \
        auto k = p.det ? spread_mma_kernel<W, true> : spread_mma_kernel<W, false>;          \
        int blocks = persistent_blocks(k, threads, 0, p.sm_count);                           \
        k<<<blocks, threads, 0, s>>>(P.x, P.y, P.z, P.id, perm, strengths, q, p.cell_start,   \
                                     p.grid,                                                 \
                                     p.n, p.seg, nseg, p.h, p.beta, poly, p.work, p.items,   \
                                     nitems, wc, P.count, det);                              \
        break;                                                                               \
    }
        switch (p.w) {
            PIF_SPREAD_CASE(2)
            PIF_SPREAD_CASE(3)
            PIF_SPREAD_CASE(4)
            PIF_SPREAD_CASE(5)
            PIF_SPREAD_CASE(6)
            PIF_SPREAD_CASE(7)
            PIF_SPREAD_CASE(8)
            default:
                set_error("unsupported window width");
                return PIF_ERR_VALUE;
        }
#undef PIF_SPREAD_CASE
        if (p.det) {
            e = cudaGetLastError();
            if (e != cudaSuccess) return fail_cuda(e, "spread kernel");
            det_reduce_kernel<<<grid_for(p.n3, 256, p.sm_count), 256, 0, s>>>(
                p.dbuf, det.stride, p.seg_off, p.seg_parts, p.n, p.seg, nseg, p.w, p.grid);
        }
    } else if (ring_path_ok(p) && p.density >= p.ring_spread_min) {
        const int nseg = (p.n + p.seg - 1) / p.seg;
        const int *nitems = p.seg_off + p.n_segs;
        e = cudaMemsetAsync(p.work, 0, sizeof(unsigned int), s);
        if (e != cudaSuccess) return fail_cuda(e, "zero work counter");
        const int threads = kWarpsPerBlock * 32;
#define PIF_RING_SPREAD_CASE(W)                                                              \
    case W: {                                                                                \
        auto k = spread_ring_kernel<W>;                                                     \
        const int dyn = (int)(kWarpsPerBlock * sizeof(RingStage<W>));                        \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);           \
        int blocks = persistent_blocks(k, threads, dyn, p.sm_count);                         \
        k<<<blocks, threads, dyn, s>>>(P.x, P.y, P.z, P.id, perm, strengths, q, p.cell_start, \
                                     p.grid, p.n, p.seg, nseg, p.h, p.beta, poly, p.work,     \
                                     p.items, nitems);                                       \
        break;                                                                               \
    }
        switch (p.w) {
            PIF_RING_SPREAD_CASE(8)
            PIF_RING_SPREAD_CASE(9)
            PIF_RING_SPREAD_CASE(10)
            PIF_RING_SPREAD_CASE(11)
            PIF_RING_SPREAD_CASE(12)
            PIF_RING_SPREAD_CASE(13)
            PIF_RING_SPREAD_CASE(14)
            PIF_RING_SPREAD_CASE(15)
            PIF_RING_SPREAD_CASE(16)
            PIF_RING_SPREAD_CASE(17)
            default:
                set_error("unsupported window width");
                return PIF_ERR_VALUE;
        }
#undef PIF_RING_SPREAD_CASE
    } else {
        spread_generic_kernel<<<grid_for(P.count, 128, p.sm_count), 128, 0, s>>>(
            P, strengths, q, p.grid, p.n, p.w, p.h, p.beta);
    }
    return fail_cuda(cudaGetLastError(), "spread kernel");
}

// dynamic shared memory of interp_mma_kernel: the per-warp partial sums (+ the
// second weight stage when the weight cache is in use)
constexpr int kGatherDyn = (int)(kGatherWarps * sizeof(GatherPartials));
constexpr int kGatherDynMax = kGatherDyn + (int)(kGatherWarps * sizeof(WarpChunk));

// spread -> gather window-weight cache, [24][M] doubles, grown on demand
int ensure_wcache(Plan &p, int64_t M) {
    if (24 * M <= p.wcache_cap) return PIF_OK;
    if (p.wcache) cudaFree(p.wcache);
    p.wcache = nullptr;
    p.wcache_cap = 0;
    cudaError_t e = cudaMalloc(&p.wcache, sizeof(double) * 24 * M);
    if (e != cudaSuccess) {
        cudaGetLastError();
        p.wcache_on = false;   // no room: run without the cache
        return PIF_ERR_CUDA;
    }
    p.wcache_cap = 24 * M;
    return PIF_OK;
}

namespace {
int interp_impl(Plan &p, const pif_soa_t &P, const int32_t *perm, pif_soa_t &Q, bool push,
                double half, double dt, const double *tq, const double *sq, int has_b,
                int e_kind, int32_t *key, int32_t *rank, double *diag, double *E_out,
                double *eslot, int64_t eslot_id0, cudaStream_t s) {
    if (!p.field_valid) {
        set_error("no field grid: solve the fields before gathering");
        return PIF_ERR_STATE;
    }
    PushParams pp = make_push(p, half, dt, tq, sq, has_b, e_kind);
    pp.eslot = eslot;
    if (eslot) pp.mid0 = eslot_id0;
    const EsPoly poly = device_poly(p);
    const double4 *field = reinterpret_cast<const double4 *>(p.field);
    cudaError_t e;
    int blocks = 1;
    if (P.count > 0 && fast_path_ok(p)) {
        const int nseg = (p.n + p.seg - 1) / p.seg;
        const int *nitems = p.seg_off + p.n_segs;
        e = cudaMemsetAsync(p.work, 0, sizeof(unsigned int), s);
        if (e != cudaSuccess) return fail_cuda(e, "zero work counter");
        // weights cached by the spread at exactly these particles / this order
        const double *wc = (p.wcache_on && p.wcache_valid && p.wcache_x == P.x &&
                            p.wcache_perm == perm && p.wcache_count == P.count)
                               ? p.wcache
                               : nullptr;
        const size_t dyn = kGatherDyn + (wc ? kGatherWarps * sizeof(WarpChunk) : 0);
        const int gthreads = kGatherWarps * 32;
        const bool longseg = p.seg > 31;
#define PIF_INTERP_CASE(W)                                                                    \
    case W: {                                                                                 \
        if (push) {                                                                           \
            auto k = longseg ? (wc ? interp_mma_kernel<W, true, true, true, false>            \
                                   : interp_mma_kernel<W, true, true, false, false>)          \
                   : p.push_agg ? (wc ? interp_mma_kernel<W, true, false, true, true>          \
                                      : interp_mma_kernel<W, true, false, false, true>)       \
                                : (wc ? interp_mma_kernel<W, true, false, true, false>         \
                                      : interp_mma_kernel<W, true, false, false, false>);     \
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kGatherDynMax); \
            blocks = persistent_blocks(k, gthreads, dyn, p.sm_count);                         \
            if (blocks > p.partial_blocks) blocks = p.partial_blocks;                         \
            k<<<blocks, gthreads, dyn, s>>>(P, perm, Q, p.cell_start, field, p.seg, nseg,     \
                                                  p.beta,                                     \
                                         poly, pp,                                            \
                                         key, rank, p.cell_count, p.partials, E_out, p.work,   \
                                         p.items, nitems, wc, P.count);                       \
        } else {                                                                              \
            auto k = longseg ? (wc ? interp_mma_kernel<W, false, true, true, false>           \
                                   : interp_mma_kernel<W, false, true, false, false>)         \
                             : (wc ? interp_mma_kernel<W, false, false, true, false>          \
                                   : interp_mma_kernel<W, false, false, false, false>);       \
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kGatherDynMax); \
            blocks = persistent_blocks(k, gthreads, dyn, p.sm_count);                         \
            k<<<blocks, gthreads, dyn, s>>>(P, perm, Q, p.cell_start, field, p.seg, nseg,     \
                                                  p.beta,                                     \
                                         poly, pp,                                            \
                                         key, rank, p.cell_count, p.partials, E_out, p.work,   \
                                         p.items, nitems, wc, P.count);                       \
        }                                                                                     \
        break;                                                                                \
    }
        switch (p.w) {
            PIF_INTERP_CASE(2)
            PIF_INTERP_CASE(3)
            PIF_INTERP_CASE(4)
            PIF_INTERP_CASE(5)
            PIF_INTERP_CASE(6)
            PIF_INTERP_CASE(7)
            PIF_INTERP_CASE(8)
            default:
                set_error("unsupported window width");
                return PIF_ERR_VALUE;
        }
#undef PIF_INTERP_CASE
    } else if (eslot && P.count > 0) {
        set_error("split gather: DMMA kernels (w <= 8) only");
        return PIF_ERR_STATE;
    } else if (P.count > 0 && ring_path_ok(p) && p.density >= p.ring_gather_min) {
        const int nseg = (p.n + p.seg - 1) / p.seg;
        const int *nitems = p.seg_off + p.n_segs;
        e = cudaMemsetAsync(p.work, 0, sizeof(unsigned int), s);
        if (e != cudaSuccess) return fail_cuda(e, "zero work counter");
        const int threads = kWarpsPerBlock * 32;
#define PIF_RING_INTERP_CASE(W)                                                               \
    case W: {                                                                                 \
        const size_t dyn = kWarpsPerBlock * (sizeof(RingStage<W>) + sizeof(RingGather<W>));   \
        if (ensure_ring_scratch(p, P.count) != PIF_OK) return PIF_ERR_CUDA;                    \
        constexpr bool split = RingSplit<W>::G > 1;                                           \
        if (split) {   /* sub-warps add their partials into the scratch */                    \
            e = cudaMemsetAsync(p.ring_scratch, 0, sizeof(double) * 3 * P.count, s);          \
            if (e != cudaSuccess) return fail_cuda(e, "zero ring scratch");                    \
        }                                                                                     \
        auto k = push ? interp_ring_kernel<W, true> : interp_ring_kernel<W, false>;           \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);       \
        blocks = persistent_blocks(k, threads, dyn, p.sm_count);                              \
        if (blocks > p.partial_blocks) blocks = p.partial_blocks;                             \
        k<<<blocks, threads, dyn, s>>>(P, perm, Q, p.cell_start, field, p.seg, nseg, p.beta,   \
                                       poly, pp, key, rank, p.cell_count, p.partials, E_out,  \
                                       p.ring_scratch, p.work, p.items, nitems);              \
        if (split) {                                                                          \
            blocks = grid_for(P.count, 128, p.sm_count);                                      \
            if (blocks > p.partial_blocks) blocks = p.partial_blocks;                         \
            auto kp = push ? ring_push_kernel<true> : ring_push_kernel<false>;                \
            kp<<<blocks, 128, 0, s>>>(P, perm, Q, pp, key, rank, p.cell_count, p.partials,    \
                                      E_out, p.ring_scratch);                                 \
        }                                                                                     \
        break;                                                                                \
    }
        switch (p.w) {
            PIF_RING_INTERP_CASE(8)
            PIF_RING_INTERP_CASE(9)
            PIF_RING_INTERP_CASE(10)
            PIF_RING_INTERP_CASE(11)
            PIF_RING_INTERP_CASE(12)
            PIF_RING_INTERP_CASE(13)
            PIF_RING_INTERP_CASE(14)
            PIF_RING_INTERP_CASE(15)
            PIF_RING_INTERP_CASE(16)
            PIF_RING_INTERP_CASE(17)
            default:
                set_error("unsupported window width");
                return PIF_ERR_VALUE;
        }
#undef PIF_RING_INTERP_CASE
    } else {
        blocks = grid_for(P.count, 128, p.sm_count);
        if (blocks > p.partial_blocks) blocks = p.partial_blocks;
        interp_generic_kernel<<<blocks, 128, 0, s>>>(P, perm, Q, field, p.beta, pp, push ? 1 : 0,
                                                     key,
                                                     rank, p.cell_count, p.partials, E_out);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail_cuda(e, "interp kernel");
    if (push) p.wcache_valid = false;   // the particles moved
    if (push) {
        if (P.count == 0) {
            e = cudaMemsetAsync(diag, 0, sizeof(double) * kDiagSlots, s);
            return fail_cuda(e, "zero diag");
        }
        finish_diag_kernel<<<1, 32 * kDiagSlots, 0, s>>>(p.partials, blocks, diag);
        return fail_cuda(cudaGetLastError(), "finish_diag_kernel");
    }
    return PIF_OK;
}
}  // namespace

int launch_interp(Plan &p, const pif_soa_t &P, const int32_t *perm, pif_soa_t &Q, bool push,
                  double half, double dt, const double *tq, const double *sq, int has_b,
                  int e_kind, int32_t *key, int32_t *rank, double *diag, double *E_out,
                  cudaStream_t s) {
    p.split_valid = false;
    return interp_impl(p, P, perm, Q, push, half, dt, tq, sq, has_b, e_kind, key, rank, diag,
                       E_out, nullptr, 0, s);
}

bool split_supported(const Plan &p) { return fast_path_ok(p); }

int launch_interp_split(Plan &p, const pif_soa_t &P, const int32_t *perm, int64_t id0,
                        cudaStream_t s) {
    p.split_valid = false;
    if (!split_supported(p)) {
        set_error("split gather: DMMA kernels (w <= 8) only");
        return PIF_ERR_STATE;
    }
    if (ensure_ring_scratch(p, P.count) != PIF_OK) return PIF_ERR_CUDA;
    pif_soa_t Q = P;
    const int rc = interp_impl(p, P, perm, Q, false, 0.0, 1.0, nullptr, nullptr, 0, PIF_EXT_NONE,
                               nullptr, nullptr, nullptr, nullptr, p.ring_scratch, id0, s);
    if (rc == PIF_OK) {
        p.split_valid = true;
        p.split_count = P.count;
        p.split_parts = 0;
    }
    return rc;
}

int launch_push_ids(Plan &p, double *x, double *v, int64_t M, int64_t r0, int64_t r1,
                    double half, double dt, const double *tq, const double *sq, int has_b,
                    int e_kind, double *diag, cudaStream_t s) {
    if (!p.split_valid || p.split_count != M) {
        set_error("pif_push_ids: no split gather of these particles (pif_interp_split first)");
        return PIF_ERR_STATE;
    }
    if (r0 == 0) p.split_parts = 0;
    p.wcache_valid = false;   // the particles move
    PushParams pp = make_push(p, half, dt, tq, sq, has_b, e_kind);
    // the chunk's share of the diagnostic partial slots (rows / M of them)
    int blocks = grid_for(r1 - r0, 256, p.sm_count);
    const int share = (int)(((int64_t)p.partial_blocks * (r1 - r0)) / (M > 0 ? M : 1));
    if (blocks > share) blocks = share > 0 ? share : 1;
    const int room = p.partial_blocks - p.split_parts;
    if (blocks > room) blocks = room;
    if (blocks < 1) {
        set_error("pif_push_ids: too many row chunks for the diagnostic partials");
        return PIF_ERR_VALUE;
    }
    if (r1 > r0) {
        push_ids_kernel<<<blocks, 256, 0, s>>>(x, v, p.ring_scratch, r0, r1, pp,
                                               p.partials + (size_t)p.split_parts * kDiagSlots);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail_cuda(e, "push_ids_kernel");
        p.split_parts += blocks;
    }
    if (r1 < M) return PIF_OK;
    p.split_valid = false;   // every row pushed
    if (p.split_parts == 0) {
        const cudaError_t e = cudaMemsetAsync(diag, 0, sizeof(double) * kDiagSlots, s);
        return fail_cuda(e, "zero diag");
    }
    finish_diag_kernel<<<1, 32 * kDiagSlots, 0, s>>>(p.partials, p.split_parts, diag);
    return fail_cuda(cudaGetLastError(), "finish_diag_kernel");
}

int launch_particle_diag(Plan &p, const pif_soa_t &P, int e_kind, double *diag, cudaStream_t s) {
    int blocks = grid_for(P.count, 256, p.sm_count);
    if (blocks > p.partial_blocks) blocks = p.partial_blocks;
    particle_diag_kernel<<<blocks, 256, 0, s>>>(P, p.L, e_kind, p.partials);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail_cuda(e, "particle_diag_kernel");
    finish_diag_kernel<<<1, 32 * kDiagSlots, 0, s>>>(p.partials, blocks, diag);
    return fail_cuda(cudaGetLastError(), "finish_diag_kernel");
}

int launch_type1_complex_spread(Plan &p, const double *pts, const double *vals, int64_t M,
                                cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(p.cgrid, 0, sizeof(double2) * p.n3, s);
    if (e != cudaSuccess) return fail_cuda(e, "zero complex grid");
    if (M == 0) return PIF_OK;
    spread_complex_kernel<<<grid_for(M, 128, p.sm_count), 128, 0, s>>>(
        pts, reinterpret_cast<const double2 *>(vals), M, p.cgrid, p.n, p.w, p.h, p.beta);
    return fail_cuda(cudaGetLastError(), "spread_complex_kernel");
}

int launch_type2_complex_interp(Plan &p, const double *pts, int64_t M, double *out,
                                cudaStream_t s) {
    if (M == 0) return PIF_OK;
    interp_complex_kernel<<<grid_for(M, 128, p.sm_count), 128, 0, s>>>(
        p.cgrid, pts, M, reinterpret_cast<double2 *>(out), p.n, p.w, p.h, p.beta);
    return fail_cuda(cudaGetLastError(), "interp_complex_kernel");
}

}  // namespace pif
