// Particle-side kernels of the PD-PIF step on sm_100a:
//   binning (ES-stencil cell keys, counting-sort scatter),
//   type-1 spreading (replaces _kernels.spread_r, _kernels.py:57-96),
//   type-2 gather fused with the Boris push (replaces _kernels.interp_r3,
//   _kernels.py:125-183, and pif.boris_push, pif.py:140-158),
//   diagnostics sums (strategies.py:96-106), generic wide-window fallbacks.
//
// Fast kernels (w <= 8): one warp owns a work item = a z-segment of one
// (i0x, i0y) column of stencil cells.  All particles of a cell share one
// w x w x w footprint, so a lane keeps its footprint points in registers:
// lane owns (a,b) pairs q = lane and lane+32 of the w*w xy-footprint, times w
// z planes.  Moving to the next cell along z rotates the register planes by
// one (a register move, no reload of the other w-1 planes), so per cell only
// one new plane is flushed (spread, REDG.ADD.F64) or loaded (gather).
#include <cub/cub.cuh>

#include "pif_internal.cuh"

namespace pif {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int cell_index_of(double c, int w, int n) {
    return pmod((int)stencil_start(c, w), n);
}

__device__ __forceinline__ int cell_key(double x, double y, double z, double h, int w, int n) {
    int kx = cell_index_of(axis_coord(x, h), w, n);
    int ky = cell_index_of(axis_coord(y, h), w, n);
    int kz = cell_index_of(axis_coord(z, h), w, n);
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
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        int k = cell_key(x[i], y[i], z[i], h, w, n);
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

// ----------------------------------------------------------------------------
// shared per-warp staging of one sub-batch (<= kSub particles of one cell)
// ----------------------------------------------------------------------------

template <int W>
struct WarpStage {
    double wt[kSub][3][W];   // window weights; x row optionally scaled by strength
    double c[kSub][3];       // coordinates in grid units
    double i0[kSub][3];      // stencil starts
};

// Phase 1: coordinates + stencil starts (24 lanes, one (particle, axis) each).
// Phase 2: 3*W*kSub weights spread over the 32 lanes.
template <int W>
__device__ __forceinline__ void stage_weights(WarpStage<W> &st, int lane, int p0, int cnt,
                                              const double *__restrict__ px,
                                              const double *__restrict__ py,
                                              const double *__restrict__ pz,
                                              const int64_t *__restrict__ pid,
                                              const double *__restrict__ strengths, double q,
                                              bool scale_x, double h, double beta) {
    if (lane < 3 * kSub) {
        const int j = lane / 3, d = lane - 3 * (lane / 3);
        if (j < cnt) {
            const double *src = d == 0 ? px : (d == 1 ? py : pz);
            double c = axis_coord(src[p0 + j], h);
            st.c[j][d] = c;
            st.i0[j][d] = stencil_start(c, W);
        }
    }
    __syncwarp();
    constexpr double inv_half = 2.0 / W;
#pragma unroll
    for (int t0 = 0; t0 < kSub * 3 * W; t0 += 32) {
        const int t = t0 + lane;
        if (t < kSub * 3 * W) {
            const int j = t / (3 * W);
            const int r = t - j * (3 * W);
            const int d = r / W;
            const int a = r - d * W;
            double v = 0.0;
            if (j < cnt) {
                v = es_weight(st.c[j][d], st.i0[j][d] + (double)a, inv_half, beta);
                if (scale_x && d == 0) {
                    double s = strengths ? strengths[pid[p0 + j]] : q;
                    v = __dmul_rn(s, v);   // sa = s * wx[a] (_kernels.py:81)
                }
            }
            st.wt[j][d][a] = v;
        }
    }
    __syncwarp();
}

// ----------------------------------------------------------------------------
// fused spreading (w <= 8)
// ----------------------------------------------------------------------------

template <int W>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
spread_fast_kernel(const double *__restrict__ px, const double *__restrict__ py,
                   const double *__restrict__ pz, const int64_t *__restrict__ pid,
                   const double *__restrict__ strengths, double q,
                   const int32_t *__restrict__ cell_start, double *__restrict__ grid, int n,
                   int seg, int nseg, double h, double beta, unsigned int *work, int nitems) {
    __shared__ WarpStage<W> stage[kWarpsPerBlock];
    const int lane = threadIdx.x & 31;
    WarpStage<W> &st = stage[threadIdx.x >> 5];
    const int q0 = lane, q1 = lane + 32;
    const bool v0 = q0 < W * W, v1 = q1 < W * W;
    const int a0 = v0 ? q0 / W : 0, b0 = v0 ? q0 % W : 0;
    const int a1 = v1 ? q1 / W : 0, b1 = v1 ? q1 % W : 0;

    for (;;) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(work, 1u);
        item = __shfl_sync(kFull, item, 0);
        if (item >= nitems) break;
        const int col = item / nseg, sg = item - col * nseg;
        const int ix = col / n, iy = col - ix * n;
        const int k0 = sg * seg, k1 = min(k0 + seg, n);
        const int base = col * n;
        if (cell_start[base + k0] == cell_start[base + k1]) continue;

        const int64_t row0 = ((int64_t)((ix + a0) % n) * n + (iy + b0) % n) * n;
        const int64_t row1 = ((int64_t)((ix + a1) % n) * n + (iy + b1) % n) * n;
        double acc0[W], acc1[W];
#pragma unroll
        for (int s = 0; s < W; ++s) acc0[s] = acc1[s] = 0.0;

        for (int k = k0; k < k1; ++k) {
            const int cs = cell_start[base + k], ce = cell_start[base + k + 1];
            for (int p0 = cs; p0 < ce; p0 += kSub) {
                const int cnt = min(kSub, ce - p0);
                stage_weights<W>(st, lane, p0, cnt, px, py, pz, pid, strengths, q, true, h, beta);
                for (int j = 0; j < cnt; ++j) {
                    // sab = (s * wx[a]) * wy[b]; grid += sab * wz[c]  (_kernels.py:81-87)
                    const double s0 = st.wt[j][0][a0] * st.wt[j][1][b0];
                    const double s1 = st.wt[j][0][a1] * st.wt[j][1][b1];
#pragma unroll
                    for (int c = 0; c < W; ++c) {
                        const double wz = st.wt[j][2][c];
                        acc0[c] = fma(s0, wz, acc0[c]);
                        acc1[c] = fma(s1, wz, acc1[c]);
                    }
                }
                __syncwarp();
            }
            // plane k is complete: flush slot 0, rotate the window by one plane
            const int z = k;  // k < n
            if (v0 && acc0[0] != 0.0) atomicAdd(grid + row0 + z, acc0[0]);
            if (v1 && acc1[0] != 0.0) atomicAdd(grid + row1 + z, acc1[0]);
#pragma unroll
            for (int s = 0; s + 1 < W; ++s) {
                acc0[s] = acc0[s + 1];
                acc1[s] = acc1[s + 1];
            }
            acc0[W - 1] = acc1[W - 1] = 0.0;
        }
#pragma unroll
        for (int s = 0; s + 1 < W; ++s) {
            const int z = (k1 + s) % n;
            if (v0 && acc0[s] != 0.0) atomicAdd(grid + row0 + z, acc0[s]);
            if (v1 && acc1[s] != 0.0) atomicAdd(grid + row1 + z, acc1[s]);
        }
    }
}

// ----------------------------------------------------------------------------
// fused gather (+ Boris push) (w <= 8)
// ----------------------------------------------------------------------------

struct PushParams {
    double half, dt, L, h;
    double tq[3], sq[3];
    int has_b, e_kind, n, w;
};

// Boris push of one particle (pif.py:146-157), external quadrupole
// (pif.py:52-57), periodic wrap (particles.py:65-70); no FMA contraction so the
// update rounds like numpy.  Accumulates diagnostics of the updated particle.
__device__ __forceinline__ void boris_one(const PushParams &pp, double E0, double E1, double E2,
                                          double &x, double &y, double &z, double &vx,
                                          double &vy, double &vz, double *dg) {
    double et0 = E0, et1 = E1, et2 = E2;
    const double L = pp.L;
    if (pp.e_kind == PIF_EXT_QUADRUPOLE) {
        const double c = L / 2.0;
        et0 = __dadd_rn(et0, __dmul_rn(-15.0 / L, __dsub_rn(x, c)));
        et1 = __dadd_rn(et1, __dmul_rn(-15.0 / L, __dsub_rn(y, c)));
        et2 = __dadd_rn(et2, __dmul_rn(30.0 / L, __dsub_rn(z, c)));
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
        const double c = L / 2.0;
        const double dx = x - c, dy = y - c, dz = z - c;
        dg[4] += (7.5 / L) * (dx * dx + dy * dy) - (15.0 / L) * (dz * dz);
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

// Transposed warp reduction of part[kSub][3]: after it, every lane of group
// g = (lane >> 2) & 7 holds the full 32-lane sum for particle g.
__device__ __forceinline__ void reduce_scatter8(double (&part)[kSub][3], int lane, double *e) {
    double r1[4][3], r2[2][3];
    const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double keep = h16 ? part[j + 4][d] : part[j][d];
            double send = h16 ? part[j][d] : part[j + 4][d];
            r1[j][d] = keep + __shfl_xor_sync(kFull, send, 16);
        }
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double keep = h8 ? r1[j + 2][d] : r1[j][d];
            double send = h8 ? r1[j][d] : r1[j + 2][d];
            r2[j][d] = keep + __shfl_xor_sync(kFull, send, 8);
        }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double keep = h4 ? r2[1][d] : r2[0][d];
        double send = h4 ? r2[0][d] : r2[1][d];
        double v = keep + __shfl_xor_sync(kFull, send, 4);
        v += __shfl_xor_sync(kFull, v, 2);
        v += __shfl_xor_sync(kFull, v, 1);
        e[d] = v;
    }
}

template <int W, bool PUSH>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
interp_fast_kernel(pif_soa_t P, const int32_t *__restrict__ cell_start,
                   const double4 *__restrict__ field, int seg, int nseg, double beta,
                   PushParams pp, int32_t *__restrict__ key, int32_t *__restrict__ rank,
                   int32_t *__restrict__ count, double *__restrict__ partials,
                   double *__restrict__ E_out, unsigned int *work, int nitems) {
    __shared__ WarpStage<W> stage[kWarpsPerBlock];
    const int lane = threadIdx.x & 31;
    WarpStage<W> &st = stage[threadIdx.x >> 5];
    const int n = pp.n;
    const double h = pp.h;
    const int q0 = lane, q1 = lane + 32;
    const bool v0 = q0 < W * W, v1 = q1 < W * W;
    const int a0 = v0 ? q0 / W : 0, b0 = v0 ? q0 % W : 0;
    const int a1 = v1 ? q1 / W : 0, b1 = v1 ? q1 % W : 0;
    const int grp = (lane >> 2) & 7;
    double dg[5] = {0.0, 0.0, 0.0, 0.0, 0.0};

    for (;;) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(work, 1u);
        item = __shfl_sync(kFull, item, 0);
        if (item >= nitems) break;
        const int col = item / nseg, sg = item - col * nseg;
        const int ix = col / n, iy = col - ix * n;
        const int k0 = sg * seg, k1 = min(k0 + seg, n);
        const int base = col * n;
        if (cell_start[base + k0] == cell_start[base + k1]) continue;

        const int64_t row0 = ((int64_t)((ix + a0) % n) * n + (iy + b0) % n) * n;
        const int64_t row1 = ((int64_t)((ix + a1) % n) * n + (iy + b1) % n) * n;
        // window of W planes: g0/g1[s] = field at plane k + s for the two pairs
        double g0[W][3], g1[W][3];
#pragma unroll
        for (int s = 0; s < W; ++s) {
            const int z = (k0 + s) % n;
            double4 f0 = v0 ? field[row0 + z] : make_double4(0, 0, 0, 0);
            double4 f1 = v1 ? field[row1 + z] : make_double4(0, 0, 0, 0);
            g0[s][0] = f0.x; g0[s][1] = f0.y; g0[s][2] = f0.z;
            g1[s][0] = f1.x; g1[s][1] = f1.y; g1[s][2] = f1.z;
        }
        for (int k = k0; k < k1; ++k) {
            if (k > k0) {
#pragma unroll
                for (int s = 0; s + 1 < W; ++s)
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        g0[s][d] = g0[s + 1][d];
                        g1[s][d] = g1[s + 1][d];
                    }
                const int z = (k + W - 1) % n;
                double4 f0 = v0 ? field[row0 + z] : make_double4(0, 0, 0, 0);
                double4 f1 = v1 ? field[row1 + z] : make_double4(0, 0, 0, 0);
                g0[W - 1][0] = f0.x; g0[W - 1][1] = f0.y; g0[W - 1][2] = f0.z;
                g1[W - 1][0] = f1.x; g1[W - 1][1] = f1.y; g1[W - 1][2] = f1.z;
            }
            const int cs = cell_start[base + k], ce = cell_start[base + k + 1];
            for (int p0 = cs; p0 < ce; p0 += kSub) {
                const int cnt = min(kSub, ce - p0);
                stage_weights<W>(st, lane, p0, cnt, P.x, P.y, P.z, P.id, nullptr, 0.0, false, h,
                                 beta);
                double part[kSub][3];
#pragma unroll
                for (int j = 0; j < kSub; ++j) {
                    if (j < cnt) {
                        double h0[3] = {0.0, 0.0, 0.0}, h1[3] = {0.0, 0.0, 0.0};
#pragma unroll
                        for (int c = 0; c < W; ++c) {
                            const double wz = st.wt[j][2][c];
#pragma unroll
                            for (int d = 0; d < 3; ++d) {
                                h0[d] = fma(g0[c][d], wz, h0[d]);
                                h1[d] = fma(g1[c][d], wz, h1[d]);
                            }
                        }
                        const double w0 = st.wt[j][0][a0] * st.wt[j][1][b0];
                        const double w1 = v1 ? st.wt[j][0][a1] * st.wt[j][1][b1] : 0.0;
#pragma unroll
                        for (int d = 0; d < 3; ++d) part[j][d] = fma(w0, h0[d], w1 * h1[d]);
                    } else {
#pragma unroll
                        for (int d = 0; d < 3; ++d) part[j][d] = 0.0;
                    }
                }
                double e[3];
                reduce_scatter8(part, lane, e);
                if ((lane & 3) == 0 && grp < cnt) {
                    const int64_t i = p0 + grp;
                    if (PUSH) {
                        double x = P.x[i], y = P.y[i], z = P.z[i];
                        double vx = P.vx[i], vy = P.vy[i], vz = P.vz[i];
                        boris_one(pp, e[0], e[1], e[2], x, y, z, vx, vy, vz, dg);
                        P.x[i] = x; P.y[i] = y; P.z[i] = z;
                        P.vx[i] = vx; P.vy[i] = vy; P.vz[i] = vz;
                        const int kk = cell_key(x, y, z, h, pp.w, n);
                        key[i] = kk;
                        rank[i] = atomicAdd(&count[kk], 1);
                    } else {
                        const int64_t o = 3 * P.id[i];
                        E_out[o] = e[0];
                        E_out[o + 1] = e[1];
                        E_out[o + 2] = e[2];
                    }
                }
                __syncwarp();
            }
        }
    }
    if (PUSH) block_diag_store(dg, partials);
}

// ----------------------------------------------------------------------------
// generic one-thread-per-particle kernels (any w <= kMaxW)
// ----------------------------------------------------------------------------

__device__ __forceinline__ int axis_stencil(double xv, double h, int w, double beta, int n,
                                            double *wt, int *idx) {
    const double c = axis_coord(xv, h);
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

__global__ void interp_generic_kernel(pif_soa_t P, const double4 *__restrict__ field, double beta,
                                      PushParams pp, int push, int32_t *__restrict__ key,
                                      int32_t *__restrict__ rank, int32_t *__restrict__ count,
                                      double *__restrict__ partials, double *__restrict__ E_out) {
    double wx[kMaxW], wy[kMaxW], wz[kMaxW];
    int ixs[kMaxW], iys[kMaxW], izs[kMaxW];
    const int n = pp.n, w = pp.w;
    double dg[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P.count;
         i += (int64_t)gridDim.x * blockDim.x) {
        axis_stencil(P.x[i], pp.h, w, beta, n, wx, ixs);
        axis_stencil(P.y[i], pp.h, w, beta, n, wy, iys);
        axis_stencil(P.z[i], pp.h, w, beta, n, wz, izs);
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
            double x = P.x[i], y = P.y[i], z = P.z[i];
            double vx = P.vx[i], vy = P.vy[i], vz = P.vz[i];
            boris_one(pp, e0, e1, e2, x, y, z, vx, vy, vz, dg);
            P.x[i] = x; P.y[i] = y; P.z[i] = z;
            P.vx[i] = vx; P.vy[i] = vy; P.vz[i] = vz;
            const int kk = cell_key(x, y, z, pp.h, w, n);
            key[i] = kk;
            rank[i] = atomicAdd(&count[kk], 1);
        } else {
            const int64_t o = 3 * P.id[i];
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

PushParams make_push(const Plan &p, double half, double dt, const double *tq, const double *sq,
                     int has_b, int e_kind) {
    PushParams pp;
    pp.half = half;
    pp.dt = dt;
    pp.L = p.L;
    pp.h = p.h;
    for (int d = 0; d < 3; ++d) {
        pp.tq[d] = tq ? tq[d] : 0.0;
        pp.sq[d] = sq ? sq[d] : 0.0;
    }
    pp.has_b = has_b;
    pp.e_kind = e_kind;
    pp.n = p.n;
    pp.w = p.w;
    return pp;
}

}  // namespace

// ============================================================================
// launchers
// ============================================================================

int launch_wrap(Plan &p, double *x, double *y, double *z, int64_t M, cudaStream_t s) {
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
    return fail_cuda(cudaMemsetAsync(p.cell_count, 0, sizeof(int32_t) * (p.n3 + 1), s),
                     "reset cell counts");
}

int launch_spread(Plan &p, const pif_soa_t &P, const double *strengths, double q,
                  cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(p.grid, 0, sizeof(double) * p.n3, s);
    if (e != cudaSuccess) return fail_cuda(e, "zero grid");
    if (P.count == 0) return PIF_OK;
    if (p.w <= kMaxFastW) {
        const int nseg = (p.n + p.seg - 1) / p.seg;
        const int nitems = p.n * p.n * nseg;
        e = cudaMemsetAsync(p.work, 0, sizeof(unsigned int), s);
        if (e != cudaSuccess) return fail_cuda(e, "zero work counter");
        const int threads = kWarpsPerBlock * 32;
#define PIF_SPREAD_CASE(W)                                                                   \
    case W: {                                                                                \
        auto k = spread_fast_kernel<W>;                                                      \
        int blocks = persistent_blocks(k, threads, 0, p.sm_count);                           \
        k<<<blocks, threads, 0, s>>>(P.x, P.y, P.z, P.id, strengths, q, p.cell_start, p.grid, \
                                     p.n, p.seg, nseg, p.h, p.beta, p.work, nitems);         \
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
    } else {
        spread_generic_kernel<<<grid_for(P.count, 128, p.sm_count), 128, 0, s>>>(
            P, strengths, q, p.grid, p.n, p.w, p.h, p.beta);
    }
    return fail_cuda(cudaGetLastError(), "spread kernel");
}

int launch_interp(Plan &p, pif_soa_t &P, bool push, double half, double dt, const double *tq,
                  const double *sq, int has_b, int e_kind, int32_t *key, int32_t *rank,
                  double *diag, double *E_out, cudaStream_t s) {
    if (!p.field_valid) {
        set_error("no field grid: solve the fields before gathering");
        return PIF_ERR_STATE;
    }
    PushParams pp = make_push(p, half, dt, tq, sq, has_b, e_kind);
    const double4 *field = reinterpret_cast<const double4 *>(p.field);
    cudaError_t e;
    int blocks = 1;
    if (P.count > 0 && p.w <= kMaxFastW) {
        const int nseg = (p.n + p.seg - 1) / p.seg;
        const int nitems = p.n * p.n * nseg;
        e = cudaMemsetAsync(p.work, 0, sizeof(unsigned int), s);
        if (e != cudaSuccess) return fail_cuda(e, "zero work counter");
        const int threads = kWarpsPerBlock * 32;
#define PIF_INTERP_CASE(W)                                                                    \
    case W: {                                                                                 \
        if (push) {                                                                           \
            auto k = interp_fast_kernel<W, true>;                                             \
            blocks = persistent_blocks(k, threads, 0, p.sm_count);                            \
            if (blocks > p.partial_blocks) blocks = p.partial_blocks;                         \
            k<<<blocks, threads, 0, s>>>(P, p.cell_start, field, p.seg, nseg, p.beta, pp, key, \
                                         rank, p.cell_count, p.partials, E_out, p.work,        \
                                         nitems);                                             \
        } else {                                                                              \
            auto k = interp_fast_kernel<W, false>;                                            \
            blocks = persistent_blocks(k, threads, 0, p.sm_count);                            \
            k<<<blocks, threads, 0, s>>>(P, p.cell_start, field, p.seg, nseg, p.beta, pp, key, \
                                         rank, p.cell_count, p.partials, E_out, p.work,        \
                                         nitems);                                             \
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
    } else {
        blocks = grid_for(P.count, 128, p.sm_count);
        if (blocks > p.partial_blocks) blocks = p.partial_blocks;
        interp_generic_kernel<<<blocks, 128, 0, s>>>(P, field, p.beta, pp, push ? 1 : 0, key,
                                                     rank, p.cell_count, p.partials, E_out);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail_cuda(e, "interp kernel");
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
