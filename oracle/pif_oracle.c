/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's numba window kernels
 * (/root/reference/pkg/src/pifsim/_kernels.py).  Only tests/, the smoke check in
 * __graft_entry__.py and bench.py's cpu_baseline / --impl reference legs may load
 * this library; the product path (paper_2605_10729_b200) never does.
 *
 * Arithmetic is kept in the reference's order, one particle at a time, without
 * FMA contraction (built with -ffp-contract=off), so results agree with the
 * numba kernels to the last bit or ulp (pinned in tests/test_oracle.py).
 *
 * Layouts follow the reference: points are (M,3) row-major doubles, grids are
 * flat C-order n^3 arrays with index (ix*n + iy)*n + iz, complex values are
 * interleaved (re, im) pairs.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define WMAX 32

/* Stencil of one coordinate: the reference's _stencil (_kernels.py:11-28).
 * c is the coordinate in fine-grid units.  Returns the first (unwrapped) index
 * i0 = ceil(c - w/2); fills w window weights and the wrapped indices. */
static int64_t stencil(double c, int64_t n, int w, double half, double inv_half,
                       double beta, double *wt, int64_t *idx)
{
    int64_t i0 = (int64_t)ceil(c - half);
    for (int a = 0; a < w; ++a) {
        int64_t i = i0 + a;
        double t = (c - (double)i) * inv_half;
        double u = 1.0 - t * t;
        if (u < 0.0) u = 0.0;
        wt[a] = exp(beta * (sqrt(u) - 1.0));
        int64_t m = i % n;             /* python-style non-negative modulo */
        idx[a] = m < 0 ? m + n : m;
    }
    return i0;
}

static int64_t pmod(int64_t i, int64_t n) { int64_t m = i % n; return m < 0 ? m + n : m; }

/* Real-strength spreading, reference spread_r (_kernels.py:57-96).
 * Accumulates into grid (caller zeroes it). */
void oracle_spread_r(const double *pts, const double *vals, double *grid,
                     int64_t M, int64_t n, double h, int w, double beta)
{
    double wx[WMAX], wy[WMAX], wz[WMAX];
    int64_t ix[WMAX], iy[WMAX], iz[WMAX];
    const double half = 0.5 * w, inv_half = 2.0 / w;
    for (int64_t p = 0; p < M; ++p) {
        stencil(pts[3 * p + 0] / h, n, w, half, inv_half, beta, wx, ix);
        stencil(pts[3 * p + 1] / h, n, w, half, inv_half, beta, wy, iy);
        int64_t z0 = pmod(stencil(pts[3 * p + 2] / h, n, w, half, inv_half, beta, wz, iz), n);
        const double s = vals[p];
        const int contiguous = (z0 + w <= n);
        for (int a = 0; a < w; ++a) {
            const double sa = s * wx[a];
            const int64_t ra = ix[a] * n;
            for (int b = 0; b < w; ++b) {
                const double sab = sa * wy[b];
                if (contiguous) {
                    double *row = grid + (ra + iy[b]) * n + z0;
                    for (int c = 0; c < w; ++c) row[c] += sab * wz[c];
                } else {
                    double *row = grid + (ra + iy[b]) * n;
                    for (int c = 0; c < w; ++c) row[iz[c]] += sab * wz[c];
                }
            }
        }
    }
}

/* Complex-strength spreading, reference spread_c (_kernels.py:31-54). */
void oracle_spread_c(const double *pts, const double *vals /* 2M */, double *grid /* 2n^3 */,
                     int64_t M, int64_t n, double h, int w, double beta)
{
    double wx[WMAX], wy[WMAX], wz[WMAX];
    int64_t ix[WMAX], iy[WMAX], iz[WMAX];
    const double half = 0.5 * w, inv_half = 2.0 / w;
    for (int64_t p = 0; p < M; ++p) {
        stencil(pts[3 * p + 0] / h, n, w, half, inv_half, beta, wx, ix);
        stencil(pts[3 * p + 1] / h, n, w, half, inv_half, beta, wy, iy);
        stencil(pts[3 * p + 2] / h, n, w, half, inv_half, beta, wz, iz);
        const double sr = vals[2 * p], si = vals[2 * p + 1];
        for (int a = 0; a < w; ++a) {
            const double ar = sr * wx[a], ai = si * wx[a];
            const int64_t ra = ix[a] * n;
            for (int b = 0; b < w; ++b) {
                const double br = ar * wy[b], bi = ai * wy[b];
                const int64_t base = (ra + iy[b]) * n;
                for (int c = 0; c < w; ++c) {
                    double *g = grid + 2 * (base + iz[c]);
                    g[0] += br * wz[c];
                    g[1] += bi * wz[c];
                }
            }
        }
    }
}

/* Complex gather from one grid, reference interp_c (_kernels.py:99-122). */
void oracle_interp_c(const double *pts, const double *grid /* 2n^3 */, double *out /* 2M */,
                     int64_t M, int64_t n, double h, int w, double beta)
{
    double wx[WMAX], wy[WMAX], wz[WMAX];
    int64_t ix[WMAX], iy[WMAX], iz[WMAX];
    const double half = 0.5 * w, inv_half = 2.0 / w;
    for (int64_t p = 0; p < M; ++p) {
        stencil(pts[3 * p + 0] / h, n, w, half, inv_half, beta, wx, ix);
        stencil(pts[3 * p + 1] / h, n, w, half, inv_half, beta, wy, iy);
        stencil(pts[3 * p + 2] / h, n, w, half, inv_half, beta, wz, iz);
        double accr = 0.0, acci = 0.0;
        for (int a = 0; a < w; ++a) {
            const int64_t ra = ix[a] * n;
            for (int b = 0; b < w; ++b) {
                const int64_t base = (ra + iy[b]) * n;
                const double wab = wx[a] * wy[b];
                for (int c = 0; c < w; ++c) {
                    const double k = wab * wz[c];
                    const double *g = grid + 2 * (base + iz[c]);
                    accr += g[0] * k;
                    acci += g[1] * k;
                }
            }
        }
        out[2 * p] = accr;
        out[2 * p + 1] = acci;
    }
}

/* Three-component real gather, reference interp_r3 (_kernels.py:125-183):
 * per-z-lane partial sums, then an ordered dot product with the z weights. */
void oracle_interp_r3(const double *pts, const double *g0, const double *g1, const double *g2,
                      double *out /* (M,3) */, int64_t M, int64_t n, double h, int w, double beta)
{
    double wx[WMAX], wy[WMAX], wz[WMAX];
    double l0[WMAX], l1[WMAX], l2[WMAX];
    int64_t ix[WMAX], iy[WMAX], iz[WMAX];
    const double half = 0.5 * w, inv_half = 2.0 / w;
    for (int64_t p = 0; p < M; ++p) {
        stencil(pts[3 * p + 0] / h, n, w, half, inv_half, beta, wx, ix);
        stencil(pts[3 * p + 1] / h, n, w, half, inv_half, beta, wy, iy);
        int64_t z0 = pmod(stencil(pts[3 * p + 2] / h, n, w, half, inv_half, beta, wz, iz), n);
        for (int c = 0; c < w; ++c) l0[c] = l1[c] = l2[c] = 0.0;
        const int contiguous = (z0 + w <= n);
        for (int a = 0; a < w; ++a) {
            const int64_t ra = ix[a] * n;
            for (int b = 0; b < w; ++b) {
                const double wab = wx[a] * wy[b];
                const int64_t base = (ra + iy[b]) * n;
                for (int c = 0; c < w; ++c) {
                    const int64_t j = contiguous ? base + z0 + c : base + iz[c];
                    l0[c] += g0[j] * wab;
                    l1[c] += g1[j] * wab;
                    l2[c] += g2[j] * wab;
                }
            }
        }
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        for (int c = 0; c < w; ++c) {
            a0 += l0[c] * wz[c];
            a1 += l1[c] * wz[c];
            a2 += l2[c] * wz[c];
        }
        out[3 * p + 0] = a0;
        out[3 * p + 1] = a1;
        out[3 * p + 2] = a2;
    }
}

/* Window weights of one coordinate, exported so tests can compare the device
 * weight evaluation against the reference formula point by point. */
int64_t oracle_stencil(double c, int64_t n, int w, double beta, double *wt, int64_t *idx)
{
    return stencil(c, n, w, 0.5 * w, 2.0 / w, beta, wt, idx);
}
