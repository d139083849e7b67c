// Fast fp64 exponential-of-semicircle weight for the sm_100a kernels.
//
// phi(t) = exp(beta (sqrt(1 - t^2) - 1)) (_kernels.py:21-26) with
//  * sqrt from the MUFU.RSQ64H seed + two Newton corrections (full fp64), and
//  * exp by Cody-Waite reduction onto a 32-entry 2^(j/32) table in shared memory
//    plus a degree-6 polynomial (|r| <= ln2/64, truncation < 4e-18).
// About 24 FP64-pipe instructions per weight instead of ~42 for libdevice
// exp()+sqrt(); agreement with the reference formula is ~1e-15 relative
// (tools/dmma_probe.cu measures it on the GPU).
#pragma once

namespace pif {

__device__ __constant__ static const double kExp2Table[32] = {
    1.0, 1.0218971486541166, 1.0442737824274138, 1.0671404006768237, 1.0905077326652577,
    1.1143867425958924, 1.1387886347566916, 1.1637248587775775, 1.189207115002721,
    1.215247359980469, 1.241857812073484, 1.2690509571917332, 1.2968395546510096,
    1.3252366431597413, 1.3542555469368927, 1.383909881963832, 1.4142135623730951,
    1.4451808069770467, 1.4768261459394993, 1.5091644275934228, 1.5422108254079407,
    1.5759808451078865, 1.6104903319492543, 1.645755478153965, 1.681792830507429,
    1.718619298122478, 1.7562521603732995, 1.7947090750031072, 1.8340080864093424,
    1.8741676341103, 1.9152065613971474, 1.9571441241754002};

// e^y for y in [-40, 0]; tab = kExp2Table staged in shared memory
__device__ __forceinline__ double exp_neg_fast(double y, const double *tab) {
    const double magic = 6755399441055744.0;  // 1.5 * 2^52
    double kd = fma(y, 46.16624130844683, magic);  // 32/ln2
    const int k = __double2loint(kd);
    kd -= magic;
    double r = fma(kd, -0.021660849392475257, y);  // ln2/32 (hi, 40 bits)
    r = fma(kd, -2.303438301614937e-14, r);        // ln2/32 (lo)
    double p = 1.0 / 720.0;
    p = fma(p, r, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    double v = tab[k & 31] * p;
    return __hiloint2double(__double2hiint(v) + ((k >> 5) << 20), __double2loint(v));
}

__device__ __forceinline__ double rsqrt_seed(double u) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(u));
    return y;
}

// sqrt(u) for u in [1e-300, 1]: seed + Newton on 1/sqrt + one sqrt correction
__device__ __forceinline__ double sqrt_fast(double u) {
    double y = rsqrt_seed(u);
    double e = fma(-u * y, y, 1.0);
    y = fma(0.5 * y, e, y);
    double s = u * y;
    return fma(0.5 * y, fma(-s, s, u), s);
}

__device__ __forceinline__ double es_weight_fast(double c, double i, double inv_half, double beta,
                                                 const double *tab) {
    const double t = __dmul_rn(__dsub_rn(c, i), inv_half);
    const double u = fmax(fma(-t, t, 1.0), 1e-300);
    return exp_neg_fast(fma(beta, sqrt_fast(u), -beta), tab);
}

}  // namespace pif

namespace pif {

// Interior window weights as polynomials.  For a coordinate c (grid units) with
// x = c - w/2, i0 = ceil(x) and f = i0 - x in [0, 1) (both steps exact), weight a
// is phi(1 - (2/w)(a + f)).  For 1 <= a <= w-2 this is analytic on f in [0, 1]
// (the sqrt branch points of phi sit at a + f = 0 and a + f = w), so it is
// a degree-kEsDeg polynomial p_a in u = 2f - 1 (coefficients from Chebyshev
// interpolation in extended precision at plan creation, build_es_poly in
// capi.cu).  phi is even, so weight w-1-a is p_a(-u): each mirrored pair is
// evaluated from one even part E(u^2) and one odd part O(u^2) as E +/- u O,
// half the Horner steps of two separate chains.  The error of exactly this
// evaluation is checked on the host (< 4e-15 absolute).  The two edge weights
// keep the exact formula.
constexpr int kEsDeg = 14;
constexpr int kEsEven = kEsDeg / 2;          // E has coefficients c[0], c[2], .., c[14]
constexpr int kEsOdd = (kEsDeg - 1) / 2;     // O has coefficients c[1], c[3], .., c[13]
// From this width on every interior weight is a polynomial (launchers route a
// plan with exact_mask != 0 to the generic kernels), so no exact branch is compiled.
constexpr int kPolyOnlyW = 6;

struct EsPoly {
    double c[kMaxFastW - 2][kEsDeg + 1];   // [a - 1][power], rows a <= (w-1)/2 used
    int exact_mask;                        // bit a-1 set: evaluate weight a exactly
};

template <int W>
__device__ __forceinline__ void es_axis_weights(double c, double beta, const EsPoly &P,
                                                const double *tab, double (&wt)[W]) {
    constexpr double inv_half = 2.0 / W;
    const double i0 = stencil_start(c, W);
    wt[0] = es_weight_fast(c, i0, inv_half, beta, tab);
    if (W > 1) wt[W - 1] = es_weight_fast(c, i0 + (double)(W - 1), inv_half, beta, tab);
    const double f = i0 - __dsub_rn(c, 0.5 * W);
    const double u = fma(2.0, f, -1.0);
    const double v = u * u;
#pragma unroll
    for (int a = 1; 2 * a <= W - 1; ++a) {
        const int b = W - 1 - a;
        if (W < kPolyOnlyW && (P.exact_mask & (1 << (a - 1)))) {
            wt[a] = es_weight_fast(c, i0 + (double)a, inv_half, beta, tab);
            if (b != a) wt[b] = es_weight_fast(c, i0 + (double)b, inv_half, beta, tab);
        } else {
            double e = P.c[a - 1][2 * kEsEven], o = P.c[a - 1][2 * kEsOdd + 1];
#pragma unroll
            for (int k = kEsEven - 1; k >= 0; --k) {
                e = fma(e, v, P.c[a - 1][2 * k]);
                if (k < kEsOdd) o = fma(o, v, P.c[a - 1][2 * k + 1]);
            }
            wt[a] = fma(u, o, e);
            if (b != a) wt[b] = fma(-u, o, e);
        }
    }
}

}  // namespace pif

namespace pif {

// All three axes at once: the 3 x (pairs) even/odd Horner chains advance
// together (power-outer loop) so a warp has many independent FMAs in flight.
template <int W>
__device__ __forceinline__ void es_xyz_weights(const double (&c)[3], double beta, const EsPoly &P,
                                               const double *tab, double (&wt)[3][W]) {
    constexpr double inv_half = 2.0 / W;
    constexpr int NP = (W - 1) / 2;          // pairs (a, w-1-a), a = 1 .. NP (+ middle if odd)
    double u[3], v[3], i0[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        i0[d] = stencil_start(c[d], W);
        u[d] = fma(2.0, i0[d] - __dsub_rn(c[d], 0.5 * W), -1.0);
        v[d] = u[d] * u[d];
    }
    if (NP > 0) {
        double e[3][NP > 0 ? NP : 1], o[3][NP > 0 ? NP : 1];
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
            for (int a = 0; a < NP; ++a) {
                e[d][a] = P.c[a][2 * kEsEven];
                o[d][a] = P.c[a][2 * kEsOdd + 1];
            }
#pragma unroll
        for (int k = kEsEven - 1; k >= 0; --k)
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int a = 0; a < NP; ++a) {
                    e[d][a] = fma(e[d][a], v[d], P.c[a][2 * k]);
                    if (k < kEsOdd) o[d][a] = fma(o[d][a], v[d], P.c[a][2 * k + 1]);
                }
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
            for (int a = 0; a < NP; ++a) {
                wt[d][a + 1] = fma(u[d], o[d][a], e[d][a]);
                if (W - 2 - a != a + 1) wt[d][W - 2 - a] = fma(-u[d], o[d][a], e[d][a]);
            }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        wt[d][0] = es_weight_fast(c[d], i0[d], inv_half, beta, tab);
        if (W > 1) wt[d][W - 1] = es_weight_fast(c[d], i0[d] + (double)(W - 1), inv_half, beta, tab);
#pragma unroll
        for (int a = 1; a + 1 < W; ++a)
            if (W < kPolyOnlyW && (P.exact_mask & (1 << (min(a, W - 1 - a) - 1))))
                wt[d][a] = es_weight_fast(c[d], i0[d] + (double)a, inv_half, beta, tab);
    }
}

}  // namespace pif
