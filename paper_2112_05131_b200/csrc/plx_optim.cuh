// plx_optim.cuh -- the RMSProp / SGD element update (K:572-590) and the
// device-side divergence guard, shared by the single-GPU optimiser kernels
// (plx_grid_ops.cu) and the data-parallel exchange kernels (plx_dp.cu).
#pragma once

#include "plx_common.cuh"

namespace plx {

// lr*g / (sqrt(nv) + eps) in float64 without the IEEE div/sqrt subroutines
// (they were ~60 % of this kernel's instructions): MUFU reciprocal-sqrt and
// reciprocal seeds, Newton steps with explicit FMAs, and one residual
// correction each, so both the root and the quotient are within ~1 ulp of
// float64.  The result is rounded to the f32 table afterwards, where it
// equals the correctly rounded float64 path except at f32 rounding ties
// (~2^-29 of values).  nv > 0 and sqrt(nv) + eps >= 1e-8 here (g != 0).
__device__ __forceinline__ double rms_quot(double num, double nv, double eps) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(nv));
    const double hn = 0.5 * nv;
    y = y * fma(-hn * y, y, 1.5);
    y = y * fma(-hn * y, y, 1.5);
    double s = nv * y;
    s = fma(0.5 * y, fma(-s, s, nv), s);   // sqrt(nv), corrected
    const double den = s + eps;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
    r = r * fma(-den, r, 2.0);
    r = r * fma(-den, r, 2.0);
    double q = num * r;
    q = fma(r, fma(-den, q, num), q);      // num / den, corrected
    return q;
}

// Divergence guard (trainer.py T:473-480 on the device): guard[0..3] are
// the step's loss sums, guard[4] a sticky halt flag.  True = skip the step.
__device__ __forceinline__ bool guard_halts(double *guard) {
    if (!guard) return false;
    bool bad = guard[4] != 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) bad |= !isfinite(guard[i]);
    return bad;
}

// The update of one float4 of one row (K:578-590), float64 arithmetic.
struct OptHyper {
    double lr_sigma, lr_sh, beta, eps;
    int rmsprop;
};

__device__ __forceinline__ void opt_apply4(const OptHyper &a, int quad, float4 &g4, float4 &t4,
                                           float4 &v4) {
    float g[4] = {g4.x, g4.y, g4.z, g4.w};
    float t[4] = {t4.x, t4.y, t4.z, t4.w};
    float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (g[e] == 0.0f) continue;   // K:581-583: stale state
        const double gd = (double)g[e];
        const double lr = (quad == 0 && e == 0) ? a.lr_sigma : a.lr_sh;
        if (a.rmsprop) {
            const double nv = a.beta * (double)v[e] + (1.0 - a.beta) * gd * gd;
            v[e] = (float)nv;
            t[e] = (float)((double)t[e] - rms_quot(lr * gd, nv, a.eps));
        } else {
            t[e] = (float)((double)t[e] - lr * gd);
        }
    }
    t4 = make_float4(t[0], t[1], t[2], t[3]);
    v4 = make_float4(v[0], v[1], v[2], v[3]);
}

}  // namespace plx
