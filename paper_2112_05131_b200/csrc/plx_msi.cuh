// plx_msi.cuh -- the multi-sphere-image background's device helpers, shared
// by plx_msi.cu (forward render, TV, update) and plx_render.cu (the
// background stage of the 360 backward, msi_bg_kernel).
// Reference: pkg/src/plenoxel/_kernels.py K:603-658.
#pragma once

#include "plx_common.cuh"

namespace plx {

constexpr int kMaxCross = 256;   // sphere crossings per ray (layers - 1)

struct MsiDev {
    const double *data;   // [L][H][W][4]
    const double *radii;  // [L]
    int L, H, W;
};

// K:606-645 (_bg_stencil): bilinear texel stencil within one layer at the
// sphere angles of p; texel centres at half texels, phi wraps, theta clamps.
__device__ __forceinline__ void bg_stencil(int H, int W, double px, double py, double pz,
                                           int *idx4, double *w4) {
    const double pi = 3.141592653589793;
    const double r = sqrt(px * px + py * py + pz * pz);
    const double phi = atan2(py, px);
    double ct = pz / r;
    if (ct > 1.0) ct = 1.0;
    if (ct < -1.0) ct = -1.0;
    const double theta = acos(ct);
    double u = (phi + pi) / (2.0 * pi) * (double)W - 0.5;
    u = u - floor(u / (double)W) * (double)W;
    double vv = theta / pi * (double)H - 0.5;
    if (vv < 0.0) vv = 0.0;
    if (vv > (double)H - 1.0) vv = (double)H - 1.0;
    int i0 = (int)u;
    if (i0 > W - 1) i0 = W - 1;
    const double fu = u - (double)i0;
    int i1 = i0 + 1;
    if (i1 >= W) i1 = 0;
    int j0 = (int)vv;
    if (j0 > H - 2) j0 = H - 2;
    const double fv = vv - (double)j0;
    idx4[0] = j0 * W + i0;
    idx4[1] = j0 * W + i1;
    idx4[2] = (j0 + 1) * W + i0;
    idx4[3] = (j0 + 1) * W + i1;
    w4[0] = (1.0 - fu) * (1.0 - fv);
    w4[1] = fu * (1.0 - fv);
    w4[2] = (1.0 - fu) * fv;
    w4[3] = fu * fv;
}

// K:648-658 (_bg_fetch): texel-major accumulation of the 4 channels.
__device__ __forceinline__ void bg_fetch(const MsiDev &B, int layer, const int *idx4,
                                         const double *w4, double *out4) {
    out4[0] = out4[1] = out4[2] = out4[3] = 0.0;
    const double4 *base = reinterpret_cast<const double4 *>(B.data) + (int64_t)layer * B.H * B.W;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double2 *tp = reinterpret_cast<const double2 *>(base + idx4[q]);
        const double2 ta = __ldg(tp), tb = __ldg(tp + 1);
        const double4 tx = make_double4(ta.x, ta.y, tb.x, tb.y);
        out4[0] += w4[q] * tx.x;
        out4[1] += w4[q] * tx.y;
        out4[2] += w4[q] * tx.z;
        out4[3] += w4[q] * tx.w;
    }
}

}  // namespace plx
