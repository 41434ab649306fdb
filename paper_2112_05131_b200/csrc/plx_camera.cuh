// plx_camera.cuh -- rays generated on the device from (view, pixel) ids.
//
// The reference builds its training rays on the host once per dataset
// (camera.py:91-100 generate_rays, camera.py:103-134 to_ndc, camera.py:292-
// 314 all_rays: 96 bytes of float64 per ray).  Here a ray pool is the camera
// records plus the float32 ground-truth colours (12 B per ray); the kernels
// rebuild a ray from its pool row whenever they need it, in the reference's
// float64 operation order (translation units are compiled -fmad=false; the
// matmul's FMAs below are explicit, matching numpy's OpenBLAS dgemm), so the
// rays are bit-identical to the reference's arrays.
#pragma once

#include <stdint.h>

#include "../../include/plx.h"

namespace plx {

struct CamPool {
    const double *cams;      // [n_views][PLX_CAM]
    const float *rgb;        // [pool rows][3] or nullptr
    const int64_t *pixel;    // optional global pixel id per pool row
    int64_t ppv, W, H;       // pixels per view, width, height
    int ndc;
    double scale;
};

inline CamPool make_campool(const plx_cameras *c) {
    CamPool p{};
    if (!c) return p;
    p.cams = c->cams;
    p.rgb = c->rgb;
    p.pixel = c->pixel;
    p.W = c->width;
    p.H = c->height;
    p.ppv = c->width * c->height;
    p.ndc = c->ndc;
    p.scale = c->scale;
    return p;
}

// camera.py:91-100 for one pixel: world origin and unit direction.
//   xs = (i + 0.5 - W/2) / f,   ys = -(j + 0.5 - H/2) / f
//   d  = d_cam @ R^T, d_cam = (x, y, -1): numpy's (N,3)@(3,3) runs OpenBLAS
//        dgemm, whose k loop accumulates with FMAs from zero
//   d /= sqrt((d0 d0 + d1 d1) + d2 d2)           (np.linalg.norm, axis=-1)
__device__ __forceinline__ const double *cam_pixel_ray(const CamPool &C, int64_t row, double *o,
                                                      double *d) {
    const int64_t gp = C.pixel ? C.pixel[row] : row;
    const int64_t view = gp / C.ppv, p = gp - view * C.ppv;
    const int64_t j = p / C.W, i = p - j * C.W;
    const double *cam = C.cams + view * PLX_CAM;
    const double f = cam[12];
    const double x = (((double)i + 0.5) - cam[13] / 2.0) / f;
    const double y = (-(((double)j + 0.5) - cam[14] / 2.0)) / f;
    double v[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double *r = cam + 4 * a;
        v[a] = fma(-1.0, r[2], fma(y, r[1], x * r[0]));
    }
    const double nrm = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        d[a] = v[a] / nrm;
        o[a] = cam[4 * a + 3];
    }
    return cam;
}

// camera.py:103-134 (to_ndc) of one world ray in place; returns valid.
__device__ __forceinline__ bool cam_to_ndc(const double *cam, double *o, double *d) {
    double near = cam[15];
    if (near <= 0.0) near = 1.0;
    const bool ok = fabs(d[2]) > 1e-10;
    const double dz = ok ? d[2] : 1.0;
    const double t = -(near + o[2]) / dz;
    const double p0 = o[0] + t * d[0], p1 = o[1] + t * d[1], p2 = o[2] + t * d[2];
    const double oz = fabs(p2) > 1e-12 ? p2 : -1e-12;
    const double fx = cam[12] / (cam[13] / 2.0), fy = cam[12] / (cam[14] / 2.0);
    const double dn0 = -fx * (d[0] / dz - p0 / oz);
    const double dn1 = -fy * (d[1] / dz - p1 / oz);
    const double dn2 = -2.0 * near / oz;
    o[0] = -fx * p0 / oz;
    o[1] = -fy * p1 / oz;
    o[2] = 1.0 + 2.0 * near / oz;
    d[0] = dn0;
    d[1] = dn1;
    d[2] = dn2;
    return ok;
}

// The march ray (origin, direction) of pool row `row`: all_rays (camera.py:
// 292-314) -- NDC-warped for forward-facing pools, origins pre-scaled for
// 360 pools (T:375-377).
__device__ __forceinline__ void cam_march_ray(const CamPool &C, int64_t row, double *o,
                                              double *d) {
    const double *cam = cam_pixel_ray(C, row, o, d);
    if (C.scale != 1.0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) o[a] = o[a] * C.scale;
    }
    if (C.ndc) cam_to_ndc(cam, o, d);
}

// The view (SH) direction of pool row `row`: the unit world direction.
__device__ __forceinline__ void cam_view_dir(const CamPool &C, int64_t row, double *v) {
    double o[3];
    cam_pixel_ray(C, row, o, v);
}

}  // namespace plx
