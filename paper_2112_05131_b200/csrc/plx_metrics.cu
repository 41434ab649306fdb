// plx_metrics.cu -- evaluation metrics on the device:
// losses.psnr / losses.ssim (pkg/src/plenoxel/losses.py:110-165) of one
// rendered view, so trainer.evaluate (T:309-347) copies back two scalars per
// view instead of the image.
//
// SSIM: an 11x11 separable Gaussian (sigma 1.5) with scipy's correlate1d
// zero padding, axis 0 then axis 1, statistics over the valid interior
// [5:-5, 5:-5].  For interior outputs every tap lies inside the image, so
// the padding never enters: pass 1 filters the five moments (x, y, xx, yy,
// xy) along axis 0 for the interior rows, pass 2 filters them along axis 1
// for the interior columns, forms the SSIM map and reduces it.  float64
// throughout (the summation order differs from scipy's: ~1e-16 relative).
#include <cuda_runtime.h>

#include "../../include/plx.h"

namespace {

constexpr int R = 5, K = 2 * R + 1;

struct Window {
    double w[K];
};

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// sum (a - b)^2 over all n values
__global__ void sq_err_kernel(const double *a, const double *b, int64_t n, double *out) {
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double d = a[i] - b[i];
        s += d * d;
    }
    s = warp_sum_d(s);
    if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(out, s);
}

// pass 1: m[q][r][x][ch] (q = moment, r = interior row index) filtered along
// axis 0.  Layout: 5 planes of (h - 10) x w x c.
__global__ void ssim_rows_kernel(const double *a, const double *b, int64_t h, int64_t w, int64_t c,
                                 Window win, double *m) {
    const int64_t hi = h - 2 * R, plane = hi * w * c;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < plane;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ch = t % c, x = (t / c) % w, r = t / (c * w);
        double sx = 0.0, sy = 0.0, sxx = 0.0, syy = 0.0, sxy = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int64_t i = ((r + k) * w + x) * c + ch;   // row (r + R) + (k - R)
            const double xv = a[i], yv = b[i], wk = win.w[k];
            sx += wk * xv;
            sy += wk * yv;
            sxx += wk * (xv * xv);
            syy += wk * (yv * yv);
            sxy += wk * (xv * yv);
        }
        m[t] = sx;
        m[plane + t] = sy;
        m[2 * plane + t] = sxx;
        m[3 * plane + t] = syy;
        m[4 * plane + t] = sxy;
    }
}

// pass 2: filter along axis 1 at the interior columns, the SSIM map
// (losses.py:155-162), summed.
__global__ void ssim_cols_kernel(const double *m, int64_t h, int64_t w, int64_t c, Window win,
                                 double c1, double c2, double *out) {
    const int64_t hi = h - 2 * R, wi = w - 2 * R, plane = hi * w * c;
    const int64_t n = hi * wi * c;
    double acc = 0.0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ch = t % c, x = (t / c) % wi, r = t / (c * wi);
        double mu[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int64_t i = (r * w + (x + k)) * c + ch;    // column (x + R) + (k - R)
            const double wk = win.w[k];
#pragma unroll
            for (int q = 0; q < 5; ++q) mu[q] += wk * m[q * plane + i];
        }
        const double mx = mu[0], my = mu[1];
        const double vx = mu[2] - mx * mx, vy = mu[3] - my * my, cov = mu[4] - mx * my;
        const double num = (2.0 * mx * my + c1) * (2.0 * cov + c2);
        const double den = (mx * mx + my * my + c1) * (vx + vy + c2);
        acc += num / den;
    }
    acc = warp_sum_d(acc);
    if ((threadIdx.x & 31) == 0 && acc != 0.0) atomicAdd(out + 1, acc);
}

int grid_for(int64_t n) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    int64_t b = (n + 255) / 256;
    if (b > (int64_t)sms * 8) b = (int64_t)sms * 8;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

extern "C" int64_t plx_image_metrics_scratch_bytes(int64_t h, int64_t w, int64_t c) {
    if (h <= 2 * R || w <= 2 * R || c < 1) return -1;
    return 5 * (h - 2 * R) * w * c * (int64_t)sizeof(double);
}

extern "C" int plx_image_metrics(const double *a, const double *b, int64_t h, int64_t w, int64_t c,
                                 const double *window, double k1, double k2, double *out_sums,
                                 void *scratch, int64_t scratch_bytes, void *stream) {
    if (!a || !b || !out_sums || h < 1 || w < 1 || c < 1) return PLX_EINVAL;
    // losses.py:136-137: the SSIM window must fit the image (window == NULL:
    // the squared error alone, any size)
    if (window && (h <= 2 * R || w <= 2 * R)) return PLX_EINVAL;
    if (window && (!scratch || scratch_bytes < plx_image_metrics_scratch_bytes(h, w, c)))
        return PLX_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = h * w * c;
    sq_err_kernel<<<grid_for(n), 256, 0, s>>>(a, b, n, out_sums);
    if (!window) return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA;
    Window win;
    for (int k = 0; k < K; ++k) win.w[k] = window[k];
    double *m = reinterpret_cast<double *>(scratch);
    ssim_rows_kernel<<<grid_for((h - 2 * R) * w * c), 256, 0, s>>>(a, b, h, w, c, win, m);
    ssim_cols_kernel<<<grid_for((h - 2 * R) * (w - 2 * R) * c), 256, 0, s>>>(
        m, h, w, c, win, k1 * k1, k2 * k2, out_sums);
    return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA;
}
