/*
 * plx_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A sequential, double-precision CPU restatement of the Plenoxels optimisation
 * hot path of the reference package `plenoxel` (arxiv 2112.05131 reference,
 * pkg/src/plenoxel/_kernels.py lines 27-600 and grid.py lines 154-285).
 * It is the CHECKER that the CUDA path in paper_2112_05131_b200/ is compared
 * against; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load it.  The product path never calls it.
 *
 * Pinning: tests/test_oracle_golden.py checks every function below against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py
 * imports /root/reference/pkg/src/plenoxel and runs its numba kernels).
 *
 * Floating point: the reference's numba kernels are compiled without fast-math
 * (no FMA contraction), so this file must be compiled with -ffp-contract=off
 * and keeps the reference's operation order everywhere; libm exp/log/sqrt are
 * the same functions numba binds to.  Outputs match the reference bit-for-bit
 * on the golden cases (see the test), except where noted (upsample values use
 * a left-to-right 8-term sum; numpy's einsum order is unspecified).
 *
 * Layout conventions (identical to the reference, K:1-12, G:71-92):
 *   links  int32 [Dx*Dy*Dz]  C-order (z fastest), -1 = empty
 *   table  f64   [rows*28]   col 0 sigma, cols 1..27 SH channel-major
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ROW 28

/* sh.py:18-22 */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2_0 = 1.0925484305920792;
static const double SH_C2_2 = 0.31539156525252005;
static const double SH_C2_4 = 0.5462742152960396;

/* K:27-37 */
static void sh_basis9(double x, double y, double z, double *out) {
    out[0] = SH_C0;
    out[1] = -SH_C1 * y;
    out[2] = SH_C1 * z;
    out[3] = -SH_C1 * x;
    out[4] = SH_C2_0 * x * y;
    out[5] = -SH_C2_0 * y * z;
    out[6] = SH_C2_2 * (2.0 * z * z - x * x - y * y);
    out[7] = -SH_C2_0 * x * z;
    out[8] = SH_C2_4 * (x * x - y * y);
}

/* K:40-81: clip to the AABB; t0 >= 0; miss iff t1 <= t0 */
static void ray_aabb(const double *o, const double *d, const double *lo,
                     const double *hi, double *pt0, double *pt1) {
    double t0 = 0.0, t1 = INFINITY;
    for (int a = 0; a < 3; ++a) {
        if (fabs(d[a]) < 1e-15) {
            if (o[a] < lo[a] || o[a] > hi[a]) {
                *pt0 = 1.0;
                *pt1 = 0.0;
                return;
            }
        } else {
            double ta = (lo[a] - o[a]) / d[a];
            double tb = (hi[a] - o[a]) / d[a];
            if (ta > tb) {
                double tmp = ta;
                ta = tb;
                tb = tmp;
            }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        }
    }
    *pt0 = t0;
    *pt1 = t1;
}

/* K:163-170 */
static inline double clamp_coord(double p, double lo, double scale, double dmax) {
    double g = (p - lo) * scale;
    if (g < 0.0) g = 0.0;
    if (g > dmax) g = dmax;
    return g;
}

/* K:84-123 */
static int stencil(double gx, double gy, double gz, const int32_t *links,
                   int64_t Dx, int64_t Dy, int64_t Dz, int nearest,
                   int64_t *rows, double *ws) {
    if (nearest) {
        int64_t i = (int64_t)(gx + 0.5), j = (int64_t)(gy + 0.5), k = (int64_t)(gz + 0.5);
        if (i > Dx - 1) i = Dx - 1;
        if (j > Dy - 1) j = Dy - 1;
        if (k > Dz - 1) k = Dz - 1;
        rows[0] = links[(i * Dy + j) * Dz + k];
        ws[0] = 1.0;
        return 1;
    }
    int64_t i0 = (int64_t)gx, j0 = (int64_t)gy, k0 = (int64_t)gz;
    if (i0 > Dx - 2) i0 = Dx - 2;
    if (j0 > Dy - 2) j0 = Dy - 2;
    if (k0 > Dz - 2) k0 = Dz - 2;
    double fx = gx - (double)i0, fy = gy - (double)j0, fz = gz - (double)k0;
    int n = 0;
    for (int di = 0; di < 2; ++di) {
        double wx = di == 1 ? fx : 1.0 - fx;
        for (int dj = 0; dj < 2; ++dj) {
            double wy = dj == 1 ? fy : 1.0 - fy;
            for (int dk = 0; dk < 2; ++dk) {
                double wz = dk == 1 ? fz : 1.0 - fz;
                rows[n] = links[((i0 + di) * Dy + (j0 + dj)) * Dz + (k0 + dk)];
                ws[n] = wx * wy * wz;
                ++n;
            }
        }
    }
    return 8;
}

/* K:126-135 */
static double sigma_at(const double *table, const int64_t *rows, const double *ws,
                       int n, int *occ) {
    double s = 0.0;
    *occ = 0;
    for (int q = 0; q < n; ++q) {
        int64_t r = rows[q];
        if (r >= 0) {
            *occ = 1;
            s += ws[q] * table[r * ROW];
        }
    }
    return s;
}

/* K:138-152 */
static void color_at(const double *table, const int64_t *rows, const double *ws,
                     int n, const double *basis, double *out3) {
    out3[0] = out3[1] = out3[2] = 0.0;
    for (int q = 0; q < n; ++q) {
        int64_t r = rows[q];
        if (r >= 0) {
            double w = ws[q];
            for (int ch = 0; ch < 3; ++ch) {
                double acc = 0.0;
                int base = 1 + 9 * ch;
                for (int b = 0; b < 9; ++b) acc += basis[b] * table[r * ROW + base + b];
                out3[ch] += w * acc;
            }
        }
    }
}

/* K:155-160 */
static inline void touch(int64_t row, uint8_t *tmask, int64_t *tids, int64_t *tcnt) {
    if (tmask[row] == 0) {
        tmask[row] = 1;
        tids[tcnt[0]] = row;
        tcnt[0] += 1;
    }
}

typedef struct {
    const int32_t *links;
    int64_t Dx, Dy, Dz;
    const double *table;
    const double *lo, *hi, *scale, *dmax;
    double step;
} grid_t;

/* K:173-238 */
void oracle_render_forward(const int32_t *links, int64_t Dx, int64_t Dy, int64_t Dz,
                           const double *table, const double *lo, const double *hi,
                           const double *scale, const double *dmax, double step,
                           const double *origins, const double *dirs,
                           const double *viewdirs, int64_t nray, const double *bg,
                           double stop_thresh, int nearest, int absolute,
                           const double *jitter_t, double *out_rgb, double *out_trans,
                           double *out_wsum) {
    int64_t rows[8];
    double ws[8], basis[9], col[3];
    for (int64_t ri = 0; ri < nray; ++ri) {
        const double *o = origins + 3 * ri, *d = dirs + 3 * ri, *vd = viewdirs + 3 * ri;
        sh_basis9(vd[0], vd[1], vd[2], basis);
        double t0, t1;
        ray_aabb(o, d, lo, hi, &t0, &t1);
        double cr = 0.0, cg = 0.0, cb = 0.0, T = 1.0, asum = 0.0, wsum = 0.0;
        t0 = t0 + jitter_t[ri] * step;
        double L = t1 - t0;
        if (L > 0.0) {
            int64_t nsamp = (int64_t)ceil(L / step - 1e-9);
            if (nsamp < 1) nsamp = 1;
            for (int64_t si = 0; si < nsamp; ++si) {
                double t = t0 + (double)si * step;
                double dlt = si < nsamp - 1 ? step : L - step * (double)(nsamp - 1);
                double gx = clamp_coord(o[0] + t * d[0], lo[0], scale[0], dmax[0]);
                double gy = clamp_coord(o[1] + t * d[1], lo[1], scale[1], dmax[1]);
                double gz = clamp_coord(o[2] + t * d[2], lo[2], scale[2], dmax[2]);
                int n = stencil(gx, gy, gz, links, Dx, Dy, Dz, nearest, rows, ws);
                int occ;
                double sig = sigma_at(table, rows, ws, n, &occ);
                if (!occ || sig <= 0.0) continue;
                double att = exp(-sig * dlt);
                double Tn, w;
                if (absolute) {
                    Tn = 1.0 - (asum + (1.0 - att));
                    if (Tn < 0.0) Tn = 0.0;
                    w = T - Tn;
                    asum += 1.0 - att;
                } else {
                    Tn = T * att;
                    w = T - Tn;
                }
                color_at(table, rows, ws, n, basis, col);
                if (col[0] > 0.0) cr += w * col[0];
                if (col[1] > 0.0) cg += w * col[1];
                if (col[2] > 0.0) cb += w * col[2];
                wsum += w;
                T = Tn;
                if (T < stop_thresh) break;
            }
        }
        out_rgb[3 * ri + 0] = cr + T * bg[0];
        out_rgb[3 * ri + 1] = cg + T * bg[1];
        out_rgb[3 * ri + 2] = cb + T * bg[2];
        out_trans[ri] = T;
        out_wsum[ri] = wsum;
    }
}

/* K:241-411.  Scratch buffers are allocated here (nmax from the caller,
 * R:67-69).  out_sums[0] = mse_sum, out_sums[1] = cauchy_sum. */
void oracle_render_backward(const int32_t *links, int64_t Dx, int64_t Dy, int64_t Dz,
                            const double *table, const double *lo, const double *hi,
                            const double *scale, const double *dmax, double step,
                            const double *origins, const double *dirs,
                            const double *viewdirs, int64_t nray, const double *bg,
                            double stop_thresh, int nearest, int absolute,
                            const double *jitter_t, const double *target, int mse_mode,
                            double up_scale, double lam_cauchy, double *grad,
                            uint8_t *tmask, int64_t *tids, int64_t *tcnt,
                            double *out_rgb, int64_t nmax, double *out_sums) {
    int64_t rows[8];
    double ws[8], basis[9], col[3];
    double *s_t = malloc(sizeof(double) * nmax), *s_dlt = malloc(sizeof(double) * nmax);
    double *s_sig = malloc(sizeof(double) * nmax), *s_T = malloc(sizeof(double) * nmax);
    double *s_w = malloc(sizeof(double) * nmax), *s_cpre = malloc(sizeof(double) * nmax * 3);
    double mse_sum = 0.0, cauchy_sum = 0.0;
    for (int64_t ri = 0; ri < nray; ++ri) {
        const double *o = origins + 3 * ri, *d = dirs + 3 * ri, *vd = viewdirs + 3 * ri;
        sh_basis9(vd[0], vd[1], vd[2], basis);
        double t0, t1;
        ray_aabb(o, d, lo, hi, &t0, &t1);
        double cr = 0.0, cg = 0.0, cb = 0.0, T = 1.0, asum = 0.0;
        int64_t m = 0;
        t0 = t0 + jitter_t[ri] * step;
        double L = t1 - t0;
        if (L > 0.0) {
            int64_t nsamp = (int64_t)ceil(L / step - 1e-9);
            if (nsamp < 1) nsamp = 1;
            for (int64_t si = 0; si < nsamp; ++si) {
                double t = t0 + (double)si * step;
                double dlt = si < nsamp - 1 ? step : L - step * (double)(nsamp - 1);
                double gx = clamp_coord(o[0] + t * d[0], lo[0], scale[0], dmax[0]);
                double gy = clamp_coord(o[1] + t * d[1], lo[1], scale[1], dmax[1]);
                double gz = clamp_coord(o[2] + t * d[2], lo[2], scale[2], dmax[2]);
                int n = stencil(gx, gy, gz, links, Dx, Dy, Dz, nearest, rows, ws);
                int occ;
                double sig = sigma_at(table, rows, ws, n, &occ);
                if (!occ || sig < 0.0) continue;
                double att = exp(-sig * dlt);
                double Tn, w;
                if (absolute) {
                    Tn = 1.0 - (asum + (1.0 - att));
                    if (Tn < 0.0) Tn = 0.0;
                    w = T - Tn;
                    asum += 1.0 - att;
                } else {
                    Tn = T * att;
                    w = T - Tn;
                }
                color_at(table, rows, ws, n, basis, col);
                if (col[0] > 0.0) cr += w * col[0];
                if (col[1] > 0.0) cg += w * col[1];
                if (col[2] > 0.0) cb += w * col[2];
                s_t[m] = t;
                s_dlt[m] = dlt;
                s_sig[m] = sig;
                s_T[m] = T;
                s_w[m] = w;
                s_cpre[3 * m + 0] = col[0];
                s_cpre[3 * m + 1] = col[1];
                s_cpre[3 * m + 2] = col[2];
                ++m;
                T = Tn;
                if (T < stop_thresh) break;
            }
        }
        double rr = cr + T * bg[0], rg = cg + T * bg[1], rb = cb + T * bg[2];
        out_rgb[3 * ri + 0] = rr;
        out_rgb[3 * ri + 1] = rg;
        out_rgb[3 * ri + 2] = rb;
        double upr, upg, upb;
        if (mse_mode) {
            double er = rr - target[3 * ri + 0];
            double eg = rg - target[3 * ri + 1];
            double eb = rb - target[3 * ri + 2];
            mse_sum += er * er + eg * eg + eb * eb;
            upr = up_scale * er;
            upg = up_scale * eg;
            upb = up_scale * eb;
        } else {
            upr = target[3 * ri + 0];
            upg = target[3 * ri + 1];
            upb = target[3 * ri + 2];
        }
        double sfr, sfg, sfb;
        if (absolute) {
            double bend = T > 0.0 ? 1.0 : 0.0;
            sfr = -bg[0] * bend;
            sfg = -bg[1] * bend;
            sfb = -bg[2] * bend;
        } else {
            sfr = T * bg[0];
            sfg = T * bg[1];
            sfb = T * bg[2];
        }
        for (int64_t idx = m - 1; idx >= 0; --idx) {
            double sig = s_sig[idx], dlt = s_dlt[idx], Ti = s_T[idx], w = s_w[idx];
            double c0 = s_cpre[3 * idx], c1 = s_cpre[3 * idx + 1], c2 = s_cpre[3 * idx + 2];
            double ccr = c0 > 0.0 ? c0 : 0.0, ccg = c1 > 0.0 ? c1 : 0.0, ccb = c2 > 0.0 ? c2 : 0.0;
            double att = exp(-sig * dlt);
            double gsig;
            if (absolute) {
                double Tn = Ti - w;
                double bn = Tn > 0.0 ? 1.0 : 0.0;
                double bi = Ti > 0.0 ? 1.0 : 0.0;
                double galpha = (upr * (ccr * bn + sfr) + upg * (ccg * bn + sfg) +
                                 upb * (ccb * bn + sfb));
                gsig = galpha * dlt * att;
                sfr += ccr * (bn - bi);
                sfg += ccg * (bn - bi);
                sfb += ccb * (bn - bi);
            } else {
                gsig = dlt * (upr * (Ti * att * ccr - sfr) + upg * (Ti * att * ccg - sfg) +
                              upb * (Ti * att * ccb - sfb));
                sfr += w * ccr;
                sfg += w * ccg;
                sfb += w * ccb;
            }
            if (lam_cauchy > 0.0) {
                cauchy_sum += log(1.0 + 2.0 * sig * sig);
                gsig += lam_cauchy * 4.0 * sig / (1.0 + 2.0 * sig * sig);
            }
            double gcr = c0 > 0.0 ? upr * w : 0.0;
            double gcg = c1 > 0.0 ? upg * w : 0.0;
            double gcb = c2 > 0.0 ? upb * w : 0.0;
            double t = s_t[idx];
            double gx = clamp_coord(o[0] + t * d[0], lo[0], scale[0], dmax[0]);
            double gy = clamp_coord(o[1] + t * d[1], lo[1], scale[1], dmax[1]);
            double gz = clamp_coord(o[2] + t * d[2], lo[2], scale[2], dmax[2]);
            int n = stencil(gx, gy, gz, links, Dx, Dy, Dz, nearest, rows, ws);
            for (int q = 0; q < n; ++q) {
                int64_t rw = rows[q];
                if (rw < 0) continue;
                double wq = ws[q];
                touch(rw, tmask, tids, tcnt);
                double *gr = grad + rw * ROW;
                gr[0] += wq * gsig;
                if (gcr != 0.0)
                    for (int b = 0; b < 9; ++b) gr[1 + b] += wq * gcr * basis[b];
                if (gcg != 0.0)
                    for (int b = 0; b < 9; ++b) gr[10 + b] += wq * gcg * basis[b];
                if (gcb != 0.0)
                    for (int b = 0; b < 9; ++b) gr[19 + b] += wq * gcb * basis[b];
            }
        }
    }
    free(s_t); free(s_dlt); free(s_sig); free(s_T); free(s_w); free(s_cpre);
    out_sums[0] = mse_sum;
    out_sums[1] = cauchy_sum;
}

/* K:414-453 */
void oracle_max_weight_accum(const int32_t *links, int64_t Dx, int64_t Dy, int64_t Dz,
                             const double *table, const double *lo, const double *hi,
                             const double *scale, const double *dmax, double step,
                             const double *origins, const double *dirs, int64_t nray,
                             double stop_thresh, int nearest, double *out_w) {
    int64_t rows[8];
    double ws[8];
    for (int64_t ri = 0; ri < nray; ++ri) {
        const double *o = origins + 3 * ri, *d = dirs + 3 * ri;
        double t0, t1;
        ray_aabb(o, d, lo, hi, &t0, &t1);
        double L = t1 - t0;
        if (L <= 0.0) continue;
        double T = 1.0;
        int64_t nsamp = (int64_t)ceil(L / step - 1e-9);
        if (nsamp < 1) nsamp = 1;
        for (int64_t si = 0; si < nsamp; ++si) {
            double t = t0 + (double)si * step;
            double dlt = si < nsamp - 1 ? step : L - step * (double)(nsamp - 1);
            double gx = clamp_coord(o[0] + t * d[0], lo[0], scale[0], dmax[0]);
            double gy = clamp_coord(o[1] + t * d[1], lo[1], scale[1], dmax[1]);
            double gz = clamp_coord(o[2] + t * d[2], lo[2], scale[2], dmax[2]);
            int n = stencil(gx, gy, gz, links, Dx, Dy, Dz, nearest, rows, ws);
            int occ;
            double sig = sigma_at(table, rows, ws, n, &occ);
            if (!occ || sig <= 0.0) continue;
            double att = exp(-sig * dlt);
            double w = T * (1.0 - att);
            for (int q = 0; q < n; ++q) {
                int64_t r = rows[q];
                if (r >= 0 && w > out_w[r]) out_w[r] = w;
            }
            T *= att;
            if (T < stop_thresh) break;
        }
    }
}

/* K:456-569.  out_sums[0] = sigma sum, out_sums[1] = sh sum (raw). */
void oracle_tv_grid(const int32_t *links, int64_t Dx, int64_t Dy, int64_t Dz,
                    const double *table, const int64_t *cells, int64_t ncell,
                    double fac_x, double fac_y, double fac_z, double eps,
                    double f_sigma, double f_sh, int wrap_x, int wrap_y, int wrap_z,
                    double *grad, uint8_t *tmask, int64_t *tids, int64_t *tcnt,
                    int with_grad, double *out_sums) {
    double sig_sum = 0.0, sh_sum = 0.0, e2 = eps * eps;
    for (int64_t ci = 0; ci < ncell; ++ci) {
        int64_t cid = cells[ci];
        int64_t i = cid / (Dy * Dz), rem = cid % (Dy * Dz);
        int64_t j = rem / Dz, k = rem % Dz;
        int64_t r0 = links[(i * Dy + j) * Dz + k];
        int64_t ii = i + 1, jj = j + 1, kk = k + 1;
        int hx = 1, hy = 1, hz = 1;
        if (ii >= Dx) { if (wrap_x) ii = 0; else hx = 0; }
        if (jj >= Dy) { if (wrap_y) jj = 0; else hy = 0; }
        if (kk >= Dz) { if (wrap_z) kk = 0; else hz = 0; }
        int64_t rx = hx ? links[(ii * Dy + j) * Dz + k] : -1;
        int64_t ry = hy ? links[(i * Dy + jj) * Dz + k] : -1;
        int64_t rz = hz ? links[(i * Dy + j) * Dz + kk] : -1;
        double s0 = r0 >= 0 ? table[r0 * ROW] : 0.0;
        double sx = rx >= 0 ? table[rx * ROW] : 0.0;
        double sy = ry >= 0 ? table[ry * ROW] : 0.0;
        double sz = rz >= 0 ? table[rz * ROW] : 0.0;
        double dxv = (sx - s0) * fac_x, dyv = (sy - s0) * fac_y, dzv = (sz - s0) * fac_z;
        double val = sqrt(dxv * dxv + dyv * dyv + dzv * dzv + e2);
        sig_sum += val;
        if (with_grad && val > 0.0) {
            double inv = f_sigma / val, g0 = 0.0;
            if (rx >= 0) { touch(rx, tmask, tids, tcnt); grad[rx * ROW] += dxv * fac_x * inv; }
            g0 -= dxv * fac_x * inv;
            if (ry >= 0) { touch(ry, tmask, tids, tcnt); grad[ry * ROW] += dyv * fac_y * inv; }
            g0 -= dyv * fac_y * inv;
            if (rz >= 0) { touch(rz, tmask, tids, tcnt); grad[rz * ROW] += dzv * fac_z * inv; }
            g0 -= dzv * fac_z * inv;
            if (r0 >= 0 && g0 != 0.0) { touch(r0, tmask, tids, tcnt); grad[r0 * ROW] += g0; }
        }
        if (r0 >= 0) {
            int okx = rx >= 0, oky = ry >= 0, okz = rz >= 0;
            if (okx || oky || okz) {
                for (int dd = 1; dd < 28; ++dd) {
                    double v0 = table[r0 * ROW + dd];
                    double ax = okx ? (table[rx * ROW + dd] - v0) * fac_x : 0.0;
                    double ay = oky ? (table[ry * ROW + dd] - v0) * fac_y : 0.0;
                    double az = okz ? (table[rz * ROW + dd] - v0) * fac_z : 0.0;
                    double v = sqrt(ax * ax + ay * ay + az * az + e2);
                    sh_sum += v;
                    if (with_grad && v > 0.0) {
                        double inv = f_sh / v, g0 = 0.0;
                        if (okx) { touch(rx, tmask, tids, tcnt); grad[rx * ROW + dd] += ax * fac_x * inv; g0 -= ax * fac_x * inv; }
                        if (oky) { touch(ry, tmask, tids, tcnt); grad[ry * ROW + dd] += ay * fac_y * inv; g0 -= ay * fac_y * inv; }
                        if (okz) { touch(rz, tmask, tids, tcnt); grad[rz * ROW + dd] += az * fac_z * inv; g0 -= az * fac_z * inv; }
                        if (g0 != 0.0) { touch(r0, tmask, tids, tcnt); grad[r0 * ROW + dd] += g0; }
                    }
                }
            } else {
                sh_sum += 27.0 * eps;
            }
        } else {
            sh_sum += 27.0 * eps;
        }
    }
    out_sums[0] = sig_sum;
    out_sums[1] = sh_sum;
}

/* K:572-590 */
void oracle_opt_step(double *table, double *v, const double *grad, const int64_t *tids,
                     int64_t nt, int64_t ncol, double lr_first, double lr_rest,
                     double beta, double eps, int rmsprop) {
    for (int64_t q = 0; q < nt; ++q) {
        int64_t r = tids[q];
        for (int64_t c = 0; c < ncol; ++c) {
            double g = grad[r * ncol + c];
            if (g == 0.0) continue;
            double lr = c == 0 ? lr_first : lr_rest;
            if (rmsprop) {
                double nv = beta * v[r * ncol + c] + (1.0 - beta) * g * g;
                v[r * ncol + c] = nv;
                table[r * ncol + c] -= lr * g / (sqrt(nv) + eps);
            } else {
                table[r * ncol + c] -= lr * g;
            }
        }
    }
}

/* K:593-600 */
void oracle_clear_grad(double *grad, uint8_t *tmask, int64_t *tids, int64_t *tcnt,
                       int64_t ncol) {
    for (int64_t q = 0; q < tcnt[0]; ++q) {
        int64_t r = tids[q];
        tmask[r] = 0;
        for (int64_t c = 0; c < ncol; ++c) grad[r * ncol + c] = 0.0;
    }
    tcnt[0] = 0;
}

/* G:228-258 (scipy.ndimage.binary_dilation with a 3x3x3 box and the default
 * border_value=0, then C-order compaction).  value: per-row criterion
 * (weights, or NULL for density = table[:,0]).  Returns n_keep; writes
 * new_links (cells) and kept_old (n_keep, caller sizes it >= rows). */
int64_t oracle_prune(const int32_t *links, int64_t Dx, int64_t Dy, int64_t Dz,
                     const double *table, const double *weights, double threshold,
                     int32_t *new_links, int64_t *kept_old) {
    int64_t ncell = Dx * Dy * Dz;
    uint8_t *deemed = calloc((size_t)ncell, 1);
    for (int64_t c = 0; c < ncell; ++c) {
        int32_t r = links[c];
        if (r < 0) continue;
        double val = weights ? weights[r] : table[(int64_t)r * ROW];
        deemed[c] = val >= threshold;
    }
    int64_t n_keep = 0;
    for (int64_t i = 0; i < Dx; ++i)
        for (int64_t j = 0; j < Dy; ++j)
            for (int64_t k = 0; k < Dz; ++k) {
                int64_t c = (i * Dy + j) * Dz + k;
                new_links[c] = -1;
                if (links[c] < 0) continue;
                int dil = 0;
                for (int64_t a = i - 1; a <= i + 1 && !dil; ++a) {
                    if (a < 0 || a >= Dx) continue;
                    for (int64_t b = j - 1; b <= j + 1 && !dil; ++b) {
                        if (b < 0 || b >= Dy) continue;
                        for (int64_t e = k - 1; e <= k + 1; ++e) {
                            if (e < 0 || e >= Dz) continue;
                            if (deemed[(a * Dy + b) * Dz + e]) { dil = 1; break; }
                        }
                    }
                }
                if (dil) {
                    new_links[c] = (int32_t)n_keep;
                    kept_old[n_keep] = links[c];
                    ++n_keep;
                }
            }
    free(deemed);
    return n_keep;
}

/* G:260-285 (and the numpy stencil G:154-180, same op order in f64).
 * Pass 1 (out_table == NULL): fills new_links, returns the row count.
 * Pass 2: also writes out_table (n_new*28 f64). */
int64_t oracle_upsample(const int32_t *links, int64_t Dx, int64_t Dy, int64_t Dz,
                        const double *table, const double *lo, const double *hi,
                        int64_t Nx, int64_t Ny, int64_t Nz, int32_t *new_links,
                        double *out_table) {
    double extent[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    double spacing[3] = {extent[0] / ((double)Nx - 1.0), extent[1] / ((double)Ny - 1.0),
                         extent[2] / ((double)Nz - 1.0)};
    double lscale[3] = {((double)Dx - 1.0) / extent[0], ((double)Dy - 1.0) / extent[1],
                        ((double)Dz - 1.0) / extent[2]};
    double dmax[3] = {(double)Dx - 1.0, (double)Dy - 1.0, (double)Dz - 1.0};
    int64_t dm2[3] = {Dx - 2, Dy - 2, Dz - 2};
    int64_t n_new = 0;
    for (int64_t i = 0; i < Nx; ++i)
        for (int64_t j = 0; j < Ny; ++j)
            for (int64_t k = 0; k < Nz; ++k) {
                double ijk[3] = {(double)i, (double)j, (double)k};
                double f[3];
                int64_t i0[3];
                for (int a = 0; a < 3; ++a) {
                    double p = lo[a] + ijk[a] * spacing[a];
                    double g = (p - lo[a]) * lscale[a];
                    if (g < 0.0) g = 0.0;
                    if (g > dmax[a]) g = dmax[a];
                    int64_t fl = (int64_t)floor(g);
                    i0[a] = fl < dm2[a] ? fl : dm2[a];
                    f[a] = g - (double)i0[a];
                }
                int64_t rows[8];
                double ws[8];
                int q = 0;
                for (int di = 0; di < 2; ++di) {
                    double wx = di ? f[0] : 1.0 - f[0];
                    for (int dj = 0; dj < 2; ++dj) {
                        double wy = dj ? f[1] : 1.0 - f[1];
                        for (int dk = 0; dk < 2; ++dk) {
                            double wz = dk ? f[2] : 1.0 - f[2];
                            rows[q] = links[((i0[0] + di) * Dy + (i0[1] + dj)) * Dz + (i0[2] + dk)];
                            ws[q] = wx * wy * wz;
                            ++q;
                        }
                    }
                }
                double occw = 0.0;
                for (q = 0; q < 8; ++q) occw += ws[q] * (rows[q] >= 0 ? 1.0 : 0.0);
                int64_t c = (i * Ny + j) * Nz + k;
                if (occw > 0.0) {
                    new_links[c] = (int32_t)n_new;
                    if (out_table) {
                        double *dst = out_table + n_new * ROW;
                        for (int cc = 0; cc < ROW; ++cc) {
                            double acc = 0.0;
                            for (q = 0; q < 8; ++q)
                                if (rows[q] >= 0) acc += ws[q] * table[rows[q] * ROW + cc];
                            dst[cc] = acc;
                        }
                    }
                    ++n_new;
                } else {
                    new_links[c] = -1;
                }
            }
    return n_new;
}

/* ------------------------------------------------------------------------
 * Multi-sphere-image background (360 scenes): K:603-977 and msi.py.
 * bg: f64 [L][H][W][4] (sigma, r, g, b); radii: f64[L], increasing, last inf.
 * ------------------------------------------------------------------------ */

/* K:606-645 (_bg_stencil): bilinear texel stencil within one layer at the
 * sphere angles of p; texel centres at half texels, phi wraps, theta clamps. */
static void bg_stencil(int64_t H, int64_t W, double px, double py, double pz,
                       int64_t *idx4, double *w4) {
    const double pi = 3.141592653589793;
    double r = sqrt(px * px + py * py + pz * pz);
    double phi = atan2(py, px);
    double ct = pz / r;
    if (ct > 1.0) ct = 1.0;
    if (ct < -1.0) ct = -1.0;
    double theta = acos(ct);
    double u = (phi + pi) / (2.0 * pi) * (double)W - 0.5;
    u = u - floor(u / (double)W) * (double)W;
    double vv = theta / pi * (double)H - 0.5;
    if (vv < 0.0) vv = 0.0;
    if (vv > (double)H - 1.0) vv = (double)H - 1.0;
    int64_t i0 = (int64_t)u;
    if (i0 > W - 1) i0 = W - 1;
    double fu = u - (double)i0;
    int64_t i1 = i0 + 1;
    if (i1 >= W) i1 = 0;
    int64_t j0 = (int64_t)vv;
    if (j0 > H - 2) j0 = H - 2;
    double fv = vv - (double)j0;
    idx4[0] = j0 * W + i0;
    idx4[1] = j0 * W + i1;
    idx4[2] = (j0 + 1) * W + i0;
    idx4[3] = (j0 + 1) * W + i1;
    w4[0] = (1.0 - fu) * (1.0 - fv);
    w4[1] = fu * (1.0 - fv);
    w4[2] = (1.0 - fu) * fv;
    w4[3] = fu * fv;
}

/* K:648-658 (_bg_fetch) */
static void bg_fetch(const double *bg, int64_t H, int64_t W, int64_t layer,
                     const int64_t *idx4, const double *w4, double *out4) {
    for (int c = 0; c < 4; ++c) out4[c] = 0.0;
    for (int q = 0; q < 4; ++q) {
        const double *tx = bg + ((layer * H * W) + idx4[q]) * 4;
        for (int c = 0; c < 4; ++c) out4[c] += w4[q] * tx[c];
    }
}

/* msi.py:75-108 (sample_background): trilinear over (inverse-radius layer
 * coordinate, theta, phi), terms summed in (layer, theta, phi) order, then
 * clamped at zero.  Returns -1 if a point lies inside the unit sphere. */
int oracle_bg_sample(const double *bg, int64_t L, int64_t H, int64_t W,
                     const double *pts, int64_t n, double *out4) {
    const double pi = 3.141592653589793;
    for (int64_t p = 0; p < n; ++p) {
        const double *q = pts + 3 * p;
        double r = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]);
        if (r < 1.0 - 1e-9) return -1;
        double phi = atan2(q[1], q[0]);
        double c = q[2] / r;
        if (c < -1.0) c = -1.0;
        if (c > 1.0) c = 1.0;
        double theta = acos(c);
        double u = (phi + pi) / (2.0 * pi) * (double)W - 0.5;
        u = u - floor(u / (double)W) * (double)W;
        double v = theta / pi * (double)H - 0.5;
        if (v < 0.0) v = 0.0;
        if (v > (double)H - 1.0) v = (double)H - 1.0;
        double lc = (1.0 - 1.0 / r) * (double)(L - 1);
        if (lc < 0.0) lc = 0.0;
        if (lc > (double)(L - 1)) lc = (double)(L - 1);
        int64_t l0 = (int64_t)floor(lc);
        if (l0 > L - 2) l0 = L - 2;
        double fl = lc - (double)l0;
        int64_t i0 = (int64_t)floor(u);
        if (i0 > W - 1) i0 = W - 1;
        double fu = u - (double)i0;
        int64_t i1 = (i0 + 1) % W;
        int64_t j0 = (int64_t)floor(v);
        if (j0 > H - 2) j0 = H - 2;
        double fv = v - (double)j0;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int dl = 0; dl < 2; ++dl) {
            double wl = dl ? fl : 1.0 - fl;
            for (int dj = 0; dj < 2; ++dj) {
                double wv = dj ? fv : 1.0 - fv;
                for (int di = 0; di < 2; ++di) {
                    double wu = di ? fu : 1.0 - fu;
                    int64_t ii = di ? i1 : i0;
                    const double *tx = bg + (((l0 + dl) * H + (j0 + dj)) * W + ii) * 4;
                    double w = wl * wv * wu;
                    for (int k = 0; k < 4; ++k) acc[k] += w * tx[k];
                }
            }
        }
        for (int k = 0; k < 4; ++k) out4[4 * p + k] = acc[k] > 0.0 ? acc[k] : 0.0;
    }
    return 0;
}

/* K:661-881 (render_backward_360): foreground grid then one background
 * sample per sphere crossing beyond the foreground exit, composited over
 * black; with_grad: the reverse sweep over the concatenated samples with the
 * Cauchy term (foreground) and the beta regulariser on the foreground
 * transmittance.  out_sums = {mse, cauchy_raw, beta_raw}. */
void oracle_render_360(const int32_t *links, int64_t Dx, int64_t Dy, int64_t Dz,
                       const double *table, const double *lo, const double *hi,
                       const double *scale, const double *dmax, double step,
                       const double *bg, int64_t L, int64_t H, int64_t W, const double *radii,
                       const double *origins, const double *dirs, int64_t nray,
                       double stop_thresh, int nearest, const double *target, int mse_mode,
                       double up_scale, double lam_cauchy, double lam_beta, double beta_eps,
                       double *grad, uint8_t *tmask, int64_t *tids, int64_t *tcnt,
                       double *bg_grad, uint8_t *bg_tmask, int64_t *bg_tids, int64_t *bg_tcnt,
                       double *out_rgb, double *out_tfg, double *out_trans, int64_t nmax,
                       int with_grad, double *out_sums) {
    int64_t rows[8], idx4[4], nx;
    double ws[8], basis[9], col[3], w4[4], out4[4];
    double *s_t = malloc(sizeof(double) * nmax), *s_dlt = malloc(sizeof(double) * nmax);
    double *s_sig = malloc(sizeof(double) * nmax), *s_T = malloc(sizeof(double) * nmax);
    double *s_w = malloc(sizeof(double) * nmax), *s_cpre = malloc(sizeof(double) * nmax * 3);
    int64_t *s_layer = malloc(sizeof(int64_t) * nmax);
    double *xs_t = malloc(sizeof(double) * (L > 0 ? L : 1));
    int64_t *xs_l = malloc(sizeof(int64_t) * (L > 0 ? L : 1));
    double mse_sum = 0.0, cauchy_sum = 0.0, beta_sum = 0.0;
    for (int64_t ri = 0; ri < nray; ++ri) {
        const double *o = origins + 3 * ri, *d = dirs + 3 * ri;
        sh_basis9(d[0], d[1], d[2], basis);
        double t0, t1;
        ray_aabb(o, d, lo, hi, &t0, &t1);
        double cr = 0.0, cg = 0.0, cb = 0.0, T = 1.0;
        int64_t m = 0;
        double Lf = t1 - t0;
        if (Lf > 0.0) {
            int64_t nsamp = (int64_t)ceil(Lf / step - 1e-9);
            if (nsamp < 1) nsamp = 1;
            for (int64_t si = 0; si < nsamp; ++si) {
                double t = t0 + (double)si * step;
                double dlt = si < nsamp - 1 ? step : Lf - step * (double)(nsamp - 1);
                double gx = clamp_coord(o[0] + t * d[0], lo[0], scale[0], dmax[0]);
                double gy = clamp_coord(o[1] + t * d[1], lo[1], scale[1], dmax[1]);
                double gz = clamp_coord(o[2] + t * d[2], lo[2], scale[2], dmax[2]);
                int n = stencil(gx, gy, gz, links, Dx, Dy, Dz, nearest, rows, ws);
                int occ;
                double sig = sigma_at(table, rows, ws, n, &occ);
                if (!occ || sig < 0.0) continue;
                double att = exp(-sig * dlt);
                double Tn = T * att, w = T - Tn;
                color_at(table, rows, ws, n, basis, col);
                if (col[0] > 0.0) cr += w * col[0];
                if (col[1] > 0.0) cg += w * col[1];
                if (col[2] > 0.0) cb += w * col[2];
                s_t[m] = t; s_dlt[m] = dlt; s_sig[m] = sig; s_T[m] = T; s_w[m] = w;
                s_cpre[3 * m] = col[0]; s_cpre[3 * m + 1] = col[1]; s_cpre[3 * m + 2] = col[2];
                s_layer[m] = -1;
                ++m;
                T = Tn;
                if (T < stop_thresh) break;
            }
        }
        double tfg = T;
        out_tfg[ri] = tfg;
        double t_exit = t1 > 0.0 ? t1 : 0.0;
        if (T >= stop_thresh) {
            double bdot = o[0] * d[0] + o[1] * d[1] + o[2] * d[2];
            double c0n = o[0] * o[0] + o[1] * o[1] + o[2] * o[2];
            nx = 0;
            for (int64_t l = 0; l < L - 1; ++l) {
                double rad = radii[l];
                double disc = bdot * bdot - c0n + rad * rad;
                if (disc <= 0.0) continue;
                double tl = -bdot + sqrt(disc);
                if (tl < t_exit) continue;
                xs_t[nx] = tl;
                xs_l[nx] = l;
                ++nx;
            }
            for (int64_t q = 0; q < nx; ++q) {
                double dlt;
                if (q + 1 < nx) dlt = xs_t[q + 1] - xs_t[q];
                else if (q >= 1) dlt = xs_t[q] - xs_t[q - 1];
                else dlt = 1.0;
                double t = xs_t[q];
                double px = o[0] + t * d[0], py = o[1] + t * d[1], pz = o[2] + t * d[2];
                bg_stencil(H, W, px, py, pz, idx4, w4);
                bg_fetch(bg, H, W, xs_l[q], idx4, w4, out4);
                double sig = out4[0];
                if (sig < 0.0) continue;
                double att = exp(-sig * dlt);
                double Tn = T * att, w = T - Tn;
                if (out4[1] > 0.0) cr += w * out4[1];
                if (out4[2] > 0.0) cg += w * out4[2];
                if (out4[3] > 0.0) cb += w * out4[3];
                s_t[m] = t; s_dlt[m] = dlt; s_sig[m] = sig; s_T[m] = T; s_w[m] = w;
                s_cpre[3 * m] = out4[1]; s_cpre[3 * m + 1] = out4[2]; s_cpre[3 * m + 2] = out4[3];
                s_layer[m] = xs_l[q];
                ++m;
                T = Tn;
                if (T < stop_thresh) break;
            }
        }
        out_rgb[3 * ri] = cr;
        out_rgb[3 * ri + 1] = cg;
        out_rgb[3 * ri + 2] = cb;
        out_trans[ri] = T;
        double upr, upg, upb;
        if (mse_mode) {
            double er = cr - target[3 * ri], eg = cg - target[3 * ri + 1], eb = cb - target[3 * ri + 2];
            mse_sum += er * er + eg * eg + eb * eb;
            upr = up_scale * er; upg = up_scale * eg; upb = up_scale * eb;
        } else {
            upr = target[3 * ri]; upg = target[3 * ri + 1]; upb = target[3 * ri + 2];
        }
        double tc = tfg;
        if (tc < beta_eps) tc = beta_eps;
        if (tc > 1.0 - beta_eps) tc = 1.0 - beta_eps;
        if (lam_beta > 0.0) beta_sum += log(tc) + log(1.0 - tc);
        double bup = 0.0;
        if (lam_beta > 0.0 && beta_eps < tfg && tfg < 1.0 - beta_eps)
            bup = lam_beta * (1.0 / tc - 1.0 / (1.0 - tc));
        if (!with_grad) continue;
        double sfr = 0.0, sfg = 0.0, sfb = 0.0;
        for (int64_t idx = m - 1; idx >= 0; --idx) {
            double sig = s_sig[idx], dlt = s_dlt[idx], Ti = s_T[idx], w = s_w[idx];
            double c0 = s_cpre[3 * idx], c1 = s_cpre[3 * idx + 1], c2 = s_cpre[3 * idx + 2];
            double ccr = c0 > 0.0 ? c0 : 0.0, ccg = c1 > 0.0 ? c1 : 0.0, ccb = c2 > 0.0 ? c2 : 0.0;
            double att = exp(-sig * dlt);
            double gsig = dlt * (upr * (Ti * att * ccr - sfr) + upg * (Ti * att * ccg - sfg) +
                                 upb * (Ti * att * ccb - sfb));
            sfr += w * ccr;
            sfg += w * ccg;
            sfb += w * ccb;
            int64_t lay = s_layer[idx];
            double t = s_t[idx];
            if (lay < 0) {
                if (lam_cauchy > 0.0) {
                    cauchy_sum += log(1.0 + 2.0 * sig * sig);
                    gsig += lam_cauchy * 4.0 * sig / (1.0 + 2.0 * sig * sig);
                }
                if (bup != 0.0) gsig += bup * (-dlt * tfg);
                double gcr = c0 > 0.0 ? upr * w : 0.0;
                double gcg = c1 > 0.0 ? upg * w : 0.0;
                double gcb = c2 > 0.0 ? upb * w : 0.0;
                double gx = clamp_coord(o[0] + t * d[0], lo[0], scale[0], dmax[0]);
                double gy = clamp_coord(o[1] + t * d[1], lo[1], scale[1], dmax[1]);
                double gz = clamp_coord(o[2] + t * d[2], lo[2], scale[2], dmax[2]);
                int n = stencil(gx, gy, gz, links, Dx, Dy, Dz, nearest, rows, ws);
                for (int q = 0; q < n; ++q) {
                    int64_t rw = rows[q];
                    if (rw < 0) continue;
                    double wq = ws[q];
                    touch(rw, tmask, tids, tcnt);
                    double *gr = grad + rw * ROW;
                    gr[0] += wq * gsig;
                    if (gcr != 0.0) for (int b = 0; b < 9; ++b) gr[1 + b] += wq * gcr * basis[b];
                    if (gcg != 0.0) for (int b = 0; b < 9; ++b) gr[10 + b] += wq * gcg * basis[b];
                    if (gcb != 0.0) for (int b = 0; b < 9; ++b) gr[19 + b] += wq * gcb * basis[b];
                }
            } else {
                double px = o[0] + t * d[0], py = o[1] + t * d[1], pz = o[2] + t * d[2];
                bg_stencil(H, W, px, py, pz, idx4, w4);
                for (int q = 0; q < 4; ++q) {
                    int64_t flat = lay * H * W + idx4[q];
                    double wq = w4[q];
                    touch(flat, bg_tmask, bg_tids, bg_tcnt);
                    double *gb = bg_grad + flat * 4;
                    gb[0] += wq * gsig;
                    if (c0 > 0.0) gb[1] += wq * upr * w;
                    if (c1 > 0.0) gb[2] += wq * upg * w;
                    if (c2 > 0.0) gb[3] += wq * upb * w;
                }
            }
        }
    }
    free(s_t); free(s_dlt); free(s_sig); free(s_T); free(s_w); free(s_cpre); free(s_layer);
    free(xs_t); free(xs_l);
    out_sums[0] = mse_sum;
    out_sums[1] = cauchy_sum;
    out_sums[2] = beta_sum;
}

/* K:884-977 (tv_bg): TV over the background axes (layer, theta, phi), phi
 * wrapping; opacity uses zero-valued edge neighbours, colour equal-valued
 * ones; per-axis normalisation D/256.  out_sums = raw {sigma, rgb}. */
void oracle_tv_bg(const double *bg, int64_t L, int64_t H, int64_t W, const int64_t *cells,
                  int64_t ncell, double eps, double f_sigma, double f_rgb, double *grad,
                  uint8_t *tmask, int64_t *tids, int64_t *tcnt, int with_grad,
                  double *out_sums) {
    double fl = (double)L / 256.0, fh = (double)H / 256.0, fw = (double)W / 256.0;
    double e2 = eps * eps, sig_sum = 0.0, rgb_sum = 0.0;
    for (int64_t ci = 0; ci < ncell; ++ci) {
        int64_t cid = cells[ci];
        int64_t l = cid / (H * W), rem = cid % (H * W);
        int64_t j = rem / W, i = rem % W;
        int hl = l + 1 < L, hj = j + 1 < H;
        int64_t iw = i + 1 < W ? i + 1 : 0;
        for (int c = 0; c < 4; ++c) {
            double v0 = bg[((l * H + j) * W + i) * 4 + c];
            double fac = c == 0 ? f_sigma : f_rgb;
            double vl, vj;
            if (c == 0) {
                vl = hl ? bg[(((l + 1) * H + j) * W + i) * 4 + c] : 0.0;
                vj = hj ? bg[((l * H + j + 1) * W + i) * 4 + c] : 0.0;
            } else {
                vl = hl ? bg[(((l + 1) * H + j) * W + i) * 4 + c] : v0;
                vj = hj ? bg[((l * H + j + 1) * W + i) * 4 + c] : v0;
            }
            double vi = bg[((l * H + j) * W + iw) * 4 + c];
            double da = (vl - v0) * fl, db = (vj - v0) * fh, dc = (vi - v0) * fw;
            double val = sqrt(da * da + db * db + dc * dc + e2);
            if (c == 0) sig_sum += val; else rgb_sum += val;
            if (with_grad && val > 0.0) {
                double inv = fac / val, g0 = 0.0;
                if (hl) {
                    int64_t f = (l + 1) * H * W + j * W + i;
                    touch(f, tmask, tids, tcnt);
                    grad[f * 4 + c] += da * fl * inv;
                    g0 -= da * fl * inv;
                } else if (c == 0) {
                    g0 -= da * fl * inv;
                }
                if (hj) {
                    int64_t f = l * H * W + (j + 1) * W + i;
                    touch(f, tmask, tids, tcnt);
                    grad[f * 4 + c] += db * fh * inv;
                    g0 -= db * fh * inv;
                } else if (c == 0) {
                    g0 -= db * fh * inv;
                }
                int64_t f = l * H * W + j * W + iw;
                touch(f, tmask, tids, tcnt);
                grad[f * 4 + c] += dc * fw * inv;
                g0 -= dc * fw * inv;
                if (g0 != 0.0) {
                    int64_t f0 = l * H * W + j * W + i;
                    touch(f0, tmask, tids, tcnt);
                    grad[f0 * 4 + c] += g0;
                }
            }
        }
    }
    out_sums[0] = sig_sum;
    out_sums[1] = rgb_sum;
}

/*
 * camera.py:91-100 generate_rays for a subset of pixels of one view, and the
 * NDC warp camera.py:103-134 (the reference's numpy op order).
 *   cam = {c2w row-major 3x4 (12), focal, width, height}
 *   xs = (i + 0.5 - W/2) / f;   ys = -(j + 0.5 - H/2) / f
 *   d  = d_cam @ R^T with d_cam = (x, y, -1): numpy's matmul runs OpenBLAS
 *        dgemm, whose k-loop accumulates with FMAs from zero
 *        (fma(x2, r2, fma(x1, r1, x0 r0))) -- checked bit-exact against
 *        numpy on this machine by tests/test_oracle_golden.py;
 *   d /= sqrt((d0 d0 + d1 d1) + d2 d2)    (np.linalg.norm, axis=-1)
 */
void oracle_generate_rays(const double *cam, const int64_t *pix, int64_t n, double *o, double *d) {
    const double f = cam[12];
    const int64_t W = (int64_t)cam[13], H = (int64_t)cam[14];
    (void)H;
    for (int64_t r = 0; r < n; ++r) {
        const int64_t p = pix ? pix[r] : r;
        const int64_t i = p % W, j = p / W;
        const double x = (((double)i + 0.5) - (double)W / 2.0) / f;
        const double y = (-(((double)j + 0.5) - cam[14] / 2.0)) / f;
        const double dc[3] = {x, y, -1.0};
        double v[3];
        for (int a = 0; a < 3; ++a) {
            const double *row = cam + 4 * a;   /* R[a, :] */
            v[a] = fma(dc[2], row[2], fma(dc[1], row[1], dc[0] * row[0]));
        }
        const double nrm = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
        for (int a = 0; a < 3; ++a) {
            d[3 * r + a] = v[a] / nrm;
            o[3 * r + a] = cam[4 * a + 3];
        }
    }
}

/* camera.py:103-134: o, d in place -> NDC; valid[r] = |d_z| > 1e-10 */
void oracle_to_ndc(double *o, double *d, int64_t n, double focal, double W, double H,
                   double near, uint8_t *valid) {
    if (near <= 0.0) near = 1.0;
    const double fx = focal / (W / 2.0), fy = focal / (H / 2.0);
    for (int64_t r = 0; r < n; ++r) {
        double *oo = o + 3 * r, *dd = d + 3 * r;
        const int ok = fabs(dd[2]) > 1e-10;
        const double dz = ok ? dd[2] : 1.0;
        const double t = -(near + oo[2]) / dz;
        const double p0 = oo[0] + t * dd[0], p1 = oo[1] + t * dd[1], p2 = oo[2] + t * dd[2];
        const double oz = fabs(p2) > 1e-12 ? p2 : -1e-12;
        const double on0 = -fx * p0 / oz, on1 = -fy * p1 / oz, on2 = 1.0 + 2.0 * near / oz;
        const double dn0 = -fx * (dd[0] / dz - p0 / oz);
        const double dn1 = -fy * (dd[1] / dz - p1 / oz);
        const double dn2 = -2.0 * near / oz;
        oo[0] = on0; oo[1] = on1; oo[2] = on2;
        dd[0] = dn0; dd[1] = dn1; dd[2] = dn2;
        if (valid) valid[r] = (uint8_t)ok;
    }
}
