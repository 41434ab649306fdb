// plx_grid_ops.cu -- per-row / per-cell kernels for sm_100a: TV regulariser,
// sparse RMSProp/SGD with fused gradient clear, touched-row count, prune,
// upsample, id compaction scan and the empty-space cell bitmask.
//
// Reference: pkg/src/plenoxel/_kernels.py tv_grid (K:456-569), opt_step
// (K:572-590), clear_grad (K:593-600); grid.py prune (G:228-258), upsample
// (G:260-285).  All of these are HBM-streaming kernels: coalesced float4
// row access, one pass, grids sized in multiples of the 148 SMs.
#include <stdlib.h>

#include <cub/block/block_reduce.cuh>

#include "plx_optim.cuh"

namespace plx {

// ---------------------------------------------------------------- TV ------
struct TvArgs {
    const int64_t *cells;
    const int64_t *start_dev;   // optional device copy of start (CUDA-graph replay)
    int64_t start, count, ncell;
    double fac[3], eps, f_sigma, f_sh;
    int wrap[3];
    int with_grad;
    float *grad;
    uint8_t *tmask;
    double *sums;
};

// sqrt(s) and 1/sqrt(s) for s > 0 in float64 to ~1 ulp, without the IEEE
// sqrt and division subroutines (MUFU seed + Newton steps with explicit FMAs;
// -fmad=false does not touch fma()).
__device__ __forceinline__ void root_and_rinv(double s, double &root, double &rinv) {
    if (s < 2.2250738585072014e-308) {   // subnormal (eps = 0 only): IEEE path
        root = sqrt(s);
        rinv = 1.0 / root;
        return;
    }
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
    const double hs = 0.5 * s;
    // two Newton steps take the hardware estimate to ~2^-44 -- ample for
    // rinv, which only feeds f32-rounded gradients; the root gets a final
    // Newton step of its own (~2^-88 before rounding: the sums stay f64-exact)
    y = y * fma(-hs * y, y, 1.5);
    y = y * fma(-hs * y, y, 1.5);
    double r = s * y;
    r = fma(0.5 * y, fma(-r, r, s), r);
    root = r;
    rinv = y;
}

// TV on identity-linked dense grids (every cell has an SH term): 4 cells per
// warp iteration, lane = (cell, column
// quad): the 7 lanes of a cell own its 7 float4 column groups, so the 4 rows
// (self, +x, +y, +z) of a cell are read and reduced as 7 parallel float4s
// instead of a 7-step loop per thread.  Per column the arithmetic is the
// reference's (float64, one sqrt per coefficient, K:534-568); the sigma term
// (K:505-532) is column 0, owned by quad 0.
template <int NT>
__global__ void __launch_bounds__(NT) tv_dense_kernel(DGrid G, TvArgs a) {
    const int lane = threadIdx.x & 31;
    const int sub = lane / 7, quad = lane % 7;
    const int64_t nw = (int64_t)gridDim.x * (NT / 32);
    const double e2 = a.eps * a.eps;
    const float *T = G.table;
    double sig_sum = 0.0, sh_sum = 0.0;
    for (int64_t w = (int64_t)blockIdx.x * (NT / 32) + (threadIdx.x >> 5); w * 4 < a.count;
         w += nw) {
        const int64_t ci = w * 4 + sub;
        const bool valid = lane < 28 && ci < a.count;
        int32_t r0 = -1, rx = -1, ry = -1, rz = -1;
        bool tx = false, ty = false, tz = false, t0 = false;
        float gx[4] = {0.f, 0.f, 0.f, 0.f}, gy[4] = {0.f, 0.f, 0.f, 0.f};
        float gz[4] = {0.f, 0.f, 0.f, 0.f}, g0v[4] = {0.f, 0.f, 0.f, 0.f};
        if (valid) {
            int64_t cid;   // L:41-47 (lattice < 2^31 cells: 32-bit index math)
            if (a.cells) {
                cid = a.cells[ci];
            } else {
                cid = (a.start_dev ? *a.start_dev : a.start) + ci;
                if (cid >= a.ncell) cid %= a.ncell;   // wrapped run (rare branch)
            }
            const uint32_t c32 = (uint32_t)cid, dz = (uint32_t)G.Dz;
            const uint32_t ij = c32 / dz, k = c32 - ij * dz;
            const uint32_t i = ij / (uint32_t)G.Dy, j = ij - i * (uint32_t)G.Dy;
            int64_t ii = i + 1, jj = j + 1, kk = k + 1;
            bool hx = true, hy = true, hz = true;
            if (ii >= G.Dx) { if (a.wrap[0]) ii = 0; else hx = false; }
            if (jj >= G.Dy) { if (a.wrap[1]) jj = 0; else hy = false; }
            if (kk >= G.Dz) { if (a.wrap[2]) kk = 0; else hz = false; }
            if (G.identity) {   // dense identity-linked grid: no link gathers
                r0 = (int32_t)cid;
                rx = hx ? (int32_t)flat(G, ii, j, k) : -1;
                ry = hy ? (int32_t)flat(G, i, jj, k) : -1;
                rz = hz ? (int32_t)flat(G, i, j, kk) : -1;
            } else {
                r0 = __ldg(G.links + cid);
                rx = hx ? __ldg(G.links + flat(G, ii, j, k)) : -1;
                ry = hy ? __ldg(G.links + flat(G, i, jj, k)) : -1;
                rz = hz ? __ldg(G.links + flat(G, i, j, kk)) : -1;
            }
            const bool okx = rx >= 0, oky = ry >= 0, okz = rz >= 0;
            const bool sh_on = r0 >= 0 && (okx || oky || okz);
            float4 v0 = make_float4(0, 0, 0, 0), vx = v0, vy = v0, vz = v0;
            if (sh_on) {
                v0 = __ldg(reinterpret_cast<const float4 *>(T + (int64_t)r0 * PLX_STRIDE) + quad);
                if (okx) vx = __ldg(reinterpret_cast<const float4 *>(T + (int64_t)rx * PLX_STRIDE) + quad);
                if (oky) vy = __ldg(reinterpret_cast<const float4 *>(T + (int64_t)ry * PLX_STRIDE) + quad);
                if (okz) vz = __ldg(reinterpret_cast<const float4 *>(T + (int64_t)rz * PLX_STRIDE) + quad);
            }
            if (quad == 0) {
                // opacity term (K:505-532): missing neighbours read as 0
                const double s0 = r0 >= 0 ? (double)__ldg(G.density + r0) : 0.0;
                const double sx = rx >= 0 ? (double)__ldg(G.density + rx) : 0.0;
                const double sy = ry >= 0 ? (double)__ldg(G.density + ry) : 0.0;
                const double sz = rz >= 0 ? (double)__ldg(G.density + rz) : 0.0;
                const double dxv = (sx - s0) * a.fac[0], dyv = (sy - s0) * a.fac[1],
                             dzv = (sz - s0) * a.fac[2];
                const double s2v = dxv * dxv + dyv * dyv + dzv * dzv + e2;
                double val = 0.0, rinv = 0.0;
                if (s2v > 0.0) root_and_rinv(s2v, val, rinv);
                sig_sum += val;
                if (a.with_grad && val > 0.0) {
                    const double inv = a.f_sigma * rinv;
                    double g0 = 0.0;
                    if (rx >= 0) { tx = true; gx[0] = (float)(dxv * a.fac[0] * inv); }
                    g0 -= dxv * a.fac[0] * inv;
                    if (ry >= 0) { ty = true; gy[0] = (float)(dyv * a.fac[1] * inv); }
                    g0 -= dyv * a.fac[1] * inv;
                    if (rz >= 0) { tz = true; gz[0] = (float)(dzv * a.fac[2] * inv); }
                    g0 -= dzv * a.fac[2] * inv;
                    if (r0 >= 0 && g0 != 0.0) { t0 = true; g0v[0] = (float)g0; }
                }
                if (!sh_on) sh_sum += 27.0 * a.eps;   // empty self / no neighbour
            }
            if (sh_on) {   // K:534-568, columns 4*quad .. 4*quad+3 (column 0 is sigma)
                const float c0[4] = {v0.x, v0.y, v0.z, v0.w}, cx[4] = {vx.x, vx.y, vx.z, vx.w};
                const float cy[4] = {vy.x, vy.y, vy.z, vy.w}, cz[4] = {vz.x, vz.y, vz.z, vz.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (quad == 0 && e == 0) continue;
                    const double v0d = (double)c0[e];
                    const double ax = okx ? ((double)cx[e] - v0d) * a.fac[0] : 0.0;
                    const double ay = oky ? ((double)cy[e] - v0d) * a.fac[1] : 0.0;
                    const double az = okz ? ((double)cz[e] - v0d) * a.fac[2] : 0.0;
                    const double s2v = ax * ax + ay * ay + az * az + e2;
                    double v = 0.0, rinv = 0.0;
                    if (s2v > 0.0) root_and_rinv(s2v, v, rinv);
                    sh_sum += v;
                    if (a.with_grad && v > 0.0) {
                        const double inv = a.f_sh * rinv;
                        double g0 = 0.0;
                        if (okx) { tx = true; gx[e] = (float)(ax * a.fac[0] * inv); g0 -= ax * a.fac[0] * inv; }
                        if (oky) { ty = true; gy[e] = (float)(ay * a.fac[1] * inv); g0 -= ay * a.fac[1] * inv; }
                        if (okz) { tz = true; gz[e] = (float)(az * a.fac[2] * inv); g0 -= az * a.fac[2] * inv; }
                        if (g0 != 0.0) { t0 = true; g0v[e] = (float)g0; }
                    }
                }
            }
            if (a.with_grad) {
                if (rx >= 0 && (gx[0] != 0.f || gx[1] != 0.f || gx[2] != 0.f || gx[3] != 0.f))
                    red_add_v4(a.grad + (int64_t)rx * PLX_STRIDE + 4 * quad, gx[0], gx[1], gx[2], gx[3]);
                if (ry >= 0 && (gy[0] != 0.f || gy[1] != 0.f || gy[2] != 0.f || gy[3] != 0.f))
                    red_add_v4(a.grad + (int64_t)ry * PLX_STRIDE + 4 * quad, gy[0], gy[1], gy[2], gy[3]);
                if (rz >= 0 && (gz[0] != 0.f || gz[1] != 0.f || gz[2] != 0.f || gz[3] != 0.f))
                    red_add_v4(a.grad + (int64_t)rz * PLX_STRIDE + 4 * quad, gz[0], gz[1], gz[2], gz[3]);
                if (r0 >= 0 && (g0v[0] != 0.f || g0v[1] != 0.f || g0v[2] != 0.f || g0v[3] != 0.f))
                    red_add_v4(a.grad + (int64_t)r0 * PLX_STRIDE + 4 * quad, g0v[0], g0v[1], g0v[2], g0v[3]);
            }
        }
        if (a.with_grad) {   // _touch (K:155-160): a row is touched if any column got a value
            const unsigned cell_lanes = 0x7fu << (7 * (sub & 3));
            const bool bx = __ballot_sync(PLX_FULL_MASK, tx) & cell_lanes;
            const bool by = __ballot_sync(PLX_FULL_MASK, ty) & cell_lanes;
            const bool bz = __ballot_sync(PLX_FULL_MASK, tz) & cell_lanes;
            const bool b0 = __ballot_sync(PLX_FULL_MASK, t0) & cell_lanes;
            if (valid && quad == 0) {
                if (bx) a.tmask[rx] = 1;
                if (by) a.tmask[ry] = 1;
                if (bz) a.tmask[rz] = 1;
                if (b0) a.tmask[r0] = 1;
            }
        }
    }
    // both sums in one pass: warp shuffles, one shared-memory exchange, one
    // barrier (short blocks run one iteration, so this reduction is a large
    // share of a block's work)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        sig_sum += __shfl_down_sync(PLX_FULL_MASK, sig_sum, off);
        sh_sum += __shfl_down_sync(PLX_FULL_MASK, sh_sum, off);
    }
    __shared__ double part[2][NT / 32];
    const int wid = threadIdx.x >> 5;
    if (lane == 0) {
        part[0][wid] = sig_sum;
        part[1][wid] = sh_sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int k = 0; k < NT / 32; ++k) {
            s1 += part[0][k];
            s2 += part[1][k];
        }
        atomicAdd(a.sums + 0, s1);
        atomicAdd(a.sums + 1, s2);
    }
}

// TV on sparse grids, in two phases per warp iteration of 32 cells.
//   phase 1, lane = cell: the cell's 4 links (self, +x, +y, +z; none on an
//     identity-linked grid), the sigma term (K:505-532; missing rows read as
//     0) and its gradients.  A cell whose SH term is empty -- no self row or
//     no neighbour row, K:534-568 then contributes 27 eps -- is finished here
//     (scalar reductions into column 0).
//   phase 2, the cells with an SH term, 4 at a time, lane = (cell, column
//     quad): the 7 lanes of a cell own its 7 float4 column groups, so the 4
//     rows of a cell are read and reduced as 7 parallel float4s; quad 0
//     carries the cell's sigma gradients (column 0) from phase 1 into its
//     reductions.
// On sparse grids most cells of the run are empty (C3 at 512^3: ~86 %), so
// they no longer occupy a 7-lane cell slot.  Per column the arithmetic is
// the reference's (float64, one sqrt per coefficient).
struct TvCell {
    int32_t r0, rx, ry, rz;
    float g0, gx, gy, gz;   // sigma gradients (column 0)
    unsigned flags;         // bit 0..3: sigma touched self / x / y / z
};

template <int NT>
__global__ void __launch_bounds__(NT) tv_sparse_kernel(DGrid G, TvArgs a) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int sub = lane / 7, quad = lane % 7;
    __shared__ TvCell cells[NT];           // phase-1 results, by thread
    __shared__ uint16_t shl[NT];           // the block's SH cells, compacted
    __shared__ int wcnt[NT / 32];
    const double e2 = a.eps * a.eps;
    const float *T = G.table;
    double sig_sum = 0.0, sh_sum = 0.0;
    // block-wide iterations of NT cells (a cell per thread in phase 1); the
    // SH cells of all NT are then shared out to the warps 4 at a time, so a
    // warp whose 32 cells are empty does not leave the block waiting on one
    // whose cells all carry SH terms
    for (int64_t t0 = (int64_t)blockIdx.x * NT; t0 < a.count; t0 += (int64_t)gridDim.x * NT) {
        // ---- phase 1: one cell per thread ----
        const int64_t ci = t0 + threadIdx.x;
        const bool valid = ci < a.count;
        int32_t r0 = -1, rx = -1, ry = -1, rz = -1;
        bool sh_on = false;
        if (valid) {
            int64_t cid;   // L:41-47 (lattice < 2^31 cells: 32-bit index math)
            if (a.cells) {
                cid = a.cells[ci];
            } else {
                cid = (a.start_dev ? *a.start_dev : a.start) + ci;
                if (cid >= a.ncell) cid %= a.ncell;   // wrapped run (rare branch)
            }
            const uint32_t c32 = (uint32_t)cid, dz = (uint32_t)G.Dz;
            const uint32_t ij = c32 / dz, k = c32 - ij * dz;
            const uint32_t i = ij / (uint32_t)G.Dy, j = ij - i * (uint32_t)G.Dy;
            int64_t ii = i + 1, jj = j + 1, kk = k + 1;
            bool hx = true, hy = true, hz = true;
            if (ii >= G.Dx) { if (a.wrap[0]) ii = 0; else hx = false; }
            if (jj >= G.Dy) { if (a.wrap[1]) jj = 0; else hy = false; }
            if (kk >= G.Dz) { if (a.wrap[2]) kk = 0; else hz = false; }
            if (G.identity) {   // dense identity-linked grid: no link gathers
                r0 = (int32_t)cid;
                rx = hx ? (int32_t)flat(G, ii, j, k) : -1;
                ry = hy ? (int32_t)flat(G, i, jj, k) : -1;
                rz = hz ? (int32_t)flat(G, i, j, kk) : -1;
            } else {
                r0 = __ldg(G.links + cid);
                rx = hx ? __ldg(G.links + flat(G, ii, j, k)) : -1;
                ry = hy ? __ldg(G.links + flat(G, i, jj, k)) : -1;
                rz = hz ? __ldg(G.links + flat(G, i, j, kk)) : -1;
            }
            sh_on = r0 >= 0 && (rx >= 0 || ry >= 0 || rz >= 0);
            // opacity term (K:505-532): missing neighbours read as 0
            const double s0 = r0 >= 0 ? (double)__ldg(G.density + r0) : 0.0;
            const double sx = rx >= 0 ? (double)__ldg(G.density + rx) : 0.0;
            const double sy = ry >= 0 ? (double)__ldg(G.density + ry) : 0.0;
            const double sz = rz >= 0 ? (double)__ldg(G.density + rz) : 0.0;
            const double dxv = (sx - s0) * a.fac[0], dyv = (sy - s0) * a.fac[1],
                         dzv = (sz - s0) * a.fac[2];
            const double s2v = dxv * dxv + dyv * dyv + dzv * dzv + e2;
            double val = 0.0, rinv = 0.0;
            if (s2v > 0.0) root_and_rinv(s2v, val, rinv);
            sig_sum += val;
            if (!sh_on) sh_sum += 27.0 * a.eps;   // empty self / no neighbour
            TvCell tc{r0, rx, ry, rz, 0.f, 0.f, 0.f, 0.f, 0u};
            if (a.with_grad && val > 0.0) {
                const double inv = a.f_sigma * rinv;
                double g0 = 0.0;
                if (rx >= 0) { tc.flags |= 2u; tc.gx = (float)(dxv * a.fac[0] * inv); }
                g0 -= dxv * a.fac[0] * inv;
                if (ry >= 0) { tc.flags |= 4u; tc.gy = (float)(dyv * a.fac[1] * inv); }
                g0 -= dyv * a.fac[1] * inv;
                if (rz >= 0) { tc.flags |= 8u; tc.gz = (float)(dzv * a.fac[2] * inv); }
                g0 -= dzv * a.fac[2] * inv;
                if (r0 >= 0 && g0 != 0.0) { tc.flags |= 1u; tc.g0 = (float)g0; }
            }
            if (sh_on) {
                cells[threadIdx.x] = tc;
            } else if (a.with_grad) {   // sigma-only cell: finished here
                if (tc.gx != 0.f) atomicAdd(a.grad + (int64_t)rx * PLX_STRIDE, tc.gx);
                if (tc.gy != 0.f) atomicAdd(a.grad + (int64_t)ry * PLX_STRIDE, tc.gy);
                if (tc.gz != 0.f) atomicAdd(a.grad + (int64_t)rz * PLX_STRIDE, tc.gz);
                if (tc.g0 != 0.f) atomicAdd(a.grad + (int64_t)r0 * PLX_STRIDE, tc.g0);
                if (tc.flags & 2u) a.tmask[rx] = 1;
                if (tc.flags & 4u) a.tmask[ry] = 1;
                if (tc.flags & 8u) a.tmask[rz] = 1;
                if (tc.flags & 1u) a.tmask[r0] = 1;
            }
        }
        // the block's cells with an SH term, compacted in thread order
        const unsigned shm = __ballot_sync(PLX_FULL_MASK, sh_on);
        if (lane == 0) wcnt[wib] = __popc(shm);
        __syncthreads();
        int before = 0, nsh = 0;
#pragma unroll
        for (int k = 0; k < NT / 32; ++k) {
            before += k < wib ? wcnt[k] : 0;
            nsh += wcnt[k];
        }
        if (sh_on) shl[before + __popc(shm & ((1u << lane) - 1u))] = (uint16_t)threadIdx.x;
        __syncthreads();
        // ---- phase 2: 4 SH cells per warp round, 7 lanes per cell ----
        for (int g = wib * 4; g < nsh; g += 4 * (NT / 32)) {
            const int idx = g + sub;
            const bool ok = lane < 28 && idx < nsh;
            TvCell tc{-1, -1, -1, -1, 0.f, 0.f, 0.f, 0.f, 0u};
            if (ok) tc = cells[shl[idx]];
            bool tx = false, ty = false, tz = false, t0 = false;
            float gx[4] = {0.f, 0.f, 0.f, 0.f}, gy[4] = {0.f, 0.f, 0.f, 0.f};
            float gz[4] = {0.f, 0.f, 0.f, 0.f}, g0v[4] = {0.f, 0.f, 0.f, 0.f};
            if (ok) {
                const bool okx = tc.rx >= 0, oky = tc.ry >= 0, okz = tc.rz >= 0;
                const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
                const float4 v0 = __ldg(reinterpret_cast<const float4 *>(T + (int64_t)tc.r0 * PLX_STRIDE) + quad);
                const float4 vx = okx ? __ldg(reinterpret_cast<const float4 *>(T + (int64_t)tc.rx * PLX_STRIDE) + quad) : z4;
                const float4 vy = oky ? __ldg(reinterpret_cast<const float4 *>(T + (int64_t)tc.ry * PLX_STRIDE) + quad) : z4;
                const float4 vz = okz ? __ldg(reinterpret_cast<const float4 *>(T + (int64_t)tc.rz * PLX_STRIDE) + quad) : z4;
                if (quad == 0) {   // column 0: the sigma gradients of phase 1
                    gx[0] = tc.gx;
                    gy[0] = tc.gy;
                    gz[0] = tc.gz;
                    g0v[0] = tc.g0;
                    tx = tc.flags & 2u;
                    ty = tc.flags & 4u;
                    tz = tc.flags & 8u;
                    t0 = tc.flags & 1u;
                }
                // K:534-568, columns 4*quad .. 4*quad+3 (column 0 is sigma)
                const float c0[4] = {v0.x, v0.y, v0.z, v0.w}, cx[4] = {vx.x, vx.y, vx.z, vx.w};
                const float cy[4] = {vy.x, vy.y, vy.z, vy.w}, cz[4] = {vz.x, vz.y, vz.z, vz.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (quad == 0 && e == 0) continue;
                    const double v0d = (double)c0[e];
                    const double ax = okx ? ((double)cx[e] - v0d) * a.fac[0] : 0.0;
                    const double ay = oky ? ((double)cy[e] - v0d) * a.fac[1] : 0.0;
                    const double az = okz ? ((double)cz[e] - v0d) * a.fac[2] : 0.0;
                    const double s2v = ax * ax + ay * ay + az * az + e2;
                    double v = 0.0, rinv = 0.0;
                    if (s2v > 0.0) root_and_rinv(s2v, v, rinv);
                    sh_sum += v;
                    if (a.with_grad && v > 0.0) {
                        const double inv = a.f_sh * rinv;
                        double g0 = 0.0;
                        if (okx) { tx = true; gx[e] = (float)(ax * a.fac[0] * inv); g0 -= ax * a.fac[0] * inv; }
                        if (oky) { ty = true; gy[e] = (float)(ay * a.fac[1] * inv); g0 -= ay * a.fac[1] * inv; }
                        if (okz) { tz = true; gz[e] = (float)(az * a.fac[2] * inv); g0 -= az * a.fac[2] * inv; }
                        if (g0 != 0.0) { t0 = true; g0v[e] = (float)g0; }
                    }
                }
                if (a.with_grad) {
                    if (okx && (gx[0] != 0.f || gx[1] != 0.f || gx[2] != 0.f || gx[3] != 0.f))
                        red_add_v4(a.grad + (int64_t)tc.rx * PLX_STRIDE + 4 * quad, gx[0], gx[1], gx[2], gx[3]);
                    if (oky && (gy[0] != 0.f || gy[1] != 0.f || gy[2] != 0.f || gy[3] != 0.f))
                        red_add_v4(a.grad + (int64_t)tc.ry * PLX_STRIDE + 4 * quad, gy[0], gy[1], gy[2], gy[3]);
                    if (okz && (gz[0] != 0.f || gz[1] != 0.f || gz[2] != 0.f || gz[3] != 0.f))
                        red_add_v4(a.grad + (int64_t)tc.rz * PLX_STRIDE + 4 * quad, gz[0], gz[1], gz[2], gz[3]);
                    if (g0v[0] != 0.f || g0v[1] != 0.f || g0v[2] != 0.f || g0v[3] != 0.f)
                        red_add_v4(a.grad + (int64_t)tc.r0 * PLX_STRIDE + 4 * quad, g0v[0], g0v[1], g0v[2], g0v[3]);
                }
            }
            if (a.with_grad) {   // _touch (K:155-160): a row is touched if any column got a value
                const unsigned cell_lanes = 0x7fu << (7 * (sub & 3));
                const bool bx = __ballot_sync(PLX_FULL_MASK, tx) & cell_lanes;
                const bool by = __ballot_sync(PLX_FULL_MASK, ty) & cell_lanes;
                const bool bz = __ballot_sync(PLX_FULL_MASK, tz) & cell_lanes;
                const bool b0 = __ballot_sync(PLX_FULL_MASK, t0) & cell_lanes;
                if (ok && quad == 0) {
                    if (bx) a.tmask[tc.rx] = 1;
                    if (by) a.tmask[tc.ry] = 1;
                    if (bz) a.tmask[tc.rz] = 1;
                    if (b0) a.tmask[tc.r0] = 1;
                }
            }
        }
        __syncthreads();   // cells / shl reused by the next iteration
    }
    // both sums in one pass: warp shuffles, one shared-memory exchange, one
    // barrier
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        sig_sum += __shfl_down_sync(PLX_FULL_MASK, sig_sum, off);
        sh_sum += __shfl_down_sync(PLX_FULL_MASK, sh_sum, off);
    }
    __shared__ double part[2][NT / 32];
    if (lane == 0) {
        part[0][wib] = sig_sum;
        part[1][wib] = sh_sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int k = 0; k < NT / 32; ++k) {
            s1 += part[0][k];
            s2 += part[1][k];
        }
        atomicAdd(a.sums + 0, s1);
        atomicAdd(a.sums + 1, s2);
    }
}

// ------------------------------------------------------- optimiser --------
// Persistent sweep over the touched mask (K:572-600).  A warp owns 128-row
// segments: one coalesced 128-byte load of the mask, a warp prefix sum turns
// the set bytes into a compact per-warp list in shared memory, and the
// touched rows are then updated 4 at a time (lanes 0..27 = 4 rows x 7 float4,
// fully coalesced 448-byte runs of table / grad / v).  Untouched rows cost
// one mask byte; touched rows cost exactly their compulsory 672 B.
struct OptArgs {
    float *table, *density, *v, *grad;
    const double *lr_dev;      // optional device {lr_sigma, lr_sh} (CUDA-graph replay)
    double *guard;             // optional divergence guard (see guard_halts)
    float *sigma_lat;          // optional lattice sigma mirror: kept current
    const int32_t *row_cell;   // row -> lattice point (required with sigma_lat)
    uint8_t *tmask;
    int64_t rows;
    double lr_sigma, lr_sh, beta, eps;
    int rmsprop, clear, update;
    unsigned long long *count;
    uint32_t *brick_dead;      // optional dead-brick mask (with sigma_lat): kept conservative
    int32_t Dx, Dy, Dz;
};

__device__ __forceinline__ int nonzero_bytes(uint32_t m) {
    m = (m | (m >> 4)) & 0x0f0f0f0fu;
    m = (m | (m >> 2)) & 0x03030303u;
    m = (m | (m >> 1)) & 0x01010101u;
    return __popc(m);
}

// sigma of a row at lattice point c changed: keep the lattice mirror current.
__device__ __forceinline__ void lat_update(const OptArgs &a, int32_t c, float sigma) {
    if (a.sigma_lat) a.sigma_lat[c] = sigma;
    if (a.brick_dead && sigma >= 0.f) brick_revive(a.brick_dead, c, a.Dx, a.Dy, a.Dz);
}

// The update of one float4 of one row (K:578-590), float64 arithmetic.
__device__ __forceinline__ void opt_apply(const OptArgs &a, int quad, float4 &g4, float4 &t4,
                                          float4 &v4) {
    const double ls = a.lr_dev ? a.lr_dev[0] : a.lr_sigma, lc = a.lr_dev ? a.lr_dev[1] : a.lr_sh;
    opt_apply4(OptHyper{ls, lc, a.beta, a.eps, a.rmsprop}, quad, g4, t4, v4);
}

template <int NT>
__global__ void __launch_bounds__(NT) opt_kernel(OptArgs a) {
    if (guard_halts(a.guard)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) a.guard[4] = 1.0;
        return;
    }
    __shared__ uint8_t list[NT / 32][128];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t nseg = (a.rows + 127) >> 7;
    const int64_t nw = (int64_t)gridDim.x * (NT / 32);
    unsigned long long cnt = 0;
    const int quad = lane % 7, sub = lane / 7;
    auto load_mask = [&](int64_t seg) -> uint32_t {
        const int64_t r0 = seg * 128 + lane * 4;
        uint32_t m = 0;
        if (seg >= nseg) return 0u;
        if (r0 + 3 < a.rows) {
            m = *reinterpret_cast<const volatile uint32_t *>(a.tmask + r0);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (r0 + e < a.rows && a.tmask[r0 + e]) m |= 0xffu << (8 * e);
        }
        return m;
    };
    int64_t seg = (int64_t)blockIdx.x * (NT / 32) + wib;
    uint32_t m_next = load_mask(seg);
    for (; seg < nseg; seg += nw) {
        const int64_t r0 = seg * 128 + lane * 4;
        const uint32_t m = m_next;
        m_next = load_mask(seg + nw);   // prefetch the next segment's mask
        const int c = nonzero_bytes(m);
        int incl = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(PLX_FULL_MASK, incl, off);
            if (lane >= off) incl += y;
        }
        const int total = __shfl_sync(PLX_FULL_MASK, incl, 31);
        if (total == 0) continue;
        int pos = incl - c;
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if ((m >> (8 * e)) & 0xffu) list[wib][pos++] = (uint8_t)(lane * 4 + e);
        __syncwarp();
        cnt += (unsigned long long)total;
        constexpr int U = 2;   // 2 groups x 4 rows: 6 float4 loads in flight per lane
        for (int gidx = 0; gidx < total; gidx += 4 * U) {
            float4 g4[U], t4[U], v4[U];
            float den[U];
            int64_t rw[U];
            bool act[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = gidx + 4 * u + sub;
                act[u] = lane < 28 && j < total;
                rw[u] = act[u] ? seg * 128 + list[wib][j] : 0;
                if (act[u]) {
                    g4[u] = reinterpret_cast<const float4 *>(a.grad + rw[u] * PLX_STRIDE)[quad];
                    if (a.update) {
                        t4[u] = reinterpret_cast<const float4 *>(a.table + rw[u] * PLX_STRIDE)[quad];
                        if (quad == 0) den[u] = a.density[rw[u]];
                        if (a.rmsprop)
                            v4[u] = reinterpret_cast<const float4 *>(a.v + rw[u] * PLX_STRIDE)[quad];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!act[u]) continue;
                if (a.update) {
                    if (quad == 0) t4[u].x = den[u];
                    opt_apply(a, quad, g4[u], t4[u], v4[u]);
                    if (quad == 0) {
                        a.density[rw[u]] = t4[u].x;
                        if (a.sigma_lat) lat_update(a, a.row_cell[rw[u]], t4[u].x);
                        t4[u].x = 0.f;
                    }
                    reinterpret_cast<float4 *>(a.table + rw[u] * PLX_STRIDE)[quad] = t4[u];
                    if (a.rmsprop) reinterpret_cast<float4 *>(a.v + rw[u] * PLX_STRIDE)[quad] = v4[u];
                }
                if (a.clear)
                    reinterpret_cast<float4 *>(a.grad + rw[u] * PLX_STRIDE)[quad] =
                        make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        if (a.clear && m) {
            if (r0 + 3 < a.rows) {
                *reinterpret_cast<uint32_t *>(a.tmask + r0) = 0u;
            } else {
                for (int e = 0; e < 4; ++e)
                    if (r0 + e < a.rows) a.tmask[r0 + e] = 0;
            }
        }
        __syncwarp();
    }
    if (a.count && lane == 0 && cnt) atomicAdd(a.count, cnt);
}

// Two-phase variant used when the caller provides the touched-id list of
// GradientBuffer (G:25-68 touched_ids / _count, plx_grad.tids / tcnt):
//   phase 1 (touched_compact_kernel): the mask -> a compact list of touched
//            row ids (one atomic per 8192-row tile; ids sorted within a tile,
//            tiles in atomic order -- every row is updated independently)
//            and the mask clear;
//   phase 2 (opt_rows_kernel): grid-stride over the list, 4 rows x 7 float4
//            per warp group, kOptU groups in flight per lane, so every lane
//            keeps 3*kOptU independent 16-byte loads outstanding -- the sweep
//            above serialises mask scan -> loads -> update per segment.
// One block per tile of kTileRows mask bytes: every thread reads 32 bytes
// (two uint4), the block scans the per-thread counts, takes its slice of the
// list with ONE atomic, stages the ids in shared memory in row order and
// writes them out coalesced.  The mask is HBM-streamed once; the kernel
// costs ~4 instructions per mask word plus ~4 per touched row.
constexpr int kCompactNT = 256;
constexpr int kTileRows = kCompactNT * 32;

// bit 8e+7 of the result set <=> byte e of x nonzero
__device__ __forceinline__ uint32_t nonzero_bytes_hi(uint32_t x) {
    return (((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x) & 0x80808080u;
}

__device__ __forceinline__ void load_mask_words(const uint8_t *tmask, int64_t rows, int64_t r0,
                                                uint32_t *w) {
    if (r0 + 32 <= rows) {
        const uint4 *p = reinterpret_cast<const uint4 *>(tmask + r0);
        const uint4 a0 = __ldcs(p), a1 = __ldcs(p + 1);
        w[0] = a0.x; w[1] = a0.y; w[2] = a0.z; w[3] = a0.w;
        w[4] = a1.x; w[5] = a1.y; w[6] = a1.z; w[7] = a1.w;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            w[i] = 0u;
            for (int e = 0; e < 4; ++e) {
                const int64_t r = r0 + 4 * i + e;
                if (r < rows && tmask[r]) w[i] |= 0xffu << (8 * e);
            }
        }
    }
}

// Persistent over the tiles (one resident wave), the next tile's mask words
// loaded while the current one is compacted.
__global__ void __launch_bounds__(kCompactNT, 4) touched_compact_kernel(uint8_t *tmask,
                                                                        int64_t rows,
                                                                        int32_t *tids,
                                                                        int64_t *tcnt, int clear,
                                                                        double *guard,
                                                                        double *host_sums) {
    __shared__ uint16_t sid[kTileRows];   // row offsets within the tile
    __shared__ int warp_tot[kCompactNT / 32];
    __shared__ unsigned long long blk_base;
    // the step's loss sums are final here (render + TV done): hand them to
    // the host's pinned slot directly (no memcpy node in the step graph)
    if (host_sums && blockIdx.x == 0 && threadIdx.x < 4) host_sums[threadIdx.x] = guard[threadIdx.x];
    if (guard_halts(guard)) {   // non-finite loss: no update, no clear (T:473-480)
        if (blockIdx.x == 0 && threadIdx.x == 0) guard[4] = 1.0;
        return;
    }
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t ntiles = (rows + kTileRows - 1) / kTileRows;
    uint32_t w[8], wn[8];
    int64_t t = blockIdx.x;
    if (t < ntiles) load_mask_words(tmask, rows, t * kTileRows + (int64_t)threadIdx.x * 32, w);
    for (; t < ntiles; t += gridDim.x) {
        const int64_t r0 = t * kTileRows + (int64_t)threadIdx.x * 32;
        const int64_t tn = t + gridDim.x;
        if (tn < ntiles) load_mask_words(tmask, rows, tn * kTileRows + (int64_t)threadIdx.x * 32, wn);
        int c = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            w[i] = nonzero_bytes_hi(w[i]);
            c += __popc(w[i]);
        }
        int incl = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(PLX_FULL_MASK, incl, off);
            if (lane >= off) incl += y;
        }
        if (lane == 31) warp_tot[wib] = incl;
        __syncthreads();
        int before = 0, total = 0;
#pragma unroll
        for (int k = 0; k < kCompactNT / 32; ++k) {
            const int tt = warp_tot[k];
            before += k < wib ? tt : 0;
            total += tt;
        }
        if (total != 0) {   // block-uniform
            if (threadIdx.x == 0)
                blk_base = atomicAdd(reinterpret_cast<unsigned long long *>(tcnt),
                                     (unsigned long long)total);
            int q = before + incl - c;
            const int rb = threadIdx.x * 32;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t x = w[i];
                if (!x) continue;
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (x & (0x80u << (8 * e))) sid[q++] = (uint16_t)(rb + 4 * i + e);
            }
            if (clear && c) {
                if (r0 + 32 <= rows) {
                    uint4 *p = reinterpret_cast<uint4 *>(tmask + r0);
                    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
                    p[0] = z;
                    p[1] = z;
                } else {
                    for (int r = 0; r < 32 && r0 + r < rows; ++r) tmask[r0 + r] = 0;
                }
            }
            __syncthreads();
            const int64_t base = (int64_t)blk_base;
            const int32_t tile0 = (int32_t)(t * kTileRows);
            for (int i = threadIdx.x; i < total; i += kCompactNT) tids[base + i] = tile0 + sid[i];
        }
        __syncthreads();   // smem reuse by the next tile
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = wn[i];
    }
}

static int compact_grid(int64_t rows) {
    static int bps = 0;
    if (!bps) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, touched_compact_kernel, kCompactNT, 0);
        if (bps <= 0) bps = 1;
    }
    const int64_t ntiles = (rows + kTileRows - 1) / kTileRows;
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t cap = (int64_t)(sms > 0 ? sms : 148) * bps;
    return (int)(ntiles < cap ? (ntiles > 0 ? ntiles : 1) : cap);
}

template <int UU, int MINB>
__global__ void __launch_bounds__(256, MINB) opt_rows_kernel(OptArgs a, const int32_t *tids,
                                                             const int64_t *tcnt) {
    constexpr int kOptU = UU;
    const int lane = threadIdx.x & 31;
    const int quad = lane % 7, sub = lane / 7;
    const int64_t n = *tcnt;
    const int64_t ngroups = (n + 3) >> 2;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (a.count && w == 0 && lane == 0) atomicAdd(reinterpret_cast<unsigned long long *>(a.count),
                                                  (unsigned long long)n);
    // row ids of the groups g0 + u*nw (u < kOptU); -1 = none.  The ids of the
    // next iteration are loaded before this iteration's rows are used, so
    // the id -> row dependency is off the critical path.
    auto load_ids = [&](int64_t g0, int32_t *ids) {
#pragma unroll
        for (int u = 0; u < kOptU; ++u) {
            const int64_t gi = g0 + u * nw;
            const int64_t j = gi * 4 + sub;
            ids[u] = (lane < 28 && gi < ngroups && j < n) ? __ldg(tids + j) : -1;
        }
    };
    int32_t cur[kOptU], nxt[kOptU];
    load_ids(w, cur);
    for (int64_t g0 = w; g0 < ngroups; g0 += nw * kOptU) {
        float4 g4[kOptU], t4[kOptU], v4[kOptU];
        float den[kOptU];
        int32_t cell[kOptU];
#pragma unroll
        for (int u = 0; u < kOptU; ++u) {
            if (cur[u] < 0) continue;
            const int64_t r = cur[u];
            g4[u] = reinterpret_cast<const float4 *>(a.grad + r * PLX_STRIDE)[quad];
            t4[u] = reinterpret_cast<const float4 *>(a.table + r * PLX_STRIDE)[quad];
            if (quad == 0) {   // merged after all loads are issued
                den[u] = a.density[r];
                cell[u] = a.sigma_lat ? a.row_cell[r] : 0;
            }
            if (a.rmsprop) v4[u] = reinterpret_cast<const float4 *>(a.v + r * PLX_STRIDE)[quad];
        }
        load_ids(g0 + nw * kOptU, nxt);
#pragma unroll
        for (int u = 0; u < kOptU; ++u) {
            if (cur[u] < 0) continue;
            const int64_t r = cur[u];
            if (quad == 0) t4[u].x = den[u];
            opt_apply(a, quad, g4[u], t4[u], v4[u]);
            if (quad == 0) {   // sigma lives in the density array (column 0 unused)
                a.density[r] = t4[u].x;
                lat_update(a, cell[u], t4[u].x);
                t4[u].x = 0.f;
            }
            reinterpret_cast<float4 *>(a.table + r * PLX_STRIDE)[quad] = t4[u];
            if (a.rmsprop) reinterpret_cast<float4 *>(a.v + r * PLX_STRIDE)[quad] = v4[u];
            if (a.clear)
                reinterpret_cast<float4 *>(a.grad + r * PLX_STRIDE)[quad] =
                    make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kOptU; ++u) cur[u] = nxt[u];
    }
}

static int g_num_sms = 0;
static int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

static int opt_blocks_per_sm() {
    static int nb = 0;
    if (!nb) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, opt_kernel<256>, 256, 0);
        if (nb <= 0) nb = 1;
    }
    return nb;
}

template <int NT>
__global__ void __launch_bounds__(NT) count_kernel(const uint8_t *m, int64_t n,
                                                   unsigned long long *count) {
    using BR = cub::BlockReduce<int, NT>;
    __shared__ typename BR::TempStorage tmp;
    int c = 0;
    const int64_t stride = (int64_t)gridDim.x * NT * 16;
    for (int64_t base = ((int64_t)blockIdx.x * NT + threadIdx.x) * 16; base < n; base += stride) {
        if (base + 16 <= n && ((reinterpret_cast<uintptr_t>(m) & 15) == 0)) {
            const uint4 v = *reinterpret_cast<const uint4 *>(m + base);
            const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                // count nonzero bytes
                unsigned x = w[e];
                x = (x | (x >> 4)) & 0x0f0f0f0fu;
                x = (x | (x >> 2)) & 0x03030303u;
                x = (x | (x >> 1)) & 0x01010101u;
                c += __popc(x);
            }
        } else {
            for (int64_t i = base; i < n && i < base + 16; ++i) c += m[i] != 0;
        }
    }
    const int s = BR(tmp).Sum(c);
    if (threadIdx.x == 0 && s) atomicAdd(count, (unsigned long long)s);
}

// ----------------------------------------------------------- prune --------
__global__ void prune_deem_kernel(DGrid G, const double *weights, double thr, uint8_t *deemed,
                                  int64_t ncell) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    const int32_t r = G.links[c];
    uint8_t d = 0;
    if (r >= 0) {
        const double v = weights ? weights[r] : (double)G.density[r];
        d = v >= thr;
    }
    deemed[c] = d;
}

// One axis of the separable 3x3x3 box dilation (border_value = 0).
__global__ void dilate_axis_kernel(const uint8_t *in, uint8_t *out, int64_t ncell, int64_t stride,
                                   int64_t extent, const int32_t *links_and) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    const int64_t pos = (c / stride) % extent;
    uint8_t v = in[c];
    if (pos > 0) v |= in[c - stride];
    if (pos < extent - 1) v |= in[c + stride];
    if (links_and) v = v && links_and[c] >= 0;   // survive = occ & dilated
    out[c] = v;
}

__global__ void prune_apply_kernel(DGrid G, const int32_t *new_links, int64_t ncell,
                                   int64_t *kept_old, float *new_table, float *new_density) {
    // one warp-quarter (8 lanes) per cell: 7 lanes copy the row as float4
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t c = t >> 3;
    const int part = t & 7;
    if (c >= ncell) return;
    const int32_t id = new_links[c];
    if (id < 0) return;
    const int32_t old = G.links[c];
    if (part == 7) {
        if (kept_old) kept_old[id] = old;
        new_density[id] = G.density[old];
        return;
    }
    reinterpret_cast<float4 *>(new_table + (int64_t)id * PLX_STRIDE)[part] =
        reinterpret_cast<const float4 *>(G.table + (int64_t)old * PLX_STRIDE)[part];
}

// -------------------------------------------------------- upsample --------
struct UpArgs {
    int64_t N[3];
    double spacing[3];
};

// New lattice point (i,j,k) -> stencil on the old grid (G:270-279), in the
// numpy operation order, float64, no contraction.
__device__ __forceinline__ bool up_stencil(const DGrid &G, const UpArgs &u, int64_t c,
                                           int32_t *rows, double *ws) {
    const int64_t NyNz = u.N[1] * u.N[2];
    const int64_t ijk[3] = {c / NyNz, (c % NyNz) / u.N[2], c % u.N[2]};
    const int64_t dm2[3] = {G.Dx - 2, G.Dy - 2, G.Dz - 2};
    double f[3];
    int64_t i0[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double p = G.lo[a] + (double)ijk[a] * u.spacing[a];
        double g = (p - G.lo[a]) * G.scale[a];
        if (g < 0.0) g = 0.0;
        if (g > G.dmax[a]) g = G.dmax[a];
        int64_t fl = (int64_t)floor(g);
        i0[a] = fl < dm2[a] ? fl : dm2[a];
        f[a] = g - (double)i0[a];
    }
    bool occ = false;
    int q = 0;
#pragma unroll
    for (int di = 0; di < 2; ++di) {
        const double wx = di ? f[0] : 1.0 - f[0];
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const double wy = dj ? f[1] : 1.0 - f[1];
#pragma unroll
            for (int dk = 0; dk < 2; ++dk) {
                const double wz = dk ? f[2] : 1.0 - f[2];
                const int32_t r = __ldg(G.links + flat(G, i0[0] + di, i0[1] + dj, i0[2] + dk));
                rows[q] = r;
                ws[q] = wx * wy * wz;
                occ |= (r >= 0) && ws[q] > 0.0;   // G:275-276: sum w*[occ] > 0
                ++q;
            }
        }
    }
    return occ;
}

__global__ void upsample_mark_kernel(DGrid G, UpArgs u, uint8_t *flags, int64_t ncell) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    int32_t rows[8];
    double ws[8];
    flags[c] = up_stencil(G, u, c, rows, ws);
}

__global__ void upsample_apply_kernel(DGrid G, UpArgs u, const int32_t *new_links, int64_t ncell,
                                      float *new_table, float *new_density) {
    // 7 lanes per new cell, each producing one float4 of the row (part 0
    // carries sigma from the density array in its first component)
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t c = t >> 3;
    const int part = t & 7;
    if (c >= ncell || part == 7) return;
    const int32_t id = new_links[c];
    if (id < 0) return;
    int32_t rows[8];
    double ws[8];
    up_stencil(G, u, c, rows, ws);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        if (rows[q] < 0) continue;   // empty corners read 0, no renormalisation
        float4 v = __ldg(reinterpret_cast<const float4 *>(G.table + (int64_t)rows[q] * PLX_STRIDE) + part);
        if (part == 0) v.x = __ldg(G.density + rows[q]);
        acc[0] += ws[q] * (double)v.x;
        acc[1] += ws[q] * (double)v.y;
        acc[2] += ws[q] * (double)v.z;
        acc[3] += ws[q] * (double)v.w;
    }
    if (part == 0) {
        new_density[id] = (float)acc[0];
        acc[0] = 0.0;
    }
    reinterpret_cast<float4 *>(new_table + (int64_t)id * PLX_STRIDE)[part] =
        make_float4((float)acc[0], (float)acc[1], (float)acc[2], (float)acc[3]);
}

// -------------------------------------------------- compaction scan -------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int64_t kScanTile = (int64_t)kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) scan_count_kernel(const uint8_t *flags, int64_t n,
                                                                  int64_t *partial) {
    using BR = cub::BlockReduce<int, kScanThreads>;
    __shared__ typename BR::TempStorage tmp;
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int c = 0;
#pragma unroll
    for (int e = 0; e < kScanItems; ++e) c += (base + e < n) && flags[base + e];
    const int s = BR(tmp).Sum(c);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) scan_partials_kernel(int64_t *partial, int64_t nb,
                                                             int64_t *count) {
    // single block: exclusive scan of nb partial counts
    __shared__ int64_t sh[1024];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < nb; base += 1024) {
        const int64_t i = base + threadIdx.x;
        const int64_t v = i < nb ? partial[i] : 0;
        sh[threadIdx.x] = v;
        __syncthreads();
        for (int off = 1; off < 1024; off <<= 1) {
            int64_t y = threadIdx.x >= (unsigned)off ? sh[threadIdx.x - off] : 0;
            __syncthreads();
            sh[threadIdx.x] += y;
            __syncthreads();
        }
        if (i < nb) partial[i] = carry + sh[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += sh[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) *count = carry;
}

__global__ void __launch_bounds__(kScanThreads) scan_write_kernel(const uint8_t *flags, int64_t n,
                                                                  const int64_t *partial,
                                                                  int32_t *ids) {
    __shared__ int sh[kScanThreads];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint8_t f[kScanItems];
    int c = 0;
#pragma unroll
    for (int e = 0; e < kScanItems; ++e) {
        f[e] = (base + e < n) ? flags[base + e] : 0;
        c += f[e] != 0;
    }
    sh[threadIdx.x] = c;
    __syncthreads();
    for (int off = 1; off < kScanThreads; off <<= 1) {
        int y = threadIdx.x >= (unsigned)off ? sh[threadIdx.x - off] : 0;
        __syncthreads();
        sh[threadIdx.x] += y;
        __syncthreads();
    }
    int64_t id = partial[blockIdx.x] + sh[threadIdx.x] - c;
#pragma unroll
    for (int e = 0; e < kScanItems; ++e) {
        if (base + e >= n) break;
        ids[base + e] = f[e] ? (int32_t)(id++) : -1;
    }
}

// Ordered variant: list[rank] = i for every flagged element (ascending).
__global__ void __launch_bounds__(kScanThreads) scan_list_kernel(const uint8_t *flags, int64_t n,
                                                                 const int64_t *partial,
                                                                 int32_t *list) {
    __shared__ int sh[kScanThreads];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint8_t f[kScanItems];
    int c = 0;
#pragma unroll
    for (int e = 0; e < kScanItems; ++e) {
        f[e] = (base + e < n) ? flags[base + e] : 0;
        c += f[e] != 0;
    }
    sh[threadIdx.x] = c;
    __syncthreads();
    for (int off = 1; off < kScanThreads; off <<= 1) {
        int y = threadIdx.x >= (unsigned)off ? sh[threadIdx.x - off] : 0;
        __syncthreads();
        sh[threadIdx.x] += y;
        __syncthreads();
    }
    int64_t id = partial[blockIdx.x] + sh[threadIdx.x] - c;
#pragma unroll
    for (int e = 0; e < kScanItems; ++e)
        if (f[e]) list[id++] = (int32_t)(base + e);
}

// ---------------------------------------------------- cell bitmask --------
__global__ void cell_occ_kernel(DGrid G, uint32_t *words, int64_t nwords, int64_t ncell) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nwords) return;
    const int64_t Dyz = (int64_t)G.Dy * G.Dz;
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
        const int64_t c = w * 32 + b;
        if (c >= ncell) break;
        const int64_t i = c / Dyz, j = (c % Dyz) / G.Dz, k = c % G.Dz;
        if (i >= G.Dx - 1 || j >= G.Dy - 1 || k >= G.Dz - 1) continue;
        const int32_t *p = G.links + c;
        const bool any = p[0] >= 0 || p[1] >= 0 || p[G.Dz] >= 0 || p[G.Dz + 1] >= 0 ||
                         p[Dyz] >= 0 || p[Dyz + 1] >= 0 || p[Dyz + G.Dz] >= 0 ||
                         p[Dyz + G.Dz + 1] >= 0;
        if (any) bits |= 1u << b;
    }
    words[w] = bits;
}

// Lattice sigma mirror: point c -> density of its row, NaN where empty.
__global__ void sigma_lat_kernel(DGrid G, float *out, int64_t ncell) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    const int32_t r = G.links[c];
    out[c] = r >= 0 ? G.density[r] : __int_as_float(0x7fc00000);
}

__global__ void row_cell_kernel(const int32_t *links, int64_t ncell, int32_t *row_cell) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    const int32_t r = links[c];
    if (r >= 0) row_cell[r] = (int32_t)c;
}

}  // namespace plx

using namespace plx;

namespace {
bool grid_ok(const plx_grid *g) {
    return g && g->links && g->dims[0] >= 2 && g->dims[1] >= 2 && g->dims[2] >= 2 &&
           (g->rows == 0 || (g->table && g->density)) &&
           g->dims[0] * g->dims[1] * g->dims[2] < (int64_t)1 << 31;
}
int status() { return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA; }
unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
int64_t ncell(const plx_grid *g) { return g->dims[0] * g->dims[1] * g->dims[2]; }
}  // namespace

#include "plx_internal.h"

extern "C" int plx_tv(const plx_grid *g, const int64_t *cells, int64_t start, int64_t count,
                      double fac_x, double fac_y, double fac_z, double eps, double f_sigma,
                      double f_sh, int32_t wrap_x, int32_t wrap_y, int32_t wrap_z,
                      int32_t with_grad, plx_grad *gb, double *out_sums, void *stream) {
    return plx::tv_impl(g, cells, start, nullptr, count, fac_x, fac_y, fac_z, eps, f_sigma, f_sh,
                        wrap_x, wrap_y, wrap_z, with_grad, gb, out_sums, stream, 0);
}

int plx::tv_impl(const plx_grid *g, const int64_t *cells, int64_t start, const int64_t *start_dev,
                 int64_t count, double fac_x, double fac_y, double fac_z, double eps,
                 double f_sigma, double f_sh, int32_t wrap_x, int32_t wrap_y, int32_t wrap_z,
                 int32_t with_grad, plx_grad *gb, double *out_sums, void *stream, int short_blocks) {
    if (!grid_ok(g) || !out_sums || count < 0 || (with_grad && (!gb || !gb->grad || !gb->tmask)))
        return PLX_EINVAL;
    if (count == 0) return PLX_OK;
    TvArgs a;
    a.cells = cells;
    a.start_dev = start_dev;
    a.start = start;
    a.count = count;
    a.ncell = ncell(g);
    a.fac[0] = fac_x;
    a.fac[1] = fac_y;
    a.fac[2] = fac_z;
    a.eps = eps;
    a.f_sigma = f_sigma;
    a.f_sh = f_sh;
    a.wrap[0] = wrap_x;
    a.wrap[1] = wrap_y;
    a.wrap[2] = wrap_z;
    a.with_grad = with_grad;
    a.grad = gb ? gb->grad : nullptr;
    a.tmask = gb ? gb->tmask : nullptr;
    a.sums = out_sums;
    constexpr int NT = 256;
    // 8 warps x 4 cells per block iteration, at most one resident wave
    // identity-linked dense grids: every cell has an SH term (C2: the
    // two-phase kernel measured 54.9 vs 51.3 us there); sparse grids: the
    // two-phase kernel (C3 at 512^3: 362 -> 226 us, the step 0.568 -> 0.437 ms)
    const DGrid G = make_dgrid(*g);
    static int bps_dense = 0, bps_sparse = 0;
    if (!bps_dense) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_dense, tv_dense_kernel<NT>, NT, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_sparse, tv_sparse_kernel<NT>, NT, 0);
        if (bps_dense <= 0) bps_dense = 1;
        if (bps_sparse <= 0) bps_sparse = 1;
    }
    // cells per block iteration: 32 (dense: 8 warps x 4), NT (sparse: a cell per thread)
    const int64_t per = G.identity ? 32 : NT;
    const int bps = G.identity ? bps_dense : bps_sparse;
    int64_t nb = (count + per - 1) / per;
    // short_blocks: one iteration per block, so the blocks of a background
    // TV yield their SM slots quickly to a higher-priority stream's kernels;
    // else one resident wave
    if (!short_blocks && nb > (int64_t)num_sms() * bps) nb = (int64_t)num_sms() * bps;
    if (G.identity)
        tv_dense_kernel<NT><<<(unsigned)nb, NT, 0, (cudaStream_t)stream>>>(G, a);
    else
        tv_sparse_kernel<NT><<<(unsigned)nb, NT, 0, (cudaStream_t)stream>>>(G, a);
    return status();
}

__global__ void count_from_list_kernel(const int64_t *tcnt, int64_t *out) {
    if (threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long *>(out),
                                    (unsigned long long)*tcnt);
}

// Zero the gradient rows of the compacted list (clear_grad, K:593-600):
// 7 lanes x float4 per row, no loads.
__global__ void clear_rows_kernel(float *grad, const int32_t *tids, const int64_t *tcnt) {
    const int64_t n = *tcnt;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * 7;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / 7;
        reinterpret_cast<float4 *>(grad + (int64_t)tids[j] * PLX_STRIDE)[t - j * 7] =
            make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

template <int UU, int MINB>
static void launch_rows_t(const OptArgs &a, const int32_t *tids, const int64_t *tcnt,
                          cudaStream_t s) {
    static int nbr = 0;
    if (!nbr) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbr, opt_rows_kernel<UU, MINB>, 256, 0);
        if (nbr <= 0) nbr = 1;
    }
    opt_rows_kernel<UU, MINB><<<(unsigned)(num_sms() * nbr), 256, 0, s>>>(a, tids, tcnt);
}

// 2 groups of 4 rows in flight per lane, 32 warps per SM: the A/B of 2-4
// groups x 16-32 warps measured within 2 % (the kernel runs at ~4.5 TB/s of
// scattered 112-byte row read-modify-writes).
static void launch_opt_rows(const OptArgs &a, const int32_t *tids, const int64_t *tcnt,
                            cudaStream_t s) {
    launch_rows_t<2, 4>(a, tids, tcnt, s);
}

extern "C" int plx_opt_step(plx_grid *g, float *v, plx_grad *gb, double lr_sigma, double lr_sh,
                            double beta, double eps, int32_t rmsprop, int32_t clear,
                            double *guard, int64_t *out_count, void *stream) {
    return plx::opt_step_impl(g, v, gb, lr_sigma, lr_sh, nullptr, beta, eps, rmsprop, clear, guard,
                              out_count, stream, 0, nullptr);
}

int plx::opt_step_impl(plx_grid *g, float *v, plx_grad *gb, double lr_sigma, double lr_sh,
                       const double *lr_dev, double beta, double eps, int32_t rmsprop,
                       int32_t clear, double *guard, int64_t *out_count, void *stream,
                       int tcnt_ready, double *host_sums) {
    if (!g || !gb || !gb->grad || !gb->tmask || (rmsprop && !v) ||
        (g->rows > 0 && (!g->table || !g->density)))
        return PLX_EINVAL;
    if ((gb->tids == nullptr) != (gb->tcnt == nullptr)) return PLX_EINVAL;
    if (g->rows == 0) return PLX_OK;
    // a mirror aliased to density (identity-linked dense grid) needs no upkeep
    float *lat = g->sigma_lat == g->density ? nullptr : g->sigma_lat;
    if (lat && !g->row_cell) return PLX_EINVAL;
    OptArgs a{g->table, g->density, v, gb->grad, lr_dev, guard, lat, g->row_cell, gb->tmask, g->rows,
              lr_sigma, lr_sh, beta, eps, rmsprop, clear, 1, reinterpret_cast<unsigned long long *>(out_count)};
    a.brick_dead = lat ? g->brick_dead : nullptr;
    a.Dx = (int32_t)g->dims[0];
    a.Dy = (int32_t)g->dims[1];
    a.Dz = (int32_t)g->dims[2];
    constexpr int NT = 256;
    cudaStream_t s = (cudaStream_t)stream;
    if (gb->tids) {   // two-phase: compact the touched set, then update the list
        if (!tcnt_ready && cudaMemsetAsync(gb->tcnt, 0, sizeof(int64_t), s) != cudaSuccess)
            return PLX_ECUDA;
        const int64_t nb = compact_grid(g->rows);
        touched_compact_kernel<<<(unsigned)nb, kCompactNT, 0, s>>>(gb->tmask, g->rows, gb->tids,
                                                                   gb->tcnt, clear, guard,
                                                                   host_sums);
        launch_opt_rows(a, gb->tids, gb->tcnt, s);
        return status();
    }
    const int64_t segs = (g->rows + 127) / 128;
    int64_t nb = (segs + NT / 32 - 1) / (NT / 32);
    if (nb > (int64_t)num_sms() * opt_blocks_per_sm()) nb = (int64_t)num_sms() * opt_blocks_per_sm();
    opt_kernel<NT><<<(unsigned)nb, NT, 0, s>>>(a);
    return status();
}

int plx::compact_mask_impl(uint8_t *tmask, int64_t rows, int32_t *tids, int64_t *tcnt,
                           int clear, void *stream) {
    if (!tmask || !tids || !tcnt || rows < 0) return PLX_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(tcnt, 0, sizeof(int64_t), s) != cudaSuccess) return PLX_ECUDA;
    if (rows == 0) return PLX_OK;
    const int64_t nb = compact_grid(rows);
    touched_compact_kernel<<<(unsigned)nb, kCompactNT, 0, s>>>(tmask, rows, tids, tcnt, clear,
                                                               nullptr, nullptr);
    return status();
}

extern "C" int plx_clear_grad(plx_grad *gb, int64_t rows, int64_t *out_count, void *stream) {
    if (!gb || !gb->grad || !gb->tmask || rows < 0) return PLX_EINVAL;
    if ((gb->tids == nullptr) != (gb->tcnt == nullptr)) return PLX_EINVAL;
    if (rows == 0) return PLX_OK;
    constexpr int NT = 256;
    cudaStream_t s = (cudaStream_t)stream;
    if (gb->tids) {   // compact + clear the mask, then zero the listed rows
        if (cudaMemsetAsync(gb->tcnt, 0, sizeof(int64_t), s) != cudaSuccess) return PLX_ECUDA;
        const int64_t nb = compact_grid(rows);
        touched_compact_kernel<<<(unsigned)nb, kCompactNT, 0, s>>>(gb->tmask, rows, gb->tids,
                                                                   gb->tcnt, 1, nullptr, nullptr);
        clear_rows_kernel<<<(unsigned)(num_sms() * 8), NT, 0, s>>>(gb->grad, gb->tids, gb->tcnt);
        if (out_count)
            count_from_list_kernel<<<1, 32, 0, s>>>(gb->tcnt, out_count);
        return status();
    }
    OptArgs a{nullptr, nullptr, nullptr, gb->grad, nullptr, nullptr, nullptr, nullptr, gb->tmask, rows,
              0.0, 0.0,
              0.0, 0.0, 0, 1, 0,
              reinterpret_cast<unsigned long long *>(out_count)};
    const int64_t segs = (rows + 127) / 128;
    int64_t nb = (segs + NT / 32 - 1) / (NT / 32);
    if (nb > (int64_t)num_sms() * opt_blocks_per_sm()) nb = (int64_t)num_sms() * opt_blocks_per_sm();
    opt_kernel<NT><<<(unsigned)nb, NT, 0, s>>>(a);
    return status();
}

extern "C" int plx_count_touched(const uint8_t *tmask, int64_t rows, int64_t *out_count,
                                 void *stream) {
    if (!tmask || !out_count || rows < 0) return PLX_EINVAL;
    if (rows == 0) return PLX_OK;
    constexpr int NT = 256;
    unsigned nb = blocks((rows + 15) / 16, NT);
    if (nb > 148 * 8) nb = 148 * 8;
    count_kernel<NT><<<nb, NT, 0, (cudaStream_t)stream>>>(
        tmask, rows, reinterpret_cast<unsigned long long *>(out_count));
    return status();
}

extern "C" int plx_prune_mark(const plx_grid *g, const double *weights, double threshold,
                              uint8_t *deemed_scratch, uint8_t *flags, void *stream) {
    if (!grid_ok(g) || !deemed_scratch || !flags) return PLX_EINVAL;
    const int64_t n = ncell(g);
    cudaStream_t s = (cudaStream_t)stream;
    DGrid G = make_dgrid(*g);
    uint8_t *A = deemed_scratch, *B = deemed_scratch + n;
    prune_deem_kernel<<<blocks(n, 256), 256, 0, s>>>(G, weights, threshold, A, n);
    const int64_t Dz = g->dims[2], Dy = g->dims[1], Dx = g->dims[0];
    dilate_axis_kernel<<<blocks(n, 256), 256, 0, s>>>(A, B, n, 1, Dz, nullptr);
    dilate_axis_kernel<<<blocks(n, 256), 256, 0, s>>>(B, A, n, Dz, Dy, nullptr);
    dilate_axis_kernel<<<blocks(n, 256), 256, 0, s>>>(A, flags, n, Dy * Dz, Dx, g->links);
    return status();
}

extern "C" int plx_prune_apply(const plx_grid *g, const int32_t *new_links, int64_t *kept_old,
                               float *new_table, float *new_density, void *stream) {
    if (!grid_ok(g) || !new_links || !new_table || !new_density) return PLX_EINVAL;
    const int64_t n = ncell(g);
    prune_apply_kernel<<<blocks(n * 8, 256), 256, 0, (cudaStream_t)stream>>>(
        make_dgrid(*g), new_links, n, kept_old, new_table, new_density);
    return status();
}

static UpArgs make_up(const plx_grid *g, const int64_t nd[3]) {
    UpArgs u;
    for (int a = 0; a < 3; ++a) {
        u.N[a] = nd[a];
        // G:272 spacing = extent / (new_dims - 1.0)
        u.spacing[a] = (g->hi[a] - g->lo[a]) / ((double)nd[a] - 1.0);
    }
    return u;
}

extern "C" int plx_upsample_mark(const plx_grid *g, const int64_t new_dims[3], uint8_t *flags,
                                 void *stream) {
    if (!grid_ok(g) || !new_dims || !flags || new_dims[0] < 2 || new_dims[1] < 2 || new_dims[2] < 2)
        return PLX_EINVAL;
    const int64_t n = new_dims[0] * new_dims[1] * new_dims[2];
    if (n >= (int64_t)1 << 31) return PLX_EINVAL;
    upsample_mark_kernel<<<blocks(n, 256), 256, 0, (cudaStream_t)stream>>>(make_dgrid(*g),
                                                                          make_up(g, new_dims), flags, n);
    return status();
}

extern "C" int plx_upsample_apply(const plx_grid *g, const int64_t new_dims[3],
                                  const int32_t *new_links, float *new_table, float *new_density,
                                  void *stream) {
    if (!grid_ok(g) || !new_dims || !new_links || !new_table || !new_density) return PLX_EINVAL;
    const int64_t n = new_dims[0] * new_dims[1] * new_dims[2];
    upsample_apply_kernel<<<blocks(n * 8, 256), 256, 0, (cudaStream_t)stream>>>(
        make_dgrid(*g), make_up(g, new_dims), new_links, n, new_table, new_density);
    return status();
}

extern "C" int64_t plx_scan_scratch_bytes(int64_t n) {
    return (int64_t)sizeof(int64_t) * ((n + kScanTile - 1) / kScanTile + 1);
}

extern "C" int plx_scan_ids(const uint8_t *flags, int64_t n, int32_t *ids, int64_t *count,
                            void *scratch, void *stream) {
    if (!flags || !ids || !count || !scratch || n < 0) return PLX_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nb = (n + kScanTile - 1) / kScanTile;
    int64_t *partial = reinterpret_cast<int64_t *>(scratch);
    if (nb == 0) {
        cudaMemsetAsync(count, 0, sizeof(int64_t), s);
        return status();
    }
    scan_count_kernel<<<(unsigned)nb, kScanThreads, 0, s>>>(flags, n, partial);
    scan_partials_kernel<<<1, 1024, 0, s>>>(partial, nb, count);
    scan_write_kernel<<<(unsigned)nb, kScanThreads, 0, s>>>(flags, n, partial, ids);
    return status();
}

extern "C" int plx_touched_list(const uint8_t *tmask, int64_t rows, int32_t *ids, int64_t *count,
                                void *scratch, void *stream) {
    if (!tmask || !ids || !count || !scratch || rows < 0) return PLX_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nb = (rows + kScanTile - 1) / kScanTile;
    int64_t *partial = reinterpret_cast<int64_t *>(scratch);
    if (nb == 0) {
        cudaMemsetAsync(count, 0, sizeof(int64_t), s);
        return status();
    }
    scan_count_kernel<<<(unsigned)nb, kScanThreads, 0, s>>>(tmask, rows, partial);
    scan_partials_kernel<<<1, 1024, 0, s>>>(partial, nb, count);
    scan_list_kernel<<<(unsigned)nb, kScanThreads, 0, s>>>(tmask, rows, partial, ids);
    return status();
}

extern "C" int64_t plx_cell_occ_words(const int64_t dims[3]) {
    return (dims[0] * dims[1] * dims[2] + 31) / 32;
}

extern "C" int plx_build_cell_occ(const plx_grid *g, uint32_t *cell_occ, void *stream) {
    if (!grid_ok(g) || !cell_occ) return PLX_EINVAL;
    const int64_t n = ncell(g), nw = (n + 31) / 32;
    cell_occ_kernel<<<blocks(nw, 256), 256, 0, (cudaStream_t)stream>>>(make_dgrid(*g), cell_occ, nw, n);
    return status();
}

// One block per brick, two cells per thread: a cell is skippable when its 8
// corner sigmas are all empty (NaN) or all occupied and < 0 -- exactly the
// two early exits of sigma_at -- and the brick is dead when all its cells
// are.  The mask is zeroed first; dead bricks set their bit.
__global__ void __launch_bounds__(256) brick_dead_kernel(DGrid G, uint32_t *bits) {
    const int32_t b = blockIdx.x;
    const int32_t bz = b % G.Bz, by = (b / G.Bz) % G.By, bx = b / (G.Bz * G.By);
    const int32_t sy = G.Dz, sx = G.Dy * G.Dz;
    bool dead = true;
    for (int t = threadIdx.x; t < kBrick * kBrick * kBrick; t += blockDim.x) {
        const int32_t i = bx * kBrick + t / (kBrick * kBrick), j = by * kBrick + (t / kBrick) % kBrick,
                      k = bz * kBrick + t % kBrick;
        if (i > G.Dx - 2 || j > G.Dy - 2 || k > G.Dz - 2) continue;
        const float *base = G.sigma_lat + flat(G, i, j, k);
        bool all_empty = true, all_neg = true;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float v = base[((q >> 2) & 1) * sx + ((q >> 1) & 1) * sy + (q & 1)];
            all_empty &= v != v;
            all_neg &= v < 0.f;   // NaN compares false
        }
        dead &= all_empty || all_neg;
    }
    dead = __syncthreads_and(dead);
    if (dead && threadIdx.x == 0) atomicOr(bits + (b >> 5), 1u << (b & 31));
}

extern "C" int64_t plx_brick_words(const int64_t dims[3]) {
    int64_t n = 1;
    for (int a = 0; a < 3; ++a) n *= (dims[a] - 2) / kBrick + 1;
    return (n + 31) / 32;
}

extern "C" int plx_build_brick_dead(const plx_grid *g, uint32_t *brick_dead, void *stream) {
    if (!grid_ok(g) || !brick_dead || !g->sigma_lat) return PLX_EINVAL;
    plx_grid gg = *g;
    gg.brick_dead = brick_dead;
    const DGrid G = make_dgrid(gg);
    const int64_t nb = (int64_t)G.Bx * G.By * G.Bz;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(brick_dead, 0, ((nb + 31) / 32) * sizeof(uint32_t), s) != cudaSuccess)
        return PLX_ECUDA;
    brick_dead_kernel<<<(unsigned)nb, 256, 0, s>>>(G, brick_dead);
    return status();
}

extern "C" int plx_build_sigma_lat(const plx_grid *g, float *sigma_lat, void *stream) {
    if (!grid_ok(g) || !sigma_lat) return PLX_EINVAL;
    const int64_t n = ncell(g);
    sigma_lat_kernel<<<blocks(n, 256), 256, 0, (cudaStream_t)stream>>>(make_dgrid(*g), sigma_lat, n);
    return status();
}

extern "C" int plx_build_row_cell(const plx_grid *g, int32_t *row_cell, void *stream) {
    if (!grid_ok(g) || !row_cell) return PLX_EINVAL;
    const int64_t n = ncell(g);
    row_cell_kernel<<<blocks(n, 256), 256, 0, (cudaStream_t)stream>>>(g->links, n, row_cell);
    return status();
}

// ------------------------------------------------ point sampling ---------
// SparseGrid.sample / sample_backward (G:154-223): the stencil of arbitrary
// world points in the reference's numpy order (float64 lattice coordinates,
// clipped, trilinear weights wx*wy*wz or the nearest point), one thread per
// point.  sample: out[n][28] = sum_q w_q table[row_q] over occupied corners,
// column 0 (sigma) clamped at zero.  backward: upstream * w_q added to every
// occupied corner row (touching it), the sigma entry masked where the
// interpolated sigma is negative.
template <bool NEAREST>
__device__ __forceinline__ int point_stencil(const DGrid &G, const double *p, int32_t *rows,
                                             double *w) {
    double g[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) g[a] = clamp_coord(p[a], G.lo[a], G.scale[a], G.dmax[a]);
    int ijk[3];
    if (NEAREST) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int D = a == 0 ? G.Dx : a == 1 ? G.Dy : G.Dz;
            int i = (int)floor(g[a] + 0.5);
            ijk[a] = i > D - 1 ? D - 1 : i;
        }
        rows[0] = __ldg(G.links + flat(G, ijk[0], ijk[1], ijk[2]));
        w[0] = 1.0;
        return 1;
    }
    double f[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int D = a == 0 ? G.Dx : a == 1 ? G.Dy : G.Dz;
        int i = (int)floor(g[a]);
        ijk[a] = i > D - 2 ? D - 2 : i;
        f[a] = g[a] - (double)ijk[a];
    }
    load_rows<false>(G, ijk, rows);
#pragma unroll
    for (int q = 0; q < 8; ++q) w[q] = stencil_w<false>(f, q);
    return 8;
}

template <bool NEAREST>
__global__ void grid_sample_kernel(DGrid G, const double *pts, int64_t n, double *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t rows[8];
        double w[8];
        const int nq = point_stencil<NEAREST>(G, pts + 3 * i, rows, w);
        double acc[28];
#pragma unroll
        for (int c = 0; c < 28; ++c) acc[c] = 0.0;
        for (int q = 0; q < nq; ++q) {
            if (rows[q] < 0) continue;   // empty corner reads 0 (G:193-194)
            const float *row = G.table + (int64_t)rows[q] * PLX_STRIDE;
            acc[0] += w[q] * (double)__ldg(G.density + rows[q]);
#pragma unroll
            for (int c = 1; c < 28; ++c) acc[c] += w[q] * (double)__ldg(row + c);
        }
        double *o = out + 28 * i;
        o[0] = acc[0] > 0.0 ? acc[0] : 0.0;   // G:196
#pragma unroll
        for (int c = 1; c < 28; ++c) o[c] = acc[c];
    }
}

template <bool NEAREST>
__global__ void grid_sample_bwd_kernel(DGrid G, const double *pts, const double *up, int64_t n,
                                       float *grad, uint8_t *tmask) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t rows[8];
        double w[8];
        const int nq = point_stencil<NEAREST>(G, pts + 3 * i, rows, w);
        double raw = 0.0;   // G:216-218: interpolated sigma before the clamp
        for (int q = 0; q < nq; ++q)
            if (rows[q] >= 0) raw += w[q] * (double)__ldg(G.density + rows[q]);
        const double *u = up + 28 * i;
        const double u0 = raw < 0.0 ? 0.0 : u[0];
        for (int q = 0; q < nq; ++q) {
            const int32_t r = rows[q];
            if (r < 0) continue;
            tmask[r] = 1;   // GradientBuffer.add touches the row (G:52-60)
            float *gr = grad + (int64_t)r * PLX_STRIDE;
            atomicAdd(gr, (float)(w[q] * u0));
            for (int c = 1; c < 28; ++c) {
                const float v = (float)(w[q] * u[c]);
                if (v != 0.f) atomicAdd(gr + c, v);
            }
        }
    }
}

extern "C" int plx_grid_sample(const plx_grid *g, const double *pts, int64_t n, int32_t nearest,
                               double *out, void *stream) {
    if (!grid_ok(g) || n < 0 || (n > 0 && (!pts || !out))) return PLX_EINVAL;
    if (n == 0) return PLX_OK;
    int64_t nb = (n + 255) / 256;
    if (nb > (int64_t)num_sms() * 16) nb = (int64_t)num_sms() * 16;
    plx_grid g2 = *g;
    g2.sigma_lat = nullptr;   // rows through links (the lattice mirror is not used here)
    g2.cell_occ = nullptr;
    if (nearest)
        grid_sample_kernel<true><<<(unsigned)nb, 256, 0, (cudaStream_t)stream>>>(make_dgrid(g2), pts, n, out);
    else
        grid_sample_kernel<false><<<(unsigned)nb, 256, 0, (cudaStream_t)stream>>>(make_dgrid(g2), pts, n, out);
    return status();
}

extern "C" int plx_grid_sample_backward(const plx_grid *g, const double *pts,
                                        const double *upstream, int64_t n, int32_t nearest,
                                        plx_grad *gb, void *stream) {
    if (!grid_ok(g) || n < 0 || !gb || !gb->grad || !gb->tmask ||
        (n > 0 && (!pts || !upstream)))
        return PLX_EINVAL;
    if (n == 0) return PLX_OK;
    int64_t nb = (n + 255) / 256;
    if (nb > (int64_t)num_sms() * 16) nb = (int64_t)num_sms() * 16;
    plx_grid g2 = *g;
    g2.sigma_lat = nullptr;
    g2.cell_occ = nullptr;
    if (nearest)
        grid_sample_bwd_kernel<true><<<(unsigned)nb, 256, 0, (cudaStream_t)stream>>>(
            make_dgrid(g2), pts, upstream, n, gb->grad, gb->tmask);
    else
        grid_sample_bwd_kernel<false><<<(unsigned)nb, 256, 0, (cudaStream_t)stream>>>(
            make_dgrid(g2), pts, upstream, n, gb->grad, gb->tmask);
    return status();
}

extern "C" const char *plx_version(void) { return "plx-b200 0.1.0 (sm_100a)"; }

extern "C" int plx_device_check(void) {
    int dev = 0, major = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 1;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return 1;
    return major >= 10 ? 0 : 1;
}
