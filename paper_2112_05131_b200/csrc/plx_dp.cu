// plx_dp.cu -- data-parallel gradient exchange + update for the ray-sharded
// training step.  Rays shard across GPUs, the grid is
// replicated, and every step ends with one exchange of the touched rows'
// gradients followed by the (replicated) RMSProp/SGD update, K:572-600.
//
// Two paths:
//   * NCCL (baseline): OR of the touched masks (all_reduce MAX), ordered
//     compaction of the union (plx_touched_list), rows packed
//     (plx_pack_rows), one all_reduce(SUM) of the packed rows, then
//     plx_opt_step_list updates the union straight from the packed buffer.
//   * NVLink peer memory (plx_dp_owner_update): one kernel per rank does the
//     reduce-scatter, the update and the all-gather at once.  Rank o owns a
//     contiguous 1/N slice of the rows: it ORs the N ranks' touched masks
//     for its slice, sums the N ranks' gradient rows (peer loads), updates
//     sigma / SH with its own RMSProp state, and stores the new rows into
//     every rank's grid (peer stores), so the transfer overlaps the update
//     row by row and nothing is packed.  The host brackets it with two tiny
//     NCCL all_reduces (loss sums before, touched count after) that order
//     it against the other ranks' render and clear.
#include <cuda.h>

#include "plx_optim.cuh"

namespace plx {

__global__ void pack_rows_kernel(const float *src, const int32_t *ids, const int64_t *count,
                                 float *dst) {
    const int64_t n = *count;
    const int64_t tot = n * 7;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / 7;
        const int q = (int)(t - j * 7);
        reinterpret_cast<float4 *>(dst + j * PLX_ROW)[q] =   // packed: 28-float pitch
            __ldg(reinterpret_cast<const float4 *>(src + (int64_t)ids[j] * PLX_STRIDE) + q);
    }
}

struct ListArgs {
    float *table, *density, *v, *grad;
    const float *gpack;        // packed gradients of the list (NULL = grad rows)
    uint8_t *tmask;
    float *sigma_lat;
    const int32_t *row_cell;
    uint32_t *brick_dead;      // optional dead-brick mask beside sigma_lat
    int32_t Dx, Dy, Dz;
    const int32_t *ids;
    const int64_t *count;
    double *guard;
    unsigned long long *out_count;
    OptHyper h;
    int clear;
};

// Update the rows ids[0..count) (4 rows x 7 float4 per warp iteration).
__global__ void __launch_bounds__(256, 2) opt_list_kernel(ListArgs a) {
    if (guard_halts(a.guard)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) a.guard[4] = 1.0;
        return;
    }
    const int lane = threadIdx.x & 31;
    const int quad = lane % 7, sub = lane / 7;
    const int64_t n = *a.count;
    const int64_t ngroups = (n + 3) >> 2;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (a.out_count && w == 0 && lane == 0) atomicAdd(a.out_count, (unsigned long long)n);
    for (int64_t gi = w; gi < ngroups; gi += nw) {
        const int64_t j = gi * 4 + sub;
        if (lane >= 28 || j >= n) continue;
        const int64_t r = a.ids[j];
        float4 g4 = a.gpack ? reinterpret_cast<const float4 *>(a.gpack + j * PLX_ROW)[quad]
                            : reinterpret_cast<const float4 *>(a.grad + r * PLX_STRIDE)[quad];
        float4 t4 = reinterpret_cast<const float4 *>(a.table + r * PLX_STRIDE)[quad];
        float4 v4 = a.h.rmsprop ? reinterpret_cast<const float4 *>(a.v + r * PLX_STRIDE)[quad]
                                : make_float4(0.f, 0.f, 0.f, 0.f);
        float den = 0.f;
        int32_t cell = 0;
        if (quad == 0) {
            den = a.density[r];
            cell = a.sigma_lat ? a.row_cell[r] : 0;
            t4.x = den;
        }
        opt_apply4(a.h, quad, g4, t4, v4);
        if (quad == 0) {   // sigma lives in the density array (column 0 unused)
            a.density[r] = t4.x;
            if (a.sigma_lat) a.sigma_lat[cell] = t4.x;
            if (a.brick_dead && t4.x >= 0.f) brick_revive(a.brick_dead, cell, a.Dx, a.Dy, a.Dz);
            t4.x = 0.f;
            if (a.clear) a.tmask[r] = 0;
        }
        reinterpret_cast<float4 *>(a.table + r * PLX_STRIDE)[quad] = t4;
        if (a.h.rmsprop) reinterpret_cast<float4 *>(a.v + r * PLX_STRIDE)[quad] = v4;
        if (a.clear)
            reinterpret_cast<float4 *>(a.grad + r * PLX_STRIDE)[quad] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

constexpr int kMaxPeers = 8;

struct DpArgs {  // kernel-side copy of plx_dp_peers + update scalars
    int n, rank;
    int64_t rows, lo, hi;                 // owned row range [lo, hi)
    float *grad[kMaxPeers];
    const uint8_t *tmask[kMaxPeers];
    float *table[kMaxPeers];
    float *density[kMaxPeers];
    float *lat[kMaxPeers];                // lattice sigma mirrors (may be NULL)
    float *v;                             // this rank's RMSProp state (owned rows only)
    const int32_t *row_cell;
    double *guard;
    unsigned long long *out_count;
    OptHyper h;
};

__device__ __forceinline__ int nz_bytes(uint32_t m) {
    m = (m | (m >> 4)) & 0x0f0f0f0fu;
    m = (m | (m >> 2)) & 0x03030303u;
    m = (m | (m >> 1)) & 0x01010101u;
    return __popc(m);
}

// Owner-computes: union of the N touched masks over the owned slice,
// gradient sum over the N ranks (rank order, so it is reproducible), update,
// and the new rows stored into every rank's grid.
__global__ void __launch_bounds__(256) dp_owner_update_kernel(DpArgs a) {
    __shared__ uint8_t list[8][128];
    __shared__ uint8_t ranks[8][128];   // per listed row: bit k = rank k touched it
    if (guard_halts(a.guard)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) a.guard[4] = 1.0;
        return;
    }
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int quad = lane % 7, sub = lane / 7;
    const int64_t seg0 = a.lo >> 7, seg1 = (a.hi + 127) >> 7;   // lo is 128-aligned
    const int64_t nw = (int64_t)gridDim.x * 8;
    unsigned long long cnt = 0;
    for (int64_t seg = seg0 + (int64_t)blockIdx.x * 8 + wib; seg < seg1; seg += nw) {
        const int64_t r0 = seg * 128 + lane * 4;
        uint32_t m = 0, rk = 0;   // rk: byte e = ranks that touched row r0 + e
        for (int k = 0; k < a.n; ++k) {
            uint32_t mk = 0;
            if (r0 + 3 < a.hi) {
                mk = *reinterpret_cast<const volatile uint32_t *>(a.tmask[k] + r0);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (r0 + e < a.hi && a.tmask[k][r0 + e]) mk |= 0xffu << (8 * e);
            }
            m |= mk;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if ((mk >> (8 * e)) & 0xffu) rk |= (1u << k) << (8 * e);
        }
        const int c = nz_bytes(m);
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
            if ((m >> (8 * e)) & 0xffu) {
                ranks[wib][pos] = (uint8_t)((rk >> (8 * e)) & 0xffu);
                list[wib][pos++] = (uint8_t)(lane * 4 + e);
            }
        __syncwarp();
        cnt += (unsigned long long)total;
        for (int gi = 0; gi < total; gi += 4) {
            const int j = gi + sub;
            if (lane < 28 && j < total) {
                const int64_t r = seg * 128 + list[wib][j];
                const unsigned rb = ranks[wib][j];
                float4 g4 = make_float4(0.f, 0.f, 0.f, 0.f);
                // only the ranks that touched the row hold a nonzero gradient
                // row: skip the others' peer reads (adding their zeros is the
                // identity, so the rank-order sum is unchanged)
                for (int k = 0; k < a.n; ++k) {
                    if (!((rb >> k) & 1u)) continue;
                    const float4 x = reinterpret_cast<const float4 *>(a.grad[k] + r * PLX_STRIDE)[quad];
                    g4.x += x.x;
                    g4.y += x.y;
                    g4.z += x.z;
                    g4.w += x.w;
                }
                float4 t4 = reinterpret_cast<const float4 *>(a.table[a.rank] + r * PLX_STRIDE)[quad];
                float4 v4 = a.h.rmsprop ? reinterpret_cast<const float4 *>(a.v + r * PLX_STRIDE)[quad]
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
                int32_t cell = 0;
                if (quad == 0) {
                    t4.x = a.density[a.rank][r];
                    if (a.row_cell) cell = a.row_cell[r];
                }
                opt_apply4(a.h, quad, g4, t4, v4);
                if (a.h.rmsprop) reinterpret_cast<float4 *>(a.v + r * PLX_STRIDE)[quad] = v4;
                const float sig = t4.x;
                if (quad == 0) t4.x = 0.f;
                for (int k = 0; k < a.n; ++k) {
                    reinterpret_cast<float4 *>(a.table[k] + r * PLX_STRIDE)[quad] = t4;
                    if (quad == 0) {
                        a.density[k][r] = sig;
                        if (a.lat[k]) a.lat[k][cell] = sig;
                    }
                }
            }
        }
        __syncwarp();
    }
    if (a.out_count && lane == 0 && cnt) atomicAdd(a.out_count, cnt);
    __threadfence_system();   // peer stores visible before the host's next collective
}

}  // namespace plx

using namespace plx;

namespace {
int status() { return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA; }
int sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}
}  // namespace

extern "C" int plx_pack_rows(const float *src, const int32_t *ids, const int64_t *count,
                             int64_t cap, float *dst, void *stream) {
    if (!src || !ids || !count || !dst || cap < 0) return PLX_EINVAL;
    if (cap == 0) return PLX_OK;
    int64_t nb = (cap * 7 + 255) / 256;
    if (nb > (int64_t)sms() * 8) nb = (int64_t)sms() * 8;
    pack_rows_kernel<<<(unsigned)nb, 256, 0, (cudaStream_t)stream>>>(src, ids, count, dst);
    return status();
}

extern "C" int plx_opt_step_list(plx_grid *g, float *v, plx_grad *gb, const int32_t *ids,
                                 const int64_t *count, const float *gpack, double lr_sigma,
                                 double lr_sh, double beta, double eps, int32_t rmsprop,
                                 int32_t clear, double *guard, int64_t *out_count, void *stream) {
    if (!g || !gb || !gb->grad || !gb->tmask || !ids || !count || (rmsprop && !v)) return PLX_EINVAL;
    if (g->rows > 0 && (!g->table || !g->density)) return PLX_EINVAL;
    float *lat = g->sigma_lat == g->density ? nullptr : g->sigma_lat;   // aliased: no upkeep
    if (lat && !g->row_cell) return PLX_EINVAL;
    if (g->rows == 0) return PLX_OK;
    ListArgs a;
    a.table = g->table;
    a.density = g->density;
    a.v = v;
    a.grad = gb->grad;
    a.gpack = gpack;
    a.tmask = gb->tmask;
    a.sigma_lat = lat;
    a.row_cell = g->row_cell;
    a.brick_dead = lat ? g->brick_dead : nullptr;
    a.Dx = (int32_t)g->dims[0];
    a.Dy = (int32_t)g->dims[1];
    a.Dz = (int32_t)g->dims[2];
    a.ids = ids;
    a.count = count;
    a.guard = guard;
    a.out_count = reinterpret_cast<unsigned long long *>(out_count);
    a.h = OptHyper{lr_sigma, lr_sh, beta, eps, rmsprop};
    a.clear = clear;
    static int nbr = 0;
    if (!nbr) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbr, opt_list_kernel, 256, 0);
        if (nbr <= 0) nbr = 1;
    }
    opt_list_kernel<<<(unsigned)(sms() * nbr), 256, 0, (cudaStream_t)stream>>>(a);
    return status();
}

extern "C" int plx_dp_owner_update(const plx_dp_peers *p, float *v, const int32_t *row_cell,
                                   double lr_sigma, double lr_sh, double beta, double eps,
                                   int32_t rmsprop, double *guard, int64_t *out_count,
                                   void *stream) {
    if (!p || p->n < 1 || p->n > kMaxPeers || p->rank < 0 || p->rank >= p->n || p->rows < 0 ||
        (rmsprop && !v))
        return PLX_EINVAL;
    DpArgs a;
    a.n = p->n;
    a.rank = p->rank;
    a.rows = p->rows;
    // owned slice: 128-row aligned, contiguous
    const int64_t nseg = (p->rows + 127) / 128;
    const int64_t s0 = nseg * p->rank / p->n, s1 = nseg * (p->rank + 1) / p->n;
    a.lo = s0 * 128;
    a.hi = s1 * 128 < p->rows ? s1 * 128 : p->rows;
    bool need_cell = false;
    for (int k = 0; k < p->n; ++k) {
        if (!p->grad[k] || !p->tmask[k] || !p->table[k] || !p->density[k]) return PLX_EINVAL;
        a.grad[k] = p->grad[k];
        a.tmask[k] = p->tmask[k];
        a.table[k] = p->table[k];
        a.density[k] = p->density[k];
        a.lat[k] = p->sigma_lat[k] == p->density[k] ? nullptr : p->sigma_lat[k];
        need_cell |= a.lat[k] != nullptr;
    }
    if (need_cell && !row_cell) return PLX_EINVAL;
    a.v = v;
    a.row_cell = row_cell;
    a.guard = guard;
    a.out_count = reinterpret_cast<unsigned long long *>(out_count);
    a.h = OptHyper{lr_sigma, lr_sh, beta, eps, rmsprop};
    if (a.hi <= a.lo) return PLX_OK;
    int64_t nb = (s1 - s0 + 7) / 8;
    if (nb > (int64_t)sms() * 4) nb = (int64_t)sms() * 4;
    dp_owner_update_kernel<<<(unsigned)nb, 256, 0, (cudaStream_t)stream>>>(a);
    return status();
}

// ---- CUDA IPC: map a peer process's device buffer -------------------------
extern "C" int plx_ipc_export(const void *ptr, uint8_t handle[64], int64_t *offset) {
    if (!ptr || !handle || !offset) return PLX_EINVAL;
    static CUresult (*get_range)(CUdeviceptr *, size_t *, CUdeviceptr) = nullptr;
    if (!get_range) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
                cudaSuccess || !fn)
            return PLX_ECUDA;
        get_range = reinterpret_cast<CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr)>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) return PLX_ECUDA;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)) != cudaSuccess) return PLX_ECUDA;
    memcpy(handle, &h, 64);
    *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(ptr) - base);
    return PLX_OK;
}

extern "C" int plx_ipc_import(const uint8_t handle[64], int64_t offset, void **base_out,
                              void **ptr_out) {
    if (!handle || !base_out || !ptr_out || offset < 0) return PLX_EINVAL;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    void *base = nullptr;
    if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return PLX_ECUDA;
    *base_out = base;
    *ptr_out = reinterpret_cast<char *>(base) + offset;
    return PLX_OK;
}

extern "C" int plx_ipc_close(void *base) {
    if (!base) return PLX_EINVAL;
    return cudaIpcCloseMemHandle(base) == cudaSuccess ? PLX_OK : PLX_ECUDA;
}
