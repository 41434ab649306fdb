// plx_step.cu -- one optimisation step of the trainer (T:441-486) as ONE host
// call: fused render + backward, TV, and (single GPU) the update with the
// fused clear and the device divergence guard.  The per-step Python cost of
// the reference's step body (batch gather, three kernel wrappers, loss
// check) becomes a descriptor update plus this call.  With the per-step
// scalars read from device memory (dev_tv_start, dev_lr) and the batch in a
// fixed buffer, the call's launches are captured once as a CUDA graph and
// replayed every step (Trainer, graph mode).
#include <cuda_runtime.h>

#include <cstdlib>

#include "../../include/plx.h"

#include "plx_internal.h"

namespace {
// Per-device side stream for the TV branch.  TV reads only the parameters
// (unchanged until the update) and adds into the gradient with the same
// red.add atomics and mask stores as the backward's scatter, so it can run
// beside the three backward kernels and fill their tails and the gaps
// between them (bench A/B: +1.8 % at the headline state, +3.5 % at step
// 2000; a high-priority side stream measured the same).  Created on the
// first (eager) call, never during capture.
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream g_side[64];

SideStream *side_for_current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    SideStream &ss = g_side[dev];
    if (!ss.s) {
        cudaStream_t st = nullptr;
        cudaEvent_t f = nullptr, j = nullptr;
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        if (cudaEventCreateWithFlags(&f, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&j, cudaEventDisableTiming) != cudaSuccess)
            return nullptr;
        ss.fork = f;
        ss.join = j;
        ss.s = st;
    }
    return &ss;
}
}  // namespace

// The step's first node: zeroes the loss sums (not the sticky halt flag
// sums[4]), the render scratch's 3 counters, the touched count and the
// compaction counter, and copies the per-step scalars from pinned host
// memory -- one kernel instead of four memsets and a memcpy in the graph.
__global__ void step_prologue_kernel(double *sums, int *counters, int64_t *count, int64_t *tcnt,
                                     const int64_t *host_params, int64_t *dev_params) {
    const int t = threadIdx.x;
    if (t < 4) sums[t] = 0.0;
    if (t < 3) counters[t] = 0;
    if (t == 0) {
        if (count) *count = 0;
        if (tcnt) *tcnt = 0;
    }
    if (host_params && t < 4) dev_params[t] = host_params[t];
}

extern "C" int plx_train_step(plx_grid *g, plx_grad *gb, const plx_step_args *a, void *stream) {
    if (!g || !gb || !a || !a->sums) return PLX_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    auto ev = [&](int i) {
        if (a->events[i]) cudaEventRecord((cudaEvent_t)a->events[i], s);
    };
    if (!a->scratch || (a->host_params && !a->dev_params)) return PLX_EINVAL;
    step_prologue_kernel<<<1, 32, 0, s>>>(a->sums, reinterpret_cast<int *>(a->scratch),
                                          a->update ? a->count : nullptr,
                                          a->update ? gb->tcnt : nullptr, a->host_params,
                                          a->dev_params);
    ev(0);
    // TV beside the backward unless per-leg events were asked for (timing)
    const bool timed = a->events[0] || a->events[1] || a->events[2] || a->events[3];
    SideStream *side = (a->tv_count > 0 && !timed && !getenv("PLX_TV_SERIAL"))
                           ? side_for_current_device() : nullptr;
    if (side) {
        if (cudaEventRecord(side->fork, s) != cudaSuccess ||
            cudaStreamWaitEvent(side->s, side->fork, 0) != cudaSuccess)
            return PLX_ECUDA;
        int rc = plx::tv_impl(g, nullptr, a->tv_start, a->dev_tv_start, a->tv_count, a->tv_fac[0],
                              a->tv_fac[1], a->tv_fac[2], a->tv_eps, a->tv_f_sigma, a->tv_f_sh, 0,
                              0, 0, 1, gb, a->sums + 2, side->s);
        if (rc != PLX_OK) return rc;
        if (cudaEventRecord(side->join, side->s) != cudaSuccess) return PLX_ECUDA;
    }
    int rc = plx::render_fused_bwd_impl(g, &a->rays, a->dev_idx_off, &a->opts, 1, a->up_scale,
                                        a->lam_cauchy, gb, nullptr, a->sums, a->scratch,
                                        a->scratch_bytes, stream, 1);
    if (rc != PLX_OK) return rc;
    ev(1);
    if (side) {
        if (cudaStreamWaitEvent(s, side->join, 0) != cudaSuccess) return PLX_ECUDA;
    } else if (a->tv_count > 0) {
        rc = plx::tv_impl(g, nullptr, a->tv_start, a->dev_tv_start, a->tv_count, a->tv_fac[0],
                          a->tv_fac[1], a->tv_fac[2], a->tv_eps, a->tv_f_sigma, a->tv_f_sh, 0, 0,
                          0, 1, gb, a->sums + 2, stream);
        if (rc != PLX_OK) return rc;
    }
    ev(2);
    if (a->update) {
        rc = plx::opt_step_impl(g, a->v, gb, a->lr_sigma, a->lr_sh, a->dev_lr, a->beta, a->eps,
                                a->rmsprop, 1, a->sums, a->count, stream, 1, a->host_sums);
        if (rc != PLX_OK) return rc;
    }
    ev(3);
    return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA;
}
