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
    cudaStream_t hp = nullptr;   // high-priority stream for the main path (PLX_PRIO)
    cudaEvent_t fork = nullptr, join = nullptr, in = nullptr, out = nullptr;
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
            cudaEventCreateWithFlags(&j, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.in, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.out, cudaEventDisableTiming) != cudaSuccess)
            return nullptr;
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        if (cudaStreamCreateWithPriority(&ss.hp, cudaStreamNonBlocking, greatest) != cudaSuccess)
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
    // TV beside the backward unless per-leg events were asked for (timing)
    const bool timed = a->events[0] || a->events[1] || a->events[2] || a->events[3];
    SideStream *side = (a->tv_count > 0 && !timed && !getenv("PLX_TV_SERIAL"))
                           ? side_for_current_device() : nullptr;
    // The main path runs on a high-priority stream and TV on the default-
    // priority side stream in short blocks: the block scheduler places
    // march / colour / scatter blocks first and TV fills the free slots
    // (A/B at the headline state: 9.51 M rays/s TV forked after the march,
    // 9.55 M with priorities alone, 9.67 M with short TV blocks too; step
    // 2000: 24.7 / 24.8 / 25.5 M).  PLX_PRIO=0: default-priority main path,
    // one-wave TV forked once the march is enqueued.
    const char *pe = getenv("PLX_PRIO");
    const bool prio = side && !(pe && pe[0] == '0');
    cudaStream_t m = s;
    if (prio) {
        if (cudaEventRecord(side->in, s) != cudaSuccess ||
            cudaStreamWaitEvent(side->hp, side->in, 0) != cudaSuccess)
            return PLX_ECUDA;
        m = side->hp;
    }
    if (!a->scratch || (a->host_params && !a->dev_params)) return PLX_EINVAL;
    step_prologue_kernel<<<1, 32, 0, m>>>(a->sums, reinterpret_cast<int *>(a->scratch),
                                          a->update ? a->count : nullptr,
                                          a->update ? gb->tcnt : nullptr, a->host_params,
                                          a->dev_params);
    ev(0);
    // without priorities TV forks once the march is enqueued (PLX_TV_FORK=
    // start: before it); with them it forks at the start
    const char *fe = getenv("PLX_TV_FORK");
    const bool fork_early = prio || (fe && fe[0] == 's');
    auto launch_tv = [&]() -> int {
        if (cudaStreamWaitEvent(side->s, side->fork, 0) != cudaSuccess) return PLX_ECUDA;
        int r = plx::tv_impl(g, nullptr, a->tv_start, a->dev_tv_start, a->tv_count, a->tv_fac[0],
                             a->tv_fac[1], a->tv_fac[2], a->tv_eps, a->tv_f_sigma, a->tv_f_sh, 0,
                             0, 0, 1, gb, a->sums + 2, side->s, prio ? 1 : 0);
        if (r != PLX_OK) return r;
        return cudaEventRecord(side->join, side->s) == cudaSuccess ? PLX_OK : PLX_ECUDA;
    };
    if (side && (fork_early || a->rays.n == 0)) {
        if (cudaEventRecord(side->fork, m) != cudaSuccess) return PLX_ECUDA;
        const int r = launch_tv();
        if (r != PLX_OK) return r;
    }
    int rc = plx::render_fused_bwd_impl(g, &a->rays, a->dev_idx_off, &a->opts, 1, a->up_scale,
                                        a->lam_cauchy, gb, nullptr, a->sums, a->scratch,
                                        a->scratch_bytes, (void *)m, 1,
                                        (side && !fork_early && a->rays.n > 0) ? side->fork
                                                                               : nullptr);
    if (rc != PLX_OK) return rc;
    if (side && !fork_early && a->rays.n > 0) {
        rc = launch_tv();
        if (rc != PLX_OK) return rc;
    }
    ev(1);
    if (side) {
        if (cudaStreamWaitEvent(m, side->join, 0) != cudaSuccess) return PLX_ECUDA;
    } else if (a->tv_count > 0) {
        rc = plx::tv_impl(g, nullptr, a->tv_start, a->dev_tv_start, a->tv_count, a->tv_fac[0],
                          a->tv_fac[1], a->tv_fac[2], a->tv_eps, a->tv_f_sigma, a->tv_f_sh, 0, 0,
                          0, 1, gb, a->sums + 2, stream);
        if (rc != PLX_OK) return rc;
    }
    ev(2);
    if (a->update) {
        rc = plx::opt_step_impl(g, a->v, gb, a->lr_sigma, a->lr_sh, a->dev_lr, a->beta, a->eps,
                                a->rmsprop, 1, a->sums, a->count, (void *)m, 1, a->host_sums);
        if (rc != PLX_OK) return rc;
    }
    if (prio) {
        if (cudaEventRecord(side->out, m) != cudaSuccess ||
            cudaStreamWaitEvent(s, side->out, 0) != cudaSuccess)
            return PLX_ECUDA;
    }
    ev(3);
    return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA;
}

extern "C" int plx_release_streams(void) {
    int dev0 = 0;
    cudaGetDevice(&dev0);
    for (int d = 0; d < 64; ++d) {
        SideStream &ss = g_side[d];
        if (!ss.s) continue;
        cudaSetDevice(d);
        cudaStreamSynchronize(ss.s);
        cudaStreamSynchronize(ss.hp);
        cudaEventDestroy(ss.fork);
        cudaEventDestroy(ss.join);
        cudaEventDestroy(ss.in);
        cudaEventDestroy(ss.out);
        cudaStreamDestroy(ss.s);
        cudaStreamDestroy(ss.hp);
        ss = SideStream();
    }
    cudaSetDevice(dev0);
    return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA;
}
