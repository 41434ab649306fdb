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

namespace plx {
int opt_step_impl(plx_grid *g, float *v, plx_grad *gb, double lr_sigma, double lr_sh,
                  const double *lr_dev, double beta, double eps, int32_t rmsprop, int32_t clear,
                  double *guard, int64_t *out_count, void *stream);
int tv_impl(const plx_grid *g, const int64_t *cells, int64_t start, const int64_t *start_dev,
            int64_t count, double fac_x, double fac_y, double fac_z, double eps, double f_sigma,
            double f_sh, int32_t wrap_x, int32_t wrap_y, int32_t wrap_z, int32_t with_grad,
            plx_grad *gb, double *out_sums, void *stream);
}  // namespace plx

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

extern "C" int plx_train_step(plx_grid *g, plx_grad *gb, const plx_step_args *a, void *stream) {
    if (!g || !gb || !a || !a->sums) return PLX_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    auto ev = [&](int i) {
        if (a->events[i]) cudaEventRecord((cudaEvent_t)a->events[i], s);
    };
    if (cudaMemsetAsync(a->sums, 0, 4 * sizeof(double), s) != cudaSuccess) return PLX_ECUDA;
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
    int rc = plx_render_fused_bwd(g, &a->rays, &a->opts, 1, a->up_scale, a->lam_cauchy, gb,
                                  nullptr, a->sums, a->scratch, a->scratch_bytes, stream);
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
        if (a->count && cudaMemsetAsync(a->count, 0, sizeof(int64_t), s) != cudaSuccess)
            return PLX_ECUDA;
        rc = plx::opt_step_impl(g, a->v, gb, a->lr_sigma, a->lr_sh, a->dev_lr, a->beta, a->eps,
                                a->rmsprop, 1, a->sums, a->count, stream);
        if (rc != PLX_OK) return rc;
    }
    ev(3);
    return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA;
}
