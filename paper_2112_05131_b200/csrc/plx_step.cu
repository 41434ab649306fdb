// plx_step.cu -- one optimisation step of the trainer (T:441-486) as ONE host
// call: fused render + backward, TV, and (single GPU) the update with the
// fused clear and the device divergence guard.  The per-step Python cost of
// the reference's step body (batch gather, three kernel wrappers, loss
// check) becomes a descriptor update plus this call, so the host stays ahead
// of the GPU even at ~0.3 ms steps.
#include <cuda_runtime.h>

#include "../../include/plx.h"

extern "C" int plx_train_step(plx_grid *g, plx_grad *gb, const plx_step_args *a, void *stream) {
    if (!g || !gb || !a || !a->sums) return PLX_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    auto ev = [&](int i) {
        if (a->events[i]) cudaEventRecord((cudaEvent_t)a->events[i], s);
    };
    if (cudaMemsetAsync(a->sums, 0, 4 * sizeof(double), s) != cudaSuccess) return PLX_ECUDA;
    ev(0);
    int rc = plx_render_fused_bwd(g, &a->rays, &a->opts, 1, a->up_scale, a->lam_cauchy, gb,
                                  nullptr, a->sums, a->scratch, a->scratch_bytes, stream);
    if (rc != PLX_OK) return rc;
    ev(1);
    if (a->tv_count > 0) {
        rc = plx_tv(g, nullptr, a->tv_start, a->tv_count, a->tv_fac[0], a->tv_fac[1],
                    a->tv_fac[2], a->tv_eps, a->tv_f_sigma, a->tv_f_sh, 0, 0, 0, 1, gb,
                    a->sums + 2, stream);
        if (rc != PLX_OK) return rc;
    }
    ev(2);
    if (a->update) {
        if (a->count && cudaMemsetAsync(a->count, 0, sizeof(int64_t), s) != cudaSuccess)
            return PLX_ECUDA;
        rc = plx_opt_step(g, a->v, gb, a->lr_sigma, a->lr_sh, a->beta, a->eps, a->rmsprop, 1,
                          a->sums, a->count, stream);
        if (rc != PLX_OK) return rc;
    }
    ev(3);
    return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA;
}
