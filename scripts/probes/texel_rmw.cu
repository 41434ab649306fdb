// Probe: the MSI background update's access shape -- 3M touched texels of
// 32 B (4 x f64) read-modify-written in three arrays (table, RMSProp v,
// grad) -- versus the arrays' footprint (0.25 .. 4.3 GB each) and the order
// of the touched list (random vs sorted).  Separates DRAM sector cost from
// address-translation cost.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a texel_rmw.cu -o /tmp/trmw && /tmp/trmw
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) rmw(double4 *__restrict__ t, double4 *__restrict__ v,
                                           double4 *__restrict__ g, const int *__restrict__ ids,
                                           long n) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long)gridDim.x * blockDim.x) {
        const int r = ids[i];
        double4 a = t[r], b = v[r], c = g[r];
        b.x = 0.9 * b.x + 0.1 * c.x * c.x; a.x -= 0.1 * c.x / (sqrt(b.x) + 1e-8);
        b.y = 0.9 * b.y + 0.1 * c.y * c.y; a.y -= 0.1 * c.y / (sqrt(b.y) + 1e-8);
        b.z = 0.9 * b.z + 0.1 * c.z * c.z; a.z -= 0.1 * c.z / (sqrt(b.z) + 1e-8);
        b.w = 0.9 * b.w + 0.1 * c.w * c.w; a.w -= 0.1 * c.w / (sqrt(b.w) + 1e-8);
        t[r] = a; v[r] = b; g[r] = make_double4(0, 0, 0, 0);
    }
}

// same shape, one f64 per thread (the previous kernel's (texel, channel) map)
__global__ void __launch_bounds__(256) rmw_ch(double *t, double *v, double *g,
                                              const int *ids, long n) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < 4 * n;
         i += (long)gridDim.x * blockDim.x) {
        const long e = 4L * ids[i >> 2] + (i & 3);
        const double c = g[e];
        g[e] = 0.0;
        const double b = 0.9 * v[e] + 0.1 * c * c;
        v[e] = b;
        t[e] -= 0.1 * c / (sqrt(b) + 1e-8);
    }
}

int main() {
    const long n_touch = 3000000;
    const long sizes[] = {8L << 20, 32L << 20, 134217728L};
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (long ntex : sizes) {
        double4 *t, *v, *g;
        int *ids;
        cudaMalloc(&t, ntex * 32); cudaMalloc(&v, ntex * 32); cudaMalloc(&g, ntex * 32);
        cudaMemset(t, 0, ntex * 32); cudaMemset(v, 0, ntex * 32); cudaMemset(g, 0, ntex * 32);
        cudaMalloc(&ids, n_touch * 4);
        std::mt19937_64 rng(1);
        std::vector<int> h(n_touch);
        for (auto &x : h) x = (int)(rng() % ntex);
        for (int sorted = 0; sorted < 2; ++sorted) {
            if (sorted) std::sort(h.begin(), h.end());
            cudaMemcpy(ids, h.data(), n_touch * 4, cudaMemcpyHostToDevice);
            for (int k = 0; k < 2; ++k) {
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0); cudaEventCreate(&e1);
                float best = 1e9;
                for (int rep = 0; rep < 5; ++rep) {
                    cudaEventRecord(e0);
                    if (k == 0) rmw<<<nsm * 8, 256>>>(t, v, g, ids, n_touch);
                    else rmw_ch<<<nsm * 8, 256>>>((double *)t, (double *)v, (double *)g, ids, n_touch);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    best = std::min(best, ms);
                }
                printf("footprint %6.2f GB/array  %-6s %-13s %8.1f us  %7.1f GB/s (6 x 32 B/texel)\n",
                       ntex * 32 / 1e9, sorted ? "sorted" : "random",
                       k == 0 ? "thread/texel" : "thread/f64", best * 1e3,
                       6.0 * 32 * n_touch / (best * 1e-3) / 1e9);
            }
        }
        cudaFree(t); cudaFree(v); cudaFree(g); cudaFree(ids);
    }
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
}
