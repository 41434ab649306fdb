// Probe: scattered row read-modify-write of the optimiser (grad, table,
// RMSProp v; 28 floats per row) with (A) three arrays at a 128-B pitch vs
// (B) one interleaved 384-B row {table, grad, v}.  Touched list: a dense run
// (the TV cells) + random rows, sorted -- the shape of the early-training
// touched set.  nvcc -O3 -arch=sm_100a rmw_layout.cu -o /tmp/rmw && /tmp/rmw
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int PITCH, int TOFF, int GOFF, int VOFF>
__global__ void __launch_bounds__(256, 4) rmw(float *base_t, float *base_g, float *base_v,
                                              const int *ids, long n) {
    const int lane = threadIdx.x & 31, quad = lane % 7, sub = lane / 7;
    const long ng = (n + 3) / 4;
    const long nw = (long)gridDim.x * 8, w = (long)blockIdx.x * 8 + (threadIdx.x >> 5);
    for (long g0 = w; g0 < ng; g0 += 2 * nw) {
        float4 t[2], g[2], v[2];
        int r[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const long gi = g0 + u * nw, j = gi * 4 + sub;
            r[u] = (lane < 28 && gi < ng && j < n) ? ids[j] : -1;
            if (r[u] >= 0) {
                t[u] = reinterpret_cast<float4 *>(base_t + (long)r[u] * PITCH + TOFF)[quad];
                g[u] = reinterpret_cast<float4 *>(base_g + (long)r[u] * PITCH + GOFF)[quad];
                v[u] = reinterpret_cast<float4 *>(base_v + (long)r[u] * PITCH + VOFF)[quad];
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (r[u] < 0) continue;
            v[u].x = 0.9f * v[u].x + g[u].x * g[u].x; t[u].x -= 0.1f * g[u].x * rsqrtf(v[u].x + 1e-8f);
            v[u].y = 0.9f * v[u].y + g[u].y * g[u].y; t[u].y -= 0.1f * g[u].y * rsqrtf(v[u].y + 1e-8f);
            v[u].z = 0.9f * v[u].z + g[u].z * g[u].z; t[u].z -= 0.1f * g[u].z * rsqrtf(v[u].z + 1e-8f);
            v[u].w = 0.9f * v[u].w + g[u].w * g[u].w; t[u].w -= 0.1f * g[u].w * rsqrtf(v[u].w + 1e-8f);
            reinterpret_cast<float4 *>(base_t + (long)r[u] * PITCH + TOFF)[quad] = t[u];
            reinterpret_cast<float4 *>(base_v + (long)r[u] * PITCH + VOFF)[quad] = v[u];
            reinterpret_cast<float4 *>(base_g + (long)r[u] * PITCH + GOFF)[quad] = make_float4(0, 0, 0, 0);
        }
    }
}

int main() {
    const long N = 256L * 256 * 256;
    std::mt19937_64 rng(1);
    std::vector<char> m(N, 0);
    const long run0 = 5000000, runlen = 167772;
    for (long c = run0; c < run0 + runlen; ++c) {   // TV cells + their +1 neighbours
        m[c] = 1; m[c + 1] = 1; m[c + 256] = 1; m[c + 65536] = 1;
    }
    std::uniform_int_distribution<long> U(0, N - 1);
    for (int i = 0; i < 700000; ++i) m[U(rng)] = 1;
    std::vector<int> ids;
    for (long i = 0; i < N; ++i) if (m[i]) ids.push_back((int)i);
    const long n = ids.size();
    printf("touched rows %ld (%.1f%%)\n", n, 100.0 * n / N);
    int *d_ids; cudaMalloc(&d_ids, n * 4);
    cudaMemcpy(d_ids, ids.data(), n * 4, cudaMemcpyHostToDevice);
    float *a, *b, *c, *il;
    cudaMalloc(&a, N * 128); cudaMalloc(&b, N * 128); cudaMalloc(&c, N * 128);
    cudaMalloc(&il, N * 384);
    cudaMemset(a, 0, N * 128); cudaMemset(b, 0, N * 128); cudaMemset(c, 0, N * 128);
    cudaMemset(il, 0, N * 384);
    char *flush; cudaMalloc(&flush, 512L << 20);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
        float best = 1e9, sum = 0;
        for (int it = 0; it < 12; ++it) {
            cudaMemsetAsync(flush, it, 512L << 20);
            cudaEventRecord(e0);
            if (mode == 0) rmw<32, 0, 0, 0><<<sms * 4, 256>>>(a, b, c, d_ids, n);
            else if (mode == 1) rmw<96, 0, 32, 64><<<sms * 4, 256>>>(il, il, il, d_ids, n);
            else rmw<64, 0, 32, 0><<<sms * 4, 256>>>(il, il, c, d_ids, n);   // {t,g} + v
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 2) { best = std::min(best, ms); sum += ms; }
        }
        const double bytes = n * (3 * 128.0 + 3 * 112.0);
        printf("%s: best %.1f us  mean %.1f us  (%.2f TB/s on 720 B/row)\n",
               mode == 0 ? "A separate 128-B pitch" : mode == 1 ? "B interleaved 384-B" : "C {t,g} 256-B + v",
               best * 1e3, sum / 10 * 1e3, bytes / (best * 1e-3) / 1e12);
    }
    return 0;
}
