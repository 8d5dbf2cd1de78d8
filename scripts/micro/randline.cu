// Microbenchmark: the random-line ceiling of B200 HBM3e — the speed of light for a hash
// probe that touches one random line per lookup (csrc/kv.cu).  Each thread issues R
// independent 16-byte loads at random 128-byte-aligned lines of an 8 GiB table (the C3
// table's size), for several L2 fetch-granularity limits.  Prints G lines/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o randline randline.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16; return x;
}

template <int R>
__global__ void __launch_bounds__(256) probe(const uint4 *tab, uint32_t nlines_mask, int64_t n, uint32_t seed,
                                             uint32_t *out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i * R >= n) return;
    uint32_t acc = 0;
    uint4 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t line = hash32((uint32_t)(i * R + r) ^ seed) & nlines_mask;
        v[r] = __ldg(tab + (size_t)line * 8);  // 8 x 16 B per 128-B line
    }
#pragma unroll
    for (int r = 0; r < R; ++r) acc ^= v[r].x ^ v[r].y ^ v[r].z ^ v[r].w;
    out[i] = acc;
}

int main() {
    const size_t bytes = (size_t)8 << 30;
    const uint32_t nlines = (uint32_t)(bytes / 128);
    const int64_t n = (int64_t)64 << 20;  // 64M random lines per launch
    uint4 *tab;
    uint32_t *out;
    if (cudaMalloc(&tab, bytes) != cudaSuccess || cudaMalloc(&out, n * 4) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMemset(tab, 1, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grans[] = {0, 32, 64, 128};
    for (int g : grans) {
        size_t prev = 0;
        if (g) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
        cudaDeviceGetLimit(&prev, cudaLimitMaxL2FetchGranularity);
        for (int R : {1, 2, 4}) {
            float best = 1e9f;
            for (int rep = 0; rep < 5; ++rep) {
                const int64_t threads = n / R;
                const int blocks = (int)((threads + 255) / 256);
                cudaEventRecord(e0);
                if (R == 1) probe<1><<<blocks, 256>>>(tab, nlines - 1, n, rep * 7919u, out);
                if (R == 2) probe<2><<<blocks, 256>>>(tab, nlines - 1, n, rep * 7919u, out);
                if (R == 4) probe<4><<<blocks, 256>>>(tab, nlines - 1, n, rep * 7919u, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("l2_fetch_granularity=%zu R=%d: %.3f ms, %.2f G lines/s (%.0f GB/s at 128 B/line)\n", prev, R, best,
                   n / (best * 1e-3) / 1e9, n * 128.0 / (best * 1e-3) / 1e9);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
