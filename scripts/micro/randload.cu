// Microbenchmark: random 32-byte reads from a large table with different load flavours,
// to see how many DRAM bytes each random sector costs (ncu dram__bytes_read.sum).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16; return x;
}

template <int V>
__global__ void k(const uint64_t *tab, int64_t nsec, int64_t n, uint64_t *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t s = (int64_t)(((uint64_t)hash32((uint32_t)i) * 2654435761ull + hash32((uint32_t)(i >> 7))) % (uint64_t)nsec);
    const uint64_t *p = tab + 4 * s;
    uint64_t a, b, c, d;
    if (V == 0) asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    if (V == 1) {
        asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
        asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(c), "=l"(d) : "l"(p + 2));
    }
    if (V == 2) asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    if (V == 3) {
        asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
        asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(c), "=l"(d) : "l"(p + 2));
    }
    if (V == 4) asm volatile("ld.global.cs.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    if (V == 5) asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
    out[i] = a ^ b ^ c ^ d;
}

int main() {
    const int64_t bytes = (int64_t)4 << 30, nsec = bytes / 32, n = 4 << 20;
    uint64_t *tab, *out;
    cudaMalloc(&tab, bytes);
    cudaMemset(tab, 1, bytes);
    cudaMalloc(&out, n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep)
        for (int v = 0; v < 6; ++v) {
            cudaEventRecord(e0);
            switch (v) {
                case 0: k<0><<<n / 128, 128>>>(tab, nsec, n, out); break;
                case 1: k<1><<<n / 128, 128>>>(tab, nsec, n, out); break;
                case 2: k<2><<<n / 128, 128>>>(tab, nsec, n, out); break;
                case 3: k<3><<<n / 128, 128>>>(tab, nsec, n, out); break;
                case 4: k<4><<<n / 128, 128>>>(tab, nsec, n, out); break;
                case 5: k<5><<<n / 128, 128>>>(tab, nsec, n, out); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("variant %d: %.1f us, %.2f G random sectors/s\n", v, ms * 1e3, n / (ms * 1e-3) / 1e9);
        }
    return 0;
}
