// Microbenchmark: energy / rate of the int8 tcgen05 MMA stream alone under the 1 kW cap,
// for the operand placements the scan could use (no loads, no epilogue; random operands).
//   var 0: A in smem, M=256 (2-CTA) x N=256 — the scan's current MMA
//   var 1: A in TMEM, M=256 x N=128 (A tile 256 TMEM columns + 2 x 128 accumulator columns)
//   var 2: A in smem, M=256 x N=128 (isolates the N change)
// Each variant runs back to back for SECONDS while nvidia-smi samples clocks/power
// (run by scripts/micro/mmapower.sh).  Prints int8 TOP/s per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mmapower mmapower.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <thread>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
template <int N>
__host__ __device__ constexpr uint32_t idesc() {  // D = S32, A,B = s8 K-major, M = 256
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
template <int N>
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc<N>()), "r"(acc)
                 : "memory");
}
template <int N>
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a_tmem), "l"(b), "r"(idesc<N>()), "r"(acc)
                 : "memory");
}

constexpr int THREADS = 128;
constexpr int KSTEPS = 32;  // K = 1024 int8 = 32 MMAs of K = 32

template <int VAR>
__global__ void __launch_bounds__(THREADS, 1) mma_only(int iters, uint32_t seed, int *sink) {
    constexpr int N = VAR == 0 ? 256 : 128;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *sA = smem;                  // 8 K-blocks x [128 rows x 128 B] = 128 KB
    uint8_t *sB = smem + 128 * 1024;     // 2 K-blocks x [N/2 rows x 128 B]
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    // random operands (power is data dependent)
    uint32_t x = seed ^ (blockIdx.x * 0x9E3779B9u) ^ (threadIdx.x * 0x85EBCA6Bu);
    const int fill = 128 * 1024 + 2 * (N / 2) * 128;
    for (int i = threadIdx.x * 4; i < fill; i += THREADS * 4) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        *reinterpret_cast<uint32_t *>(smem + i) = x;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (VAR == 1) {  // A tile in TMEM columns [256, 512): random words, each warp its 32 lanes
        for (int c = 0; c < 256; c += 8) {
            uint32_t v[8];
            for (int j = 0; j < 8; ++j) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; v[j] = x; }
            const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + 256 + c;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr),
                         "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                         : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (rank == 0 && threadIdx.x == 0) {
        constexpr int BB = (N / 2) * 128;
        for (int it = 0; it < iters; ++it) {
            for (int acc = 0; acc < 2; ++acc) {
                const uint32_t d = tmem + acc * N;
                for (int ks = 0; ks < KSTEPS; ++ks) {
                    const int kb = ks >> 2, k = ks & 3;
                    const uint64_t bd = sw128_desc(smem_u32(sB + (kb & 1) * BB)) + 2 * k;
                    if (VAR == 1)
                        mma_ts<N>(d, tmem + 256 + 8 * ks, bd, ks != 0);
                    else
                        mma_ss<N>(d, sw128_desc(smem_u32(sA + kb * 16384)) + 2 * k, bd, ks != 0);
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    }
    if (threadIdx.x == 0) {
        asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}"
                     ::"r"(smem_u32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    if (threadIdx.x == 0 && sink) sink[blockIdx.x] = (int)tmem;
}

template <int VAR>
static double run(double seconds, int sms) {
    constexpr int N = VAR == 0 ? 256 : 128;
    const size_t smem = 1024 + 128 * 1024 + 2 * (N / 2) * 128;
    cudaFuncSetAttribute(mma_only<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, mma_only<VAR>, iters, 1u, (int *)nullptr);  // warm
    cudaDeviceSynchronize();
    int launches = 0;
    auto t0 = std::chrono::steady_clock::now();
    cudaEventRecord(e0);
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < seconds) {
        for (int r = 0; r < 4; ++r) cudaLaunchKernelEx(&cfg, mma_only<VAR>, iters, (uint32_t)launches++, (int *)nullptr);
        cudaEventSynchronize(e0);
        // keep at most a few launches queued so wall time tracks device time
        cudaDeviceSynchronize();
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * 256.0 * N * 32.0 * KSTEPS * 2.0 * iters * launches * (sms / 2);
    printf("var %d (N=%d, A %s): %d launches, %.1f ms, %.1f TOP/s  [%s]\n", VAR, N, VAR == 1 ? "TMEM" : "smem",
           launches, ms, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
    return ops / (ms * 1e-3) / 1e12;
}

int main(int argc, char **argv) {
    const double secs = argc > 1 ? atof(argv[1]) : 4.0;
    const int sms = 148;
    for (int rep = 0; rep < 2; ++rep) {
        printf("mark var0 start %lld\n", (long long)std::chrono::duration_cast<std::chrono::milliseconds>(
                                              std::chrono::system_clock::now().time_since_epoch()).count());
        run<0>(secs, sms);
        printf("mark var1 start %lld\n", (long long)std::chrono::duration_cast<std::chrono::milliseconds>(
                                              std::chrono::system_clock::now().time_since_epoch()).count());
        run<1>(secs, sms);
        printf("mark var2 start %lld\n", (long long)std::chrono::duration_cast<std::chrono::milliseconds>(
                                              std::chrono::system_clock::now().time_since_epoch()).count());
        run<2>(secs, sms);
        printf("mark end %lld\n", (long long)std::chrono::duration_cast<std::chrono::milliseconds>(
                                      std::chrono::system_clock::now().time_since_epoch()).count());
    }
    return 0;
}
