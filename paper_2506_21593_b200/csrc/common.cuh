// Shared helpers for libpentarag: error plumbing, launch checks, small math.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/pentarag.h"

namespace pr {

// thread-local last error for pr_last_error()
void set_error(const char *fmt, ...);
const char *last_error();

#define PR_FAIL(code, ...)              \
    do {                                \
        ::pr::set_error(__VA_ARGS__);   \
        return (code);                  \
    } while (0)

#define PR_CUDA(call)                                                                         \
    do {                                                                                      \
        cudaError_t _e = (call);                                                              \
        if (_e != cudaSuccess) {                                                              \
            ::pr::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
            return (_e == cudaErrorMemoryAllocation) ? PR_ERR_NOMEM : PR_ERR_CUDA;            \
        }                                                                                     \
    } while (0)

#define PR_LAUNCH_CHECK() PR_CUDA(cudaGetLastError())

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

template <typename T>
__host__ __device__ constexpr T ceil_div(T a, T b) {
    return (a + b - 1) / b;
}
template <typename T>
__host__ __device__ constexpr T round_up(T a, T b) {
    return ceil_div(a, b) * b;
}

int sm_count();

// every kernel launch of the library goes through PR_KERNEL so the host can
// report how many of OUR kernels ran in a timed region (bench gpu_launches)
void count_launch();

// bump allocator over the scratch block
struct Carve {
    char *base;
    size_t off = 0;
    template <typename T>
    T *take(size_t n) {
        off = round_up<size_t>(off, 256);
        T *p = reinterpret_cast<T *>(base + off);
        off += n * sizeof(T);
        return p;
    }
};


// Exact-score reduction in numpy's einsum order (see oracle/einsum_order.c and
// DESIGN.md §3).  x and q point at fp32 rows padded with zeros to a multiple
// of 8; d is the true dimension.  Lane 0 accumulates elements 0,2,4,6 of each
// block of 8 in the order 6,4,2,0; lane 1 takes 7,5,3,1.  fma == mul+add here
// because every fp32*fp32 product is exact in fp64.
__device__ __forceinline__ double einsum_dot_f32(const float *__restrict__ x, const float *__restrict__ q, int d) {
    double a0 = 0.0, a1 = 0.0;
    int j = 0;
    for (; j + 8 <= d; j += 8) {
        float4 xa = __ldg(reinterpret_cast<const float4 *>(x + j));
        float4 xb = __ldg(reinterpret_cast<const float4 *>(x + j + 4));
        float4 qa = __ldg(reinterpret_cast<const float4 *>(q + j));
        float4 qb = __ldg(reinterpret_cast<const float4 *>(q + j + 4));
        a0 = fma((double)xb.z, (double)qb.z, a0);
        a1 = fma((double)xb.w, (double)qb.w, a1);
        a0 = fma((double)xb.x, (double)qb.x, a0);
        a1 = fma((double)xb.y, (double)qb.y, a1);
        a0 = fma((double)xa.z, (double)qa.z, a0);
        a1 = fma((double)xa.w, (double)qa.w, a1);
        a0 = fma((double)xa.x, (double)qa.x, a0);
        a1 = fma((double)xa.y, (double)qa.y, a1);
    }
    for (; j < d; j += 2) {  // tail, two at a time, zero padded (the padding is stored zeros)
        a0 = fma((double)x[j], (double)q[j], a0);
        a1 = fma((double)x[j + 1], (double)q[j + 1], a1);
    }
    return 0.0 + (a0 + a1);
}

// One of einsum_dot_f32's two fp64 lanes (ch 0: elements 6,4,2,0 of every block of 8;
// ch 1: 7,5,3,1; tail two at a time) over operands in ANY memory space (shared staging):
// lane pair (ch 0, ch 1) + `0.0 + (a0 + a1)` reproduces einsum_dot_f32 bit for bit.
__device__ __forceinline__ double einsum_lane(const float *x, const float *q, int d, int ch) {
    double a = 0.0;
    int j = 0;
#pragma unroll 4
    for (; j + 8 <= d; j += 8) {
        const float4 xa = *reinterpret_cast<const float4 *>(x + j);
        const float4 xb = *reinterpret_cast<const float4 *>(x + j + 4);
        const float4 qa = *reinterpret_cast<const float4 *>(q + j);
        const float4 qb = *reinterpret_cast<const float4 *>(q + j + 4);
        a = fma((double)(ch ? xb.w : xb.z), (double)(ch ? qb.w : qb.z), a);
        a = fma((double)(ch ? xb.y : xb.x), (double)(ch ? qb.y : qb.x), a);
        a = fma((double)(ch ? xa.w : xa.z), (double)(ch ? qa.w : qa.z), a);
        a = fma((double)(ch ? xa.y : xa.x), (double)(ch ? qa.y : qa.x), a);
    }
    for (; j < d; j += 2) a = fma((double)x[j + ch], (double)q[j + ch], a);
    return a;
}

// Exact einsum-order score of one stored row by a whole warp: the row is staged in shared
// memory with coalesced 16-byte loads (one DRAM round trip instead of a per-thread stream of
// 256 dependent-latency loads), then lanes 0/1 run the two fp64 chains.  Returns the score
// in lane 0.  xs: this warp's [dp8] staging buffer; qs: the query (shared or global).
__device__ __forceinline__ double warp_einsum_dot(const float *__restrict__ x, float *xs, const float *qs, int dp8,
                                                  int d) {
    const int lane = threadIdx.x & 31;
    for (int j = lane * 4; j < dp8; j += 128)
        *reinterpret_cast<float4 *>(xs + j) = __ldg(reinterpret_cast<const float4 *>(x + j));
    __syncwarp();
    const double acc = lane < 2 ? einsum_lane(xs, qs, d, lane) : 0.0;
    const double other = __shfl_xor_sync(0xffffffffu, acc, 1);
    __syncwarp();
    return 0.0 + (acc + other);
}

// (score desc, row asc) total order used everywhere results are ranked
// (index.py:176 lexsort((arange(n), -scores))).
__device__ __forceinline__ bool ranks_before(double sa, int64_t ra, double sb, int64_t rb) {
    return sa > sb || (sa == sb && ra < rb);
}

}  // namespace pr
