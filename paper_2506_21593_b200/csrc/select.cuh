// Block-level ranking helpers shared by the merge (index.cu) and the
// certified rescoring stage (tc_scan.cu).
#pragma once

#include "common.cuh"

namespace pr {

__device__ __forceinline__ void block_best(double &s, int64_t &r, double *red_s, int64_t *red_r) {
    // reduce (s, r) pairs to the one that ranks first; all threads get the result
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) {
        double os = __shfl_xor_sync(0xffffffffu, s, o);
        int64_t orr = __shfl_xor_sync(0xffffffffu, r, o);
        if (orr >= 0 && (r < 0 || ranks_before(os, orr, s, r))) { s = os; r = orr; }
    }
    if (lane == 0) { red_s[warp] = s; red_r[warp] = r; }
    __syncthreads();
    const int nw = blockDim.x >> 5;
    s = red_s[0];
    r = red_r[0];
    for (int i = 1; i < nw; ++i) {
        if (red_r[i] >= 0 && (r < 0 || ranks_before(red_s[i], red_r[i], s, r))) { s = red_s[i]; r = red_r[i]; }
    }
    __syncthreads();
}

__device__ __forceinline__ void finalize_hit(const float *__restrict__ X, int xstride, int d, const float *__restrict__ q,
                                             int64_t row, double raw, double *snap_out) {
    // self-snap: score > 1 - 1e-6 and the stored fp32 row equals the query
    // element-wise (np.array_equal, so -0.0 == 0.0)  (index.py:180-181)
    __shared__ int neq;
    double s = raw;
    if (raw > 1.0 - 1e-6) {
        if (threadIdx.x == 0) neq = 0;
        __syncthreads();
        const float *x = X + row * (int64_t)xstride;
        int mine = 0;
        for (int j = threadIdx.x; j < d; j += blockDim.x) mine |= !(x[j] == q[j]);
        if (mine) atomicOr(&neq, 1);
        __syncthreads();
        if (neq == 0) s = 1.0;
        __syncthreads();
    }
    *snap_out = fmax(-1.0, fmin(1.0, s));  // index.py:185
}

}  // namespace pr
