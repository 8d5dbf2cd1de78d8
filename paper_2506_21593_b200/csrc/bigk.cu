// Large-k search (k > 64): every exact score, then a stable segmented sort.
// Reference: index.py:173-176 — einsum scores + lexsort((arange(n), -scores)).
// A stable descending sort keeps equal scores in ascending row order, which is
// exactly lexsort's secondary key.  Used only when k exceeds the register /
// shared-memory top-k paths; queries are processed in chunks bounded to
// ~256 MB of scratch.
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>

#include "common.cuh"
#include "select.cuh"
#include "tc_scan.cuh"

namespace pr {

__global__ void bigk_pad_kernel(const float *__restrict__ q, int64_t nq, int d, int dp8, float *__restrict__ out) {
    int64_t total = nq * (int64_t)dp8;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / dp8;
        int j = (int)(t - i * dp8);
        out[t] = j < d ? q[i * d + j] : 0.0f;
    }
}

__global__ void bigk_scores_kernel(const float *__restrict__ x32, int64_t n, int dp8, int d, const float *__restrict__ qp,
                                   int64_t nqc, double *__restrict__ keys, int64_t *__restrict__ vals,
                                   int64_t *__restrict__ offs, const int64_t *__restrict__ lim) {
    int64_t total = nqc * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t qi = t / n, r = t - qi * n;
        // rows past the query's limit sort last and are never taken
        keys[t] = (lim && r >= lim[qi]) ? -INFINITY : einsum_dot_f32(x32 + r * dp8, qp + qi * dp8, d);
        vals[t] = r;
        if (r == 0) offs[qi] = t;
        if (t == total - 1) offs[nqc] = total;
    }
}

__global__ void bigk_finalize_kernel(const double *__restrict__ keys, const int64_t *__restrict__ vals, int64_t n,
                                     int64_t nqc, int64_t q0, int k, const float *__restrict__ x32, int dp8, int d,
                                     const float *__restrict__ qp, int64_t *rows, double *raw, double *rep,
                                     int32_t *count, const int64_t *__restrict__ lim) {
    const int64_t take_all = (int64_t)k < n ? (int64_t)k : n;
    for (int64_t qi = blockIdx.x; qi < nqc; qi += gridDim.x) {
        const int64_t q = q0 + qi;
        const int64_t take = lim ? min(take_all, max((int64_t)0, lim[qi])) : take_all;
        for (int64_t j = 0; j < k; ++j) {
            const int64_t o = q * k + j;
            if (j >= take) {
                if (threadIdx.x == 0) {
                    rows[o] = -1;
                    if (raw) raw[o] = 0.0;
                    if (rep) rep[o] = 0.0;
                }
                continue;
            }
            const double s = keys[qi * n + j];
            const int64_t r = vals[qi * n + j];
            double rp;
            finalize_hit(x32, dp8, d, qp + qi * dp8, r, s, &rp);
            if (threadIdx.x == 0) {
                rows[o] = r;
                if (raw) raw[o] = s;
                if (rep) rep[o] = rp;
            }
        }
        if (threadIdx.x == 0) count[q] = (int32_t)take;
    }
}

int big_k_search(const float *x32, int64_t n, int dp8, int d, const float *q, int64_t nq, int k,
                 const int64_t *row_limit, int64_t *rows, double *raw, double *rep, int32_t *count, cudaStream_t st) {
    const size_t budget = (size_t)256 << 20;
    int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(nq, (int64_t)(budget / ((size_t)n * 32 + 1))));
    float *qp = nullptr;
    double *k_in = nullptr, *k_out = nullptr;
    int64_t *v_in = nullptr, *v_out = nullptr, *offs = nullptr;
    void *temp = nullptr;
    size_t temp_bytes = 0;
    PR_CUDA(cudaMallocAsync(&qp, (size_t)chunk * dp8 * sizeof(float), st));
    PR_CUDA(cudaMallocAsync(&k_in, (size_t)chunk * n * sizeof(double), st));
    PR_CUDA(cudaMallocAsync(&k_out, (size_t)chunk * n * sizeof(double), st));
    PR_CUDA(cudaMallocAsync(&v_in, (size_t)chunk * n * sizeof(int64_t), st));
    PR_CUDA(cudaMallocAsync(&v_out, (size_t)chunk * n * sizeof(int64_t), st));
    PR_CUDA(cudaMallocAsync(&offs, (size_t)(chunk + 1) * sizeof(int64_t), st));
    PR_CUDA(cub::DeviceSegmentedSort::StableSortPairsDescending(nullptr, temp_bytes, k_in, k_out, v_in, v_out,
                                                                 chunk * n, (int)chunk, offs, offs + 1, st));
    PR_CUDA(cudaMallocAsync(&temp, temp_bytes, st));
    for (int64_t q0 = 0; q0 < nq; q0 += chunk) {
        const int64_t nqc = std::min(chunk, nq - q0);
        int g = (int)std::min<int64_t>(ceil_div<int64_t>(nqc * dp8, 256), 4096);
        ::pr::count_launch();
        bigk_pad_kernel<<<g, 256, 0, st>>>(q + q0 * d, nqc, d, dp8, qp);
        g = (int)std::min<int64_t>(ceil_div<int64_t>(nqc * n, 256), (int64_t)sm_count() * 32);
        ::pr::count_launch();
        const int64_t *lim = row_limit ? row_limit + q0 : nullptr;
        bigk_scores_kernel<<<g, 256, 0, st>>>(x32, n, dp8, d, qp, nqc, k_in, v_in, offs, lim);
        PR_LAUNCH_CHECK();
        size_t tb = temp_bytes;
        PR_CUDA(cub::DeviceSegmentedSort::StableSortPairsDescending(temp, tb, k_in, k_out, v_in, v_out, nqc * n,
                                                                     (int)nqc, offs, offs + 1, st));
        g = (int)std::min<int64_t>(nqc, (int64_t)sm_count() * 8);
        ::pr::count_launch();
        bigk_finalize_kernel<<<g, 128, 0, st>>>(k_out, v_out, n, nqc, q0, k, x32, dp8, d, qp, rows, raw, rep, count,
                                                lim);
        PR_LAUNCH_CHECK();
    }
    cudaFreeAsync(qp, st);
    cudaFreeAsync(k_in, st);
    cudaFreeAsync(k_out, st);
    cudaFreeAsync(v_in, st);
    cudaFreeAsync(v_out, st);
    cudaFreeAsync(offs, st);
    cudaFreeAsync(temp, st);
    return PR_OK;
}

}  // namespace pr
