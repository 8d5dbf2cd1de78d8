// FlatIndex store + search orchestration (reference: index.py:73-189).
//
// Data layout in HBM (per index handle):
//   x32  fp32 [cap, dp8]     exact copy, rows zero-padded to a multiple of 8
//                            (einsum-order tail reads the padding as zeros)
//   x16  fp16 [cap256, dp64] tensor-core scan copy, zero-padded to 64 columns
//                            (one 128-byte swizzle atom per K block)
// Row i == the i-th inserted id, so row order is the tie-break order.
#include <chrono>
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <atomic>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "select.cuh"
#include "tc_scan.cuh"

namespace pr {

// ---------------------------------------------------------------------------
// errors
static thread_local char g_err[1024] = "";
void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
const char *last_error() { return g_err; }

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int sm_count() {
    static int cached = -1;
    if (cached < 0) {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached = v > 0 ? v : 148;
    }
    return cached;
}

// ---------------------------------------------------------------------------
// store kernels

// fp32 [n, d] -> x32 rows (stride dp8) and x16 rows (stride dp64), zero padded.
// rows == nullptr: destination row = row0 + i; else destination row = rows[i].
__global__ void write_rows_kernel(const float *__restrict__ src, int64_t n, int d, const int64_t *__restrict__ rows,
                                  int64_t row0, float *__restrict__ x32, int dp8, __half *__restrict__ x16,
                                  int dp64) {
    int64_t total = n * (int64_t)dp64;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / dp64;
        int j = (int)(t - i * dp64);
        float v = (j < d) ? src[i * d + j] : 0.0f;
        int64_t r = rows ? rows[i] : row0 + i;
        if (j < dp8) x32[r * dp8 + j] = v;
        x16[r * dp64 + j] = __float2half_rn(v);
    }
}

__global__ void gather_rows_kernel(const float *__restrict__ sx32, const __half *__restrict__ sx16,
                                   const int64_t *__restrict__ src_rows, int64_t n, int dp8, int dp64,
                                   int64_t row0, float *__restrict__ x32, __half *__restrict__ x16) {
    int64_t total = n * (int64_t)dp64;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / dp64;
        int j = (int)(t - i * dp64);
        int64_t s = src_rows[i];
        if (j < dp8) x32[(row0 + i) * dp8 + j] = sx32[s * dp8 + j];
        x16[(row0 + i) * dp64 + j] = sx16[s * dp64 + j];
    }
}

// rows of a row-sharded store: the rows this shard holds (global row - row_offset in
// [0, count)) are copied, every other row is zero, so a SUM all-reduce over the shards'
// int32 bit patterns assembles the exact fp32 rows
__global__ void gather_owned_kernel(const float *__restrict__ x32, int dp8, int d, int64_t count,
                                    const int64_t *__restrict__ rows, int64_t n, int64_t row_offset,
                                    float *__restrict__ out) {
    const int64_t total = n * (int64_t)d;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / d;
        const int j = (int)(t - i * d);
        const int64_t r = rows[i] - row_offset;
        out[t] = (r >= 0 && r < count) ? x32[r * dp8 + j] : 0.f;
    }
}

__global__ void read_rows_kernel(const float *__restrict__ x32, int dp8, int d, int64_t row0, int64_t n,
                                 float *__restrict__ out) {
    int64_t total = n * (int64_t)d;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / d;
        int j = (int)(t - i * d);
        out[t] = x32[(row0 + i) * dp8 + j];
    }
}

// unit-norm + finiteness check, one warp per vector (index.py:63-69)
__global__ void check_unit_kernel(const float *__restrict__ v, int64_t n, int d, double tol, uint8_t *__restrict__ bad) {
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    int lane = threadIdx.x & 31;
    if (w >= n) return;
    const float *x = v + w * d;
    double ss = 0.0;
    int nonfinite = 0;
    for (int j = lane; j < d; j += 32) {
        float f = x[j];
        if (!isfinite(f)) nonfinite = 1;
        ss = fma((double)f, (double)f, ss);
    }
    for (int o = 16; o; o >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
        nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, o);
    }
    if (lane == 0) bad[w] = (nonfinite || fabs(sqrt(ss) - 1.0) > tol) ? 1 : 0;
}

// queries fp32 [nq, d] -> [nq, dp8] fp32 (zero padded)
__global__ void pad_queries_kernel(const float *__restrict__ q, int64_t nq, int d, int dp8, float *__restrict__ out) {
    int64_t total = nq * (int64_t)dp8;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / dp8;
        int j = (int)(t - i * dp8);
        out[t] = j < d ? q[i * d + j] : 0.0f;
    }
}

// listed queries: row i of the output = q[list[i]] for i < *nlist; rows past the live
// count repeat the first listed query (valid input for every scan path; never reported)
__global__ void gather_pad_queries_kernel(const float *__restrict__ q, const int32_t *__restrict__ list,
                                          const int32_t *__restrict__ nlist, int64_t nq_max, int d, int dp8,
                                          float *__restrict__ out) {
    const int64_t total = nq_max * (int64_t)dp8;
    const int32_t live = *nlist;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / dp8;
        const int c = (int)(t % dp8);
        const int64_t src = live > 0 ? list[i < live ? i : 0] : -1;
        out[t] = (src >= 0 && c < d) ? q[src * d + c] : 0.f;
    }
}

static int grid_for(int64_t total, int block = 256) {
    int64_t g = (total + block - 1) / block;
    int64_t cap = (int64_t)sm_count() * 16;
    return (int)std::max<int64_t>(1, std::min(g, cap));
}

// ---------------------------------------------------------------------------
// exact fp64 scan (numpy einsum order) with per-(query, split) top-K lists.
//
// One CTA = 256 threads = 256 consecutive rows per step, QT queries held in
// shared memory as fp64.  Each thread reduces its row against all QT queries
// (2*QT independent fp64 accumulation chains), scores go to shared memory,
// then warp w keeps the top-K of queries w, w+8, ... in shared memory with a
// warp-parallel sorted insert.  Persistent: CTAs loop over (query tile,
// row split) work items; the number of selected queries may live on the
// device (fallback lists), so no host sync is needed.
struct ScanArgs {
    const float *X;
    int64_t n;
    int xstride;  // dp8
    int d;
    const float *Q;  // padded fp32 queries [*, xstride]
    const int32_t *qsel;
    const int32_t *nsel_dev;
    int32_t nsel_host;
    int nsplit;
    int64_t rows_per_split;
    int K;
    double *part_s;
    int64_t *part_r;
    int32_t *part_c;
    const int64_t *row_limit;  // per original query: rows >= limit are invisible (nullable)
};

constexpr int SCAN_THREADS = 256;

template <int QT>
__global__ void __launch_bounds__(SCAN_THREADS) exact_scan_kernel(ScanArgs p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int qs_stride = p.xstride;
    double *qs = reinterpret_cast<double *>(smem);         // [QT][xstride]
    double *sc = qs + QT * qs_stride;                       // [QT][256]
    double *tks = sc + QT * SCAN_THREADS;                   // [QT][K]
    int64_t *tkr = reinterpret_cast<int64_t *>(tks + QT * p.K);  // [QT][K]
    int *tkc = reinterpret_cast<int *>(tkr + QT * p.K);     // [QT]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nsel = p.nsel_dev ? *p.nsel_dev : p.nsel_host;
    const int qtiles = (nsel + QT - 1) / QT;
    const int64_t work = (int64_t)qtiles * p.nsplit;
    const int d = p.d, K = p.K;
    __shared__ int64_t qlim[QT];
    __shared__ int64_t tile_lim;

    for (int64_t w = blockIdx.x; w < work; w += gridDim.x) {
        const int qt = (int)(w / p.nsplit);
        const int split = (int)(w - (int64_t)qt * p.nsplit);
        const int64_t row_begin = (int64_t)split * p.rows_per_split;
        __syncthreads();
        if (tid == 0) {
            int64_t mx = 0;
            for (int qi = 0; qi < QT; ++qi) {
                const int sel = qt * QT + qi;
                int64_t lim = 0;
                if (sel < nsel) {
                    const int qidx = p.qsel ? p.qsel[sel] : sel;
                    lim = p.row_limit ? min(p.n, p.row_limit[qidx]) : p.n;
                }
                qlim[qi] = lim;
                mx = max(mx, lim);
            }
            tile_lim = mx;
        }
        __syncthreads();
        // rows no query of this tile can see are not scanned at all
        const int64_t row_end = min(tile_lim, row_begin + p.rows_per_split);
        for (int i = tid; i < QT * qs_stride; i += SCAN_THREADS) {
            int qi = i / qs_stride, j = i - qi * qs_stride;
            int sel = qt * QT + qi;
            double v = 0.0;
            if (sel < nsel) {
                int qidx = p.qsel ? p.qsel[sel] : sel;
                v = (double)p.Q[(int64_t)qidx * qs_stride + j];
            }
            qs[i] = v;
        }
        if (tid < QT) tkc[tid] = 0;
        __syncthreads();

        for (int64_t r0 = row_begin; r0 < row_end; r0 += SCAN_THREADS) {
            const int64_t r = r0 + tid;
            double acc0[QT], acc1[QT];
#pragma unroll
            for (int qi = 0; qi < QT; ++qi) acc0[qi] = acc1[qi] = 0.0;
            if (r < row_end) {
                const float *x = p.X + r * (int64_t)p.xstride;
                int j = 0;
                for (; j + 8 <= d; j += 8) {
                    float4 xa = __ldg(reinterpret_cast<const float4 *>(x + j));
                    float4 xb = __ldg(reinterpret_cast<const float4 *>(x + j + 4));
                    const double x0 = xa.x, x1 = xa.y, x2 = xa.z, x3 = xa.w;
                    const double x4 = xb.x, x5 = xb.y, x6 = xb.z, x7 = xb.w;
#pragma unroll
                    for (int qi = 0; qi < QT; ++qi) {
                        const double2 *qq = reinterpret_cast<const double2 *>(qs + qi * qs_stride + j);
                        const double2 q67 = qq[3], q45 = qq[2], q23 = qq[1], q01 = qq[0];
                        acc0[qi] = fma(x6, q67.x, acc0[qi]);
                        acc1[qi] = fma(x7, q67.y, acc1[qi]);
                        acc0[qi] = fma(x4, q45.x, acc0[qi]);
                        acc1[qi] = fma(x5, q45.y, acc1[qi]);
                        acc0[qi] = fma(x2, q23.x, acc0[qi]);
                        acc1[qi] = fma(x3, q23.y, acc1[qi]);
                        acc0[qi] = fma(x0, q01.x, acc0[qi]);
                        acc1[qi] = fma(x1, q01.y, acc1[qi]);
                    }
                }
                for (; j < d; j += 2) {
                    const double x0 = x[j], x1 = x[j + 1];
#pragma unroll
                    for (int qi = 0; qi < QT; ++qi) {
                        acc0[qi] = fma(x0, qs[qi * qs_stride + j], acc0[qi]);
                        acc1[qi] = fma(x1, qs[qi * qs_stride + j + 1], acc1[qi]);
                    }
                }
            }
#pragma unroll
            for (int qi = 0; qi < QT; ++qi)
                sc[qi * SCAN_THREADS + tid] = (r < row_end) ? 0.0 + (acc0[qi] + acc1[qi]) : -INFINITY;
            __syncthreads();

            for (int qi = warp; qi < QT; qi += SCAN_THREADS / 32) {
                if (qt * QT + qi >= nsel) break;
                double *ls = tks + qi * K;
                int64_t *lr = tkr + qi * K;
                int cnt = tkc[qi];
                for (int c = 0; c < SCAN_THREADS / 32; ++c) {
                    const int64_t rr = r0 + c * 32 + lane;
                    const double s = sc[qi * SCAN_THREADS + c * 32 + lane];
                    const bool valid = rr < row_end && rr < qlim[qi];
                    double thr = (cnt == K) ? ls[K - 1] : -INFINITY;
                    unsigned m = __ballot_sync(0xffffffffu, valid && (cnt < K || s > thr));
                    while (m) {
                        const int src = __ffs(m) - 1;
                        m &= m - 1;
                        const double sv = __shfl_sync(0xffffffffu, s, src);
                        const int64_t rv = r0 + c * 32 + src;
                        if (cnt == K && !(sv > ls[K - 1])) continue;
                        // rows arrive in ascending order: equal scores already in the
                        // list rank first, so the insert position counts entries >= sv
                        int pos = 0;
                        for (int base = 0; base < cnt; base += 32) {
                            int j = base + lane;
                            pos += __popc(__ballot_sync(0xffffffffu, j < cnt && ls[j] >= sv));
                        }
                        const int last = min(cnt, K - 1);
                        const int j0 = lane, j1 = lane + 32;
                        const bool mv0 = j0 > pos && j0 <= last;
                        const bool mv1 = j1 > pos && j1 <= last;
                        double s0 = 0, s1 = 0;
                        int64_t q0 = 0, q1 = 0;
                        if (mv0) { s0 = ls[j0 - 1]; q0 = lr[j0 - 1]; }
                        if (mv1) { s1 = ls[j1 - 1]; q1 = lr[j1 - 1]; }
                        __syncwarp();
                        if (mv0) { ls[j0] = s0; lr[j0] = q0; }
                        if (mv1) { ls[j1] = s1; lr[j1] = q1; }
                        if (lane == 0) { ls[pos] = sv; lr[pos] = rv; }
                        __syncwarp();
                        cnt = min(cnt + 1, K);
                    }
                }
                __syncwarp();  // every lane's last read of the list precedes lane 0's count write
                if (lane == 0) tkc[qi] = cnt;
                __syncwarp();
            }
            __syncthreads();
        }

        for (int qi = warp; qi < QT; qi += SCAN_THREADS / 32) {
            const int sel = qt * QT + qi;
            if (sel >= nsel) break;
            const int cnt = tkc[qi];
            const int64_t base = ((int64_t)sel * p.nsplit + split) * K;
            for (int j = lane; j < K; j += 32) {
                p.part_s[base + j] = j < cnt ? tks[qi * K + j] : -INFINITY;
                p.part_r[base + j] = j < cnt ? tkr[qi * K + j] : -1;
            }
            if (lane == 0) p.part_c[(int64_t)sel * p.nsplit + split] = cnt;
        }
    }
}

static size_t scan_smem_bytes(int QT, int xstride, int K) {
    return sizeof(double) * ((size_t)QT * xstride + (size_t)QT * SCAN_THREADS + (size_t)QT * K) +
           sizeof(int64_t) * (size_t)QT * K + sizeof(int) * QT;
}

// ---------------------------------------------------------------------------
// merge per-split lists -> final top-k, self-snap, clamp (index.py:176-185)
struct MergeArgs {
    const double *part_s;
    const int64_t *part_r;
    int nsplit;
    int Kp;  // entries per split list
    int k;
    int64_t take;  // min(k, n)
    const int32_t *qsel;
    const int32_t *nsel_dev;
    int32_t nsel_host;
    const float *X;
    int xstride;
    int d;
    const float *Q;  // padded queries [*, xstride]
    int64_t *out_rows;
    double *out_raw;
    double *out_rep;
    int32_t *out_count;
    const int64_t *row_limit;  // nullable, per original query
};

__global__ void __launch_bounds__(128) merge_topk_kernel(MergeArgs a) {
    __shared__ double red_s[4];
    __shared__ int64_t red_r[4];
    const int nsel = a.nsel_dev ? *a.nsel_dev : a.nsel_host;
    const int M = a.nsplit * a.Kp;
    for (int sel = blockIdx.x; sel < nsel; sel += gridDim.x) {
        const int qidx = a.qsel ? a.qsel[sel] : sel;
        const double *ps = a.part_s + (int64_t)sel * M;
        const int64_t *pr_ = a.part_r + (int64_t)sel * M;
        const float *q = a.Q + (int64_t)qidx * a.xstride;
        const int64_t take = a.row_limit ? min(a.take, max((int64_t)0, a.row_limit[qidx])) : a.take;
        double last_s = INFINITY;
        int64_t last_r = -1;
        for (int j = 0; j < a.k; ++j) {
            double bs = -INFINITY;
            int64_t br = -1;
            if (j < take) {
                for (int e = threadIdx.x; e < M; e += blockDim.x) {
                    int64_t r = pr_[e];
                    if (r < 0) continue;
                    double s = ps[e];
                    bool after_last = (last_r < 0) || ranks_before(last_s, last_r, s, r);
                    if (after_last && (br < 0 || ranks_before(s, r, bs, br))) { bs = s; br = r; }
                }
            }
            block_best(bs, br, red_s, red_r);
            const int64_t o = (int64_t)qidx * a.k + j;
            if (br < 0) {
                if (threadIdx.x == 0) {
                    a.out_rows[o] = -1;
                    if (a.out_raw) a.out_raw[o] = 0.0;
                    if (a.out_rep) a.out_rep[o] = 0.0;
                }
                continue;
            }
            double rep;
            finalize_hit(a.X, a.xstride, a.d, q, br, bs, &rep);
            if (threadIdx.x == 0) {
                a.out_rows[o] = br;
                if (a.out_raw) a.out_raw[o] = bs;
                if (a.out_rep) a.out_rep[o] = rep;
            }
            last_s = bs;
            last_r = br;
        }
        if (threadIdx.x == 0) a.out_count[qidx] = (int32_t)take;
    }
}

__global__ void empty_result_kernel(int64_t nq, int k, int64_t *rows, double *raw, double *rep, int32_t *count) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < nq * k) {
        rows[t] = -1;
        if (raw) raw[t] = 0.0;
        if (rep) rep[t] = 0.0;
    }
    if (t < nq) count[t] = 0;
}


// ---------------------------------------------------------------------------
// row-sharded stores: per-shard snap flags + the all-gather merge
__global__ void snap_flags_kernel(const float *__restrict__ x32, int dp8, int d, const float *__restrict__ q,
                                  int64_t nq, int k, const int64_t *__restrict__ rows, const double *__restrict__ raw,
                                  const int32_t *__restrict__ count, int64_t row_offset, uint8_t *__restrict__ snap) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (w >= nq * k) return;
    const int64_t qi = w / k;
    const int j = (int)(w - qi * k);
    int eq = 0;
    if (j < count[qi] && raw[w] > 1.0 - 1e-6) {
        const float *x = x32 + (rows[w] - row_offset) * (int64_t)dp8;
        const float *qq = q + qi * d;
        int bad = 0;
        for (int t = lane; t < d; t += 32) bad |= !(x[t] == qq[t]);
        eq = !__any_sync(0xffffffffu, bad);
    } else {
        __syncwarp();
    }
    if (lane == 0) snap[w] = (uint8_t)eq;
}

__global__ void merge_shards_kernel(const int64_t *__restrict__ rows, const double *__restrict__ raw,
                                    const uint8_t *__restrict__ snap, const int32_t *__restrict__ count, int nshard,
                                    int64_t nq, int k, int64_t *out_rows, double *out_raw, double *out_rep,
                                    int32_t *out_count) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
        int pos[64];
        int total = 0;
        for (int s = 0; s < nshard; ++s) {
            pos[s] = 0;
            total += count[(int64_t)s * nq + q];
        }
        const int take = total < k ? total : k;
        for (int j = 0; j < k; ++j) {
            const int64_t o = q * k + j;
            if (j >= take) {
                out_rows[o] = -1;
                if (out_raw) out_raw[o] = 0.0;
                if (out_rep) out_rep[o] = 0.0;
                continue;
            }
            int bs = -1;
            double best_s = 0;
            int64_t best_r = 0;
            for (int s = 0; s < nshard; ++s) {
                if (pos[s] >= count[(int64_t)s * nq + q]) continue;
                const int64_t e = ((int64_t)s * nq + q) * k + pos[s];
                if (bs < 0 || ranks_before(raw[e], rows[e], best_s, best_r)) {
                    bs = s;
                    best_s = raw[e];
                    best_r = rows[e];
                }
            }
            const int64_t e = ((int64_t)bs * nq + q) * k + pos[bs];
            pos[bs]++;
            out_rows[o] = best_r;
            if (out_raw) out_raw[o] = best_s;
            if (out_rep) out_rep[o] = (snap && snap[e]) ? 1.0 : fmax(-1.0, fmin(1.0, best_s));
        }
        out_count[q] = take;
    }
}
}  // namespace pr

// ===========================================================================
// handle
struct pr_index {
    int dim = 0, dp8 = 0, dp64 = 0, dp128 = 0;
    int64_t count = 0, cap = 0, cap256 = 0;
    float *x32 = nullptr;
    __half *x16 = nullptr;
    pr::I8Rows r8;               // int8 scan copy [cap256, dp128] + per-row scale / error bound
    pr::TcStoreMap tmap;  // TMA descriptor of x16 (rebuilt on reallocation)
    bool tmap_ok = false;
    pr::TcStoreMap tmap8;   // TMA descriptor of x8, 256-row boxes
    pr::TcStoreMap tmap8h;  // ... 128-row boxes (2-CTA scan)
    bool tmap8_ok = false;
    bool pooled = false;  // store buffers come from the stream-ordered pool (small stores)
    pr_search_stats stats{};
    // device scratch (grown on demand, stream-ordered)
    void *scratch = nullptr;
    size_t scratch_bytes = 0, scratch_peak = 0;
    int32_t *d_counters = nullptr;  // [4]: fallback count, candidate count, ...
    cudaStream_t last_stream = nullptr;
    // the scratch block and device counters are per handle: a search on another stream
    // first waits for the previous search (handles may be shared by concurrent routers)
    cudaEvent_t scratch_ev = nullptr;
    bool scratch_ev_used = false;
    // optional per-launch timing of the dominant scan kernel (bench roofline)
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pending, ev_free;
};

namespace pr {

// keep freed blocks mapped in the device's stream-ordered pool: a growing store
// (semantic cache, AKM, seed scratch) would otherwise unmap and re-map memory at every
// growth step, and cudaFree of touched memory was measured to stall for 100+ ms at times
static void keep_pool() {
    static bool kept = false;
    if (kept) return;
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    kept = true;
}

static int ensure_scratch(pr_index *h, size_t bytes, cudaStream_t st) {
    if (h->scratch_bytes >= bytes) return PR_OK;
    keep_pool();
    if (h->scratch) PR_CUDA(cudaFreeAsync(h->scratch, st));
    h->scratch = nullptr;
    h->scratch_bytes = 0;
    // geometric growth (a store that grows every batch reallocates O(log n) times), and
    // 25 % headroom from the first allocation: growing the pool by a GB was measured to
    // stall 100-650 ms, so a batch a few queries larger than the last must not trigger it
    size_t b = std::max({bytes + bytes / 4, (size_t)(1 << 20), h->scratch_peak + h->scratch_peak / 2});
    PR_CUDA(cudaMallocAsync(&h->scratch, b, st));
    if (getenv("PR_DEBUG_RESERVE")) fprintf(stderr, "scratch -> %.1f MB\n", b / 1048576.0);
    h->scratch_bytes = b;
    h->scratch_peak = b;
    return PR_OK;
}

static int timing_pair(pr_index *h, cudaEvent_t *a, cudaEvent_t *b) {
    *a = *b = nullptr;
    if (!h->timing) return PR_OK;
    std::pair<cudaEvent_t, cudaEvent_t> p;
    if (!h->ev_free.empty()) {
        p = h->ev_free.back();
        h->ev_free.pop_back();
    } else {
        PR_CUDA(cudaEventCreate(&p.first));
        PR_CUDA(cudaEventCreate(&p.second));
    }
    h->ev_pending.push_back(p);
    *a = p.first;
    *b = p.second;
    return PR_OK;
}

static int reserve(pr_index *h, int64_t cap, cudaStream_t st) {
    if (cap <= h->cap) return PR_OK;
    // growth doubles (amortised appends); an explicit reservation is honoured as asked
    // (a 10M-row store must not round up to 16.8M rows of fp32 + fp16 + int8)
    const int64_t c = std::max<int64_t>(cap, std::max<int64_t>(2 * h->cap, 1024));
    static const bool dbg = getenv("PR_DEBUG_RESERVE") != nullptr;  // measurement knob
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = now();
    int64_t c256 = round_up<int64_t>(c, 256);
    float *nx32 = nullptr;
    __half *nx16 = nullptr;
    pr::I8Rows n8;
    n8.maxnorm = h->r8.maxnorm;
    const int64_t ntile = c256 / 256;
    const size_t b32 = (size_t)c * h->dp8 * sizeof(float), b16 = (size_t)c256 * h->dp64 * sizeof(__half),
                 b8 = (size_t)c256 * h->dp128, bt = (size_t)ntile * sizeof(pr::I8TileMeta);
    // stores up to 1 GiB live in the stream-ordered pool (growth reuses mapped memory);
    // bigger ones (the knowledge base) use plain allocations the pool cannot hoard
    const bool pooled = b32 + b16 + b8 + 2 * c256 * sizeof(float) + bt <= ((size_t)1 << 30);
    if (pooled) keep_pool();
    auto alloc = [&](void **p, size_t b) { return pooled ? cudaMallocAsync(p, b, st) : cudaMalloc(p, b); };
    auto release = [&](void *p, bool was_pooled) {
        if (p) was_pooled ? cudaFreeAsync(p, st) : cudaFree(p);
    };
    cudaError_t e = alloc((void **)&nx32, b32);
    if (e == cudaSuccess) e = alloc((void **)&nx16, b16);
    if (e == cudaSuccess) e = alloc((void **)&n8.x8, b8);
    if (e == cudaSuccess) e = alloc((void **)&n8.xs, (size_t)c256 * sizeof(float));
    if (e == cudaSuccess) e = alloc((void **)&n8.xe, (size_t)c256 * sizeof(float));
    if (e == cudaSuccess) e = alloc((void **)&n8.xt, bt);
    if (e != cudaSuccess) {
        release(nx32, pooled);
        release(nx16, pooled);
        release(n8.x8, pooled);
        release(n8.xs, pooled);
        release(n8.xe, pooled);
        cudaStreamSynchronize(st);
        PR_FAIL(PR_ERR_NOMEM, "index reserve(%lld rows): %s", (long long)c, cudaGetErrorString(e));
    }
    PR_CUDA(cudaMemsetAsync(nx16, 0, (size_t)c256 * h->dp64 * sizeof(__half), st));
    PR_CUDA(cudaMemsetAsync(n8.x8, 0, (size_t)c256 * h->dp128, st));
    PR_CUDA(cudaMemsetAsync(n8.xs, 0, (size_t)c256 * sizeof(float), st));
    PR_CUDA(cudaMemsetAsync(n8.xe, 0, (size_t)c256 * sizeof(float), st));
    PR_CUDA(cudaMemsetAsync(n8.xt, 0, (size_t)ntile * sizeof(pr::I8TileMeta), st));
    if (h->count > 0) {
        PR_CUDA(cudaMemcpyAsync(nx32, h->x32, (size_t)h->count * h->dp8 * sizeof(float), cudaMemcpyDeviceToDevice, st));
        PR_CUDA(cudaMemcpyAsync(nx16, h->x16, (size_t)h->count * h->dp64 * sizeof(__half), cudaMemcpyDeviceToDevice, st));
        PR_CUDA(cudaMemcpyAsync(n8.x8, h->r8.x8, (size_t)h->count * h->dp128, cudaMemcpyDeviceToDevice, st));
        PR_CUDA(cudaMemcpyAsync(n8.xs, h->r8.xs, (size_t)h->count * sizeof(float), cudaMemcpyDeviceToDevice, st));
        PR_CUDA(cudaMemcpyAsync(n8.xe, h->r8.xe, (size_t)h->count * sizeof(float), cudaMemcpyDeviceToDevice, st));
        PR_CUDA(cudaMemcpyAsync(n8.xt, h->r8.xt, (size_t)(h->cap256 / 256) * sizeof(pr::I8TileMeta),
                                cudaMemcpyDeviceToDevice, st));
    }
    const auto t1 = now();
    // the old buffers may still be read by a search queued on another stream
    PR_CUDA(cudaDeviceSynchronize());
    const auto t2 = now();
    release(h->x32, h->pooled);
    release(h->x16, h->pooled);
    release(h->r8.x8, h->pooled);
    release(h->r8.xs, h->pooled);
    release(h->r8.xe, h->pooled);
    release(h->r8.xt, h->pooled);
    PR_CUDA(cudaStreamSynchronize(st));  // pooled frees are stream-ordered
    h->pooled = pooled;
    if (dbg)
        fprintf(stderr, "reserve %lld -> %lld rows: malloc+enqueue %.2f ms, sync %.2f ms, free %.2f ms\n",
                (long long)h->cap, (long long)c, ms(t0, t1), ms(t1, t2), ms(t2, now()));
    h->x32 = nx32;
    h->x16 = nx16;
    h->r8 = n8;
    h->cap = c;
    h->cap256 = c256;
    h->tmap_ok = false;
    h->tmap8_ok = false;
    return PR_OK;
}

// ---------------------------------------------------------------------------
// search orchestration

constexpr int KMAX_EXACT = 64;

static int pick_qt(int nsel, int xstride, int K) {
    const size_t limit = 200 * 1024;
    int qts[5] = {16, 8, 4, 2, 1};
    for (int i = 0; i < 5; ++i) {
        int qt = qts[i];
        if (qt > 1 && nsel <= qt / 2) continue;  // don't pay for empty query slots
        if (scan_smem_bytes(qt, xstride, K) <= limit) return qt;
    }
    return 1;
}

template <int QT>
static int launch_scan_t(const ScanArgs &a, int grid, cudaStream_t st) {
    size_t smem = scan_smem_bytes(QT, a.xstride, a.K);
    static bool attr_set = false;
    if (!attr_set) {
        PR_CUDA(cudaFuncSetAttribute(exact_scan_kernel<QT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 208 * 1024));
        attr_set = true;
    }
    ::pr::count_launch();
    exact_scan_kernel<QT><<<grid, SCAN_THREADS, smem, st>>>(a);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

static int launch_scan(int QT, const ScanArgs &a, int grid, cudaStream_t st) {
    switch (QT) {
        case 16: return launch_scan_t<16>(a, grid, st);
        case 8: return launch_scan_t<8>(a, grid, st);
        case 4: return launch_scan_t<4>(a, grid, st);
        case 2: return launch_scan_t<2>(a, grid, st);
        default: return launch_scan_t<1>(a, grid, st);
    }
}

static void choose_splits(int64_t n, int qtiles_hint, int *nsplit, int64_t *rows_per_split) {
    const int sms = sm_count();
    int64_t target = std::max<int64_t>(1, (int64_t)2 * sms / std::max(1, qtiles_hint));
    int64_t max_split = std::max<int64_t>(1, ceil_div<int64_t>(n, 1024));
    int64_t ns = std::min(target, max_split);
    ns = std::min<int64_t>(ns, 4 * sms);
    int64_t rps = round_up<int64_t>(ceil_div<int64_t>(n, ns), SCAN_THREADS);
    *rows_per_split = rps;
    *nsplit = (int)ceil_div<int64_t>(n, rps);
}

// Exact path over a (possibly device-sized) selection of queries.  Results
// are scattered to the output positions qsel[i] (or i).
int exact_search(pr_index *h, const float *Qp, const int32_t *qsel, const int32_t *nsel_dev, int nsel_max, int k,
                 int64_t *rows, double *raw, double *rep, int32_t *count, Carve &cv, cudaStream_t st,
                 bool time_it, const int64_t *row_limit) {
    const int K = k;
    int QT = pick_qt(nsel_max, h->dp8, K);
    int nsplit;
    int64_t rps;
    // a device-sized selection (fallback list) is usually a handful of queries:
    // split the rows finely enough to fill the GPU even then
    const int tiles_hint = nsel_dev ? std::min(ceil_div(nsel_max, QT), 4) : ceil_div(nsel_max, QT);
    choose_splits(h->count, tiles_hint, &nsplit, &rps);
    double *ps = cv.take<double>((size_t)nsel_max * nsplit * K);
    int64_t *prr = cv.take<int64_t>((size_t)nsel_max * nsplit * K);
    int32_t *pc = cv.take<int32_t>((size_t)nsel_max * nsplit);
    ScanArgs a{h->x32, h->count, h->dp8, h->dim, Qp, qsel, nsel_dev, nsel_max, nsplit, rps, K, ps, prr, pc,
               row_limit};
    int64_t work = (int64_t)ceil_div(nsel_max, QT) * nsplit;
    int grid = (int)std::min<int64_t>(work, (int64_t)sm_count() * 2);
    if (grid < 1) grid = 1;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (time_it) {
        int trc = timing_pair(h, &e0, &e1);
        if (trc) return trc;
    }
    if (e0) PR_CUDA(cudaEventRecord(e0, st));
    int rc = launch_scan(QT, a, grid, st);
    if (rc) return rc;
    if (e1) PR_CUDA(cudaEventRecord(e1, st));
    MergeArgs m{ps, prr, nsplit, K, k, std::min<int64_t>(k, h->count), qsel, nsel_dev, nsel_max,
                h->x32, h->dp8, h->dim, Qp, rows, raw, rep, count, row_limit};
    int mgrid = std::max(1, std::min(nsel_max, sm_count() * 8));
    ::pr::count_launch();
    merge_topk_kernel<<<mgrid, 128, 0, st>>>(m);
    PR_LAUNCH_CHECK();
    h->stats.nsplit = nsplit;
    return PR_OK;
}

size_t exact_scratch_bytes(int nsel_max, int k, int64_t n) {
    int QT = 1;
    (void)QT;
    const int sms = sm_count();
    int64_t ns = std::min<int64_t>(4 * sms, std::max<int64_t>(1, ceil_div<int64_t>(n, 1024)));
    return (size_t)nsel_max * ns * k * (8 + 8) + (size_t)nsel_max * ns * 4 + 4096;
}

}  // namespace pr

// ===========================================================================
// C ABI
using namespace pr;

extern "C" {

const char *pr_last_error(void) { return pr::last_error(); }
int pr_abi_version(void) { return 2; }  // 2: pr_cascade_gate takes the L3 outcome

int pr_device_info(int *sms, int *major, int *minor) {
    int dev = 0;
    PR_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp p;
    PR_CUDA(cudaGetDeviceProperties(&p, dev));
    if (sms) *sms = p.multiProcessorCount;
    if (major) *major = p.major;
    if (minor) *minor = p.minor;
    if (p.major != 10 || p.minor != 0)
        PR_FAIL(PR_ERR_UNSUPPORTED, "libpentarag is built for sm_100a only; device is sm_%d%d", p.major, p.minor);
    return PR_OK;
}

int pr_check_unit(const float *d_vecs, int64_t n, int dim, double tol, uint8_t *d_bad, void *stream) {
    if (n < 0 || dim < 1) PR_FAIL(PR_ERR_BAD_ARG, "pr_check_unit: bad shape");
    if (n == 0) return PR_OK;
    int64_t threads = n * 32;
    ::pr::count_launch();
    check_unit_kernel<<<(unsigned)ceil_div<int64_t>(threads, 256), 256, 0, as_stream(stream)>>>(d_vecs, n, dim, tol, d_bad);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

int pr_index_create(int dim, int64_t capacity, uint32_t flags, pr_index **out) {
    (void)flags;
    if (!out) PR_FAIL(PR_ERR_BAD_ARG, "out is NULL");
    if (dim < 1) PR_FAIL(PR_ERR_BAD_ARG, "dim must be >= 1");  // index.py:77-78
    pr_index *h = new pr_index();
    h->dim = dim;
    h->dp8 = round_up(dim, 8);
    h->dp64 = round_up(dim, 64);
    h->dp128 = round_up(dim, 128);
    int rc = reserve(h, std::max<int64_t>(capacity, 1024), nullptr);
    if (rc) {
        delete h;
        return rc;
    }
    PR_CUDA(cudaMalloc(&h->d_counters, 16 * sizeof(int32_t)));
    PR_CUDA(cudaMalloc(&h->r8.maxnorm, sizeof(uint32_t)));
    PR_CUDA(cudaMemset(h->r8.maxnorm, 0, sizeof(uint32_t)));
    *out = h;
    return PR_OK;
}

int pr_index_destroy(pr_index *h) {
    if (!h) return PR_OK;
    cudaDeviceSynchronize();
    for (void *p : {(void *)h->x32, (void *)h->x16, (void *)h->r8.x8, (void *)h->r8.xs, (void *)h->r8.xe,
                    (void *)h->r8.xt}) {
        if (p) h->pooled ? cudaFreeAsync(p, 0) : cudaFree(p);
    }
    cudaDeviceSynchronize();
    cudaFree(h->r8.maxnorm);
    if (h->scratch) cudaFree(h->scratch);
    if (h->d_counters) cudaFree(h->d_counters);
    if (h->scratch_ev) cudaEventDestroy(h->scratch_ev);
    for (auto &p : h->ev_pending) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    for (auto &p : h->ev_free) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    delete h;
    return PR_OK;
}

int64_t pr_index_count(const pr_index *h) { return h ? h->count : -1; }
int pr_index_dim(const pr_index *h) { return h ? h->dim : -1; }

int pr_index_reserve(pr_index *h, int64_t capacity, void *stream) {
    if (!h || capacity < 0) PR_FAIL(PR_ERR_BAD_ARG, "bad reserve");
    return reserve(h, capacity, as_stream(stream));
}

int pr_index_append(pr_index *h, const float *d_vecs, int64_t n, void *stream) {
    if (!h || n < 0) PR_FAIL(PR_ERR_BAD_ARG, "bad append");
    if (n == 0) return PR_OK;
    cudaStream_t st = as_stream(stream);
    int rc = reserve(h, h->count + n, st);
    if (rc) return rc;
    ::pr::count_launch();
    write_rows_kernel<<<grid_for(n * h->dp64), 256, 0, st>>>(d_vecs, n, h->dim, nullptr, h->count, h->x32, h->dp8,
                                                              h->x16, h->dp64);
    PR_LAUNCH_CHECK();
    rc = pr::i8_quantize_rows(d_vecs, n, h->dim, nullptr, h->count, h->dp128, h->r8, st);
    if (rc) return rc;
    h->count += n;
    return PR_OK;
}

int pr_index_update_rows(pr_index *h, const int64_t *d_rows, const float *d_vecs, int64_t n, void *stream) {
    if (!h || n < 0) PR_FAIL(PR_ERR_BAD_ARG, "bad update");
    if (n == 0) return PR_OK;
    ::pr::count_launch();
    write_rows_kernel<<<grid_for(n * h->dp64), 256, 0, as_stream(stream)>>>(d_vecs, n, h->dim, d_rows, 0, h->x32,
                                                                             h->dp8, h->x16, h->dp64);
    PR_LAUNCH_CHECK();
    return pr::i8_quantize_rows(d_vecs, n, h->dim, d_rows, 0, h->dp128, h->r8, as_stream(stream));
}

int pr_index_clear(pr_index *h) {
    if (!h) PR_FAIL(PR_ERR_BAD_ARG, "null handle");
    h->count = 0;
    return PR_OK;
}

int pr_index_truncate(pr_index *h, int64_t n) {
    if (!h || n < 0 || n > h->count) PR_FAIL(PR_ERR_BAD_ARG, "bad truncate");
    h->count = n;
    return PR_OK;
}

int pr_index_read_rows(const pr_index *h, int64_t row0, int64_t n, float *d_out, void *stream) {
    if (!h || row0 < 0 || n < 0 || row0 + n > h->count) PR_FAIL(PR_ERR_BAD_ARG, "read_rows out of range");
    if (n == 0) return PR_OK;
    ::pr::count_launch();
    read_rows_kernel<<<grid_for(n * h->dim), 256, 0, as_stream(stream)>>>(h->x32, h->dp8, h->dim, row0, n, d_out);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

int pr_index_gather_rows(const pr_index *h, const int64_t *d_rows, int64_t n, int64_t row_offset, float *d_out,
                         void *stream) {
    if (!h || n < 0) PR_FAIL(PR_ERR_BAD_ARG, "bad gather_rows");
    if (n == 0) return PR_OK;
    ::pr::count_launch();
    gather_owned_kernel<<<std::min(grid_for(n * h->dim), pr::sm_count() * 16), 256, 0, as_stream(stream)>>>(
        h->x32, h->dp8, h->dim, h->count, d_rows, n, row_offset, d_out);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

int pr_index_append_from(pr_index *h, const pr_index *src, const int64_t *d_src_rows, int64_t n, void *stream) {
    if (!h || !src || n < 0 || src->dim != h->dim) PR_FAIL(PR_ERR_BAD_ARG, "bad append_from");
    if (n == 0) return PR_OK;
    cudaStream_t st = as_stream(stream);
    int rc = reserve(h, h->count + n, st);
    if (rc) return rc;
    ::pr::count_launch();
    gather_rows_kernel<<<grid_for(n * h->dp64), 256, 0, st>>>(src->x32, src->x16, d_src_rows, n, h->dp8, h->dp64,
                                                               h->count, h->x32, h->x16);
    PR_LAUNCH_CHECK();
    rc = pr::i8_gather_rows(src->r8, d_src_rows, n, h->dp128, h->count, h->r8, st);
    if (rc) return rc;
    h->count += n;
    return PR_OK;
}

int pr_index_search(pr_index *h, const float *d_q, int64_t nq, int k, uint32_t mode, int64_t *d_rows, double *d_raw,
                    double *d_reported, int32_t *d_count, void *stream) {
    return pr_index_search_ex(h, d_q, nq, k, mode, nullptr, d_rows, d_raw, d_reported, d_count, stream);
}

struct QueryList {
    const int32_t *list = nullptr;   // device: query index per listed position
    const int32_t *nlist = nullptr;  // device: live count
    int64_t hint = 0;                // host estimate of the live count (grid shape)
};

static int search_impl(pr_index *h, const float *d_q, int64_t nq, int k, uint32_t mode, const int64_t *d_row_limit,
                       int64_t *d_rows, double *d_raw, double *d_reported, int32_t *d_count, void *stream,
                       const QueryList &ql, double floor);

static int search_entry(pr_index *h, const float *d_q, int64_t nq, int k, uint32_t mode, const int64_t *d_row_limit,
                        int64_t *d_rows, double *d_raw, double *d_reported, int32_t *d_count, void *stream,
                        const QueryList &ql, double floor = -INFINITY) {
    if (!h) PR_FAIL(PR_ERR_BAD_ARG, "null handle");
    cudaStream_t st = as_stream(stream);
    if (!h->scratch_ev) PR_CUDA(cudaEventCreateWithFlags(&h->scratch_ev, cudaEventDisableTiming));
    if (h->scratch_ev_used && h->last_stream != st) PR_CUDA(cudaStreamWaitEvent(st, h->scratch_ev, 0));
    const int rc = search_impl(h, d_q, nq, k, mode, d_row_limit, d_rows, d_raw, d_reported, d_count, stream, ql, floor);
    if (rc == PR_OK) {
        PR_CUDA(cudaEventRecord(h->scratch_ev, st));
        h->scratch_ev_used = true;
    }
    return rc;
}

int pr_index_search_list(pr_index *h, const float *d_q, const int32_t *d_list, const int32_t *d_nlist, int64_t nq_max,
                         int64_t nq_hint, int k, uint32_t mode, const int64_t *d_row_limit, int64_t *d_rows,
                         double *d_raw, double *d_reported, int32_t *d_count, void *stream) {
    if (!d_list || !d_nlist) PR_FAIL(PR_ERR_BAD_ARG, "search_list needs a device list and count");
    QueryList ql{d_list, d_nlist, nq_hint > 0 ? nq_hint : nq_max};
    return search_entry(h, d_q, nq_max, k, mode, d_row_limit, d_rows, d_raw, d_reported, d_count, stream, ql);
}

int pr_index_search_ex(pr_index *h, const float *d_q, int64_t nq, int k, uint32_t mode, const int64_t *d_row_limit,
                       int64_t *d_rows, double *d_raw, double *d_reported, int32_t *d_count, void *stream) {
    return search_entry(h, d_q, nq, k, mode, d_row_limit, d_rows, d_raw, d_reported, d_count, stream, QueryList{});
}

int pr_index_search_floor(pr_index *h, const float *d_q, int64_t nq, int k, uint32_t mode, const int64_t *d_row_limit,
                          double floor, int64_t *d_rows, double *d_raw, double *d_reported, int32_t *d_count,
                          void *stream) {
    if (floor != floor) PR_FAIL(PR_ERR_BAD_ARG, "floor is NaN");
    return search_entry(h, d_q, nq, k, mode, d_row_limit, d_rows, d_raw, d_reported, d_count, stream, QueryList{},
                        floor);
}

static int search_impl(pr_index *h, const float *d_q, int64_t nq, int k, uint32_t mode, const int64_t *d_row_limit,
                       int64_t *d_rows, double *d_raw, double *d_reported, int32_t *d_count, void *stream,
                       const QueryList &ql, double floor) {
    if (!h) PR_FAIL(PR_ERR_BAD_ARG, "null handle");
    if (k < 1) PR_FAIL(PR_ERR_BAD_ARG, "k must be >= 1");  // index.py:161-162
    if (nq < 0 || nq > INT32_MAX / 2) PR_FAIL(PR_ERR_BAD_ARG, "bad query count");
    if (mode > PR_SEARCH_TENSOR_I8) PR_FAIL(PR_ERR_BAD_ARG, "bad mode");
    cudaStream_t st = as_stream(stream);
    h->last_stream = st;
    h->stats = pr_search_stats{};
    h->stats.queries = nq;
    if (nq == 0) return PR_OK;
    if (ql.list && k > KMAX_EXACT) PR_FAIL(PR_ERR_BAD_ARG, "listed search supports k <= %d", KMAX_EXACT);
    if (h->count == 0 || k > KMAX_EXACT) {
        if (h->count == 0) {
            ::pr::count_launch();
            empty_result_kernel<<<(unsigned)ceil_div<int64_t>(nq * k, 256), 256, 0, st>>>(nq, k, d_rows, d_raw,
                                                                                         d_reported, d_count);
            PR_LAUNCH_CHECK();
            return PR_OK;
        }
    }
    if (k > KMAX_EXACT)
        return pr::big_k_search(h->x32, h->count, h->dp8, h->dim, d_q, nq, k, d_row_limit, d_rows, d_raw, d_reported,
                                d_count, st);

    const bool tensor_ok = pr::tc_eligible(h->dim, h->count, k);
    // AUTO: the int8 scan (1.4-1.6x the fp16 scan's rate, same results) wherever a
    // tensor-core scan pays off; the fp16 scan for d > 2048; the exact scan otherwise
    // The int8 scan's per-(query, split) bounds start cold, so it needs long row splits to
    // amortise the start: below ~512k rows the fp16 scan is faster (40k x 1024, 2048
    // queries, k=10: 0.42 ms fp16 vs 3.5 ms int8; 10M rows: int8 1.6x faster).
    // a listed search decides with the list's CAPACITY, not the host's estimate of its live
    // count: the estimate comes from the previous span and can be tiny (a span the caches
    // answered), and the exact scan's cost grows with the live count — a 2M-row knowledge
    // base once scanned a 2,000-query list in fp64 for 1.5 s (the tensor path's cost for a
    // short list is bounded: its grid is still shaped by the estimate)
    const bool tc_pays = mode == PR_SEARCH_AUTO && tensor_ok && pr::tc_worthwhile(h->count, nq);
    // with a floor the int8 scan starts from a known bound (no cold start, no pilot): it
    // pays at every size a tensor-core scan does
    const bool has_floor = floor > -INFINITY;
    const bool i8_pays = tc_pays && (h->count >= ((int64_t)1 << 19) || has_floor);
    const bool use_i8 = (mode == PR_SEARCH_TENSOR_I8 || i8_pays) && tensor_ok && pr::tc8_eligible(h->dim);
    bool use_tc = !use_i8 && tensor_ok && (mode == PR_SEARCH_TENSOR || mode == PR_SEARCH_TENSOR_I8 || tc_pays);

    size_t need = (size_t)nq * h->dp8 * sizeof(float) + exact_scratch_bytes((int)nq, k, h->count) + 65536;
    if (use_tc) need += pr::tc_scratch_bytes(nq, h->dp64, h->count, k);
    if (use_i8) need += pr::tc8_scratch_bytes(nq, h->dp128, h->count);
    int rc = ensure_scratch(h, need, st);
    if (rc) return rc;
    Carve cv{reinterpret_cast<char *>(h->scratch)};
    float *Qp = cv.take<float>((size_t)nq * h->dp8);
    ::pr::count_launch();
    if (ql.list)
        gather_pad_queries_kernel<<<std::min(grid_for(nq * h->dp8), sm_count() * 16), 256, 0, st>>>(
            d_q, ql.list, ql.nlist, nq, h->dim, h->dp8, Qp);
    else
        pad_queries_kernel<<<grid_for(nq * h->dp8), 256, 0, st>>>(d_q, nq, h->dim, h->dp8, Qp);
    PR_LAUNCH_CHECK();

    if (use_i8) {
        h->stats.path = PR_SEARCH_TENSOR_I8;
        if (!h->tmap8_ok) {
            rc = pr::i8_make_store_map(&h->tmap8, h->r8.x8, h->cap256, h->dp128, 256);
            if (rc) return rc;
            rc = pr::i8_make_store_map(&h->tmap8h, h->r8.x8, h->cap256, h->dp128, 128);
            if (rc) return rc;
            h->tmap8_ok = true;
        }
        pr::Tc8Search ts{};
        ts.x32 = h->x32;
        ts.store_map = &h->tmap8;
        ts.store_map_half = &h->tmap8h;
        ts.x8_rows = h->cap256;
        ts.rows8 = h->r8;
        ts.n = h->count;
        ts.d = h->dim;
        ts.dp8 = h->dp8;
        ts.dp128 = h->dp128;
        ts.qp = Qp;
        ts.nq = nq;
        ts.k = k;
        ts.rows = d_rows;
        ts.raw = d_raw;
        ts.rep = d_reported;
        ts.count = d_count;
        ts.counters = h->d_counters;
        ts.row_limit = d_row_limit;
        ts.nq_dev = ql.nlist;
        ts.nq_hint = ql.hint;
        ts.floor = floor;
        rc = timing_pair(h, &ts.ev_begin, &ts.ev_end);
        if (rc) return rc;
        rc = pr::tc8_search(ts, cv, st, &h->stats);
        if (rc) return rc;
        // candidate-buffer overflows -> exact rescan of just those queries
        return exact_search(h, Qp, ts.fallback_list, h->d_counters, (int)nq, k, d_rows, d_raw, d_reported, d_count,
                            cv, st, false, d_row_limit);
    }
    if (!use_tc) {
        h->stats.path = PR_SEARCH_EXACT;
        return exact_search(h, Qp, nullptr, ql.nlist, (int)nq, k, d_rows, d_raw, d_reported, d_count, cv, st, true,
                            d_row_limit);
    }
    h->stats.path = PR_SEARCH_TENSOR;
    if (!h->tmap_ok) {
        rc = pr::tc_make_store_map(&h->tmap, h->x16, h->cap256, h->dp64);
        if (rc) return rc;
        h->tmap_ok = true;
    }
    pr::TcSearch ts{};
    ts.x32 = h->x32;
    ts.x16 = h->x16;
    ts.store_map = &h->tmap;
    ts.n = h->count;
    ts.d = h->dim;
    ts.dp8 = h->dp8;
    ts.dp64 = h->dp64;
    ts.q32 = d_q;
    ts.qp = Qp;
    ts.nq = nq;
    ts.k = k;
    ts.rows = d_rows;
    ts.raw = d_raw;
    ts.rep = d_reported;
    ts.count = d_count;
    ts.counters = h->d_counters;
    ts.row_limit = d_row_limit;
    rc = timing_pair(h, &ts.ev_begin, &ts.ev_end);
    if (rc) return rc;
    rc = pr::tc_search(ts, cv, st, &h->stats);
    if (rc) return rc;
    // certificate failures -> exact rescan of just those queries (device-sized list)
    return exact_search(h, Qp, ts.fallback_list, h->d_counters, (int)nq, k, d_rows, d_raw, d_reported, d_count, cv,
                        st, false, d_row_limit);
}

int pr_index_set_timing(pr_index *h, int enable) {
    if (!h) PR_FAIL(PR_ERR_BAD_ARG, "null handle");
    h->timing = enable != 0;
    return PR_OK;
}

int pr_index_scan_time(pr_index *h, double *total_ms, int64_t *launches) {
    if (!h) PR_FAIL(PR_ERR_BAD_ARG, "null handle");
    double tot = 0.0;
    int64_t n = 0;
    for (auto &p : h->ev_pending) {
        PR_CUDA(cudaEventSynchronize(p.second));
        float ms = 0.f;
        PR_CUDA(cudaEventElapsedTime(&ms, p.first, p.second));
        tot += ms;
        ++n;
        h->ev_free.push_back(p);
    }
    h->ev_pending.clear();
    if (total_ms) *total_ms = tot;
    if (launches) *launches = n;
    return PR_OK;
}

long long pr_launch_count(void) { return g_launches.load(); }

int pr_index_last_stats(pr_index *h, pr_search_stats *out) {
    if (!h || !out) PR_FAIL(PR_ERR_BAD_ARG, "null");
    if (h->stats.path == PR_SEARCH_TENSOR || h->stats.path == PR_SEARCH_TENSOR_I8) {
        int32_t c[4];
        PR_CUDA(cudaMemcpyAsync(c, h->d_counters, sizeof(c), cudaMemcpyDeviceToHost, h->last_stream));
        PR_CUDA(cudaStreamSynchronize(h->last_stream));
        h->stats.fallback = c[0];
        h->stats.candidates = c[1];
        if (h->stats.path == PR_SEARCH_TENSOR)
            h->stats.collected = c[2];
        else
            h->stats.appended = c[3];
        h->stats.tensor_queries = h->stats.queries;
    }
    *out = h->stats;
    return PR_OK;
}

int pr_index_snap_flags(const pr_index *h, const float *d_q, int64_t nq, int k, const int64_t *d_rows,
                        const double *d_raw, const int32_t *d_count, int64_t row_offset, uint8_t *d_snap,
                        void *stream) {
    if (!h || nq < 0 || k < 1) PR_FAIL(PR_ERR_BAD_ARG, "bad snap_flags");
    if (nq == 0) return PR_OK;
    int64_t threads = nq * k * 32;
    ::pr::count_launch();
    snap_flags_kernel<<<(unsigned)ceil_div<int64_t>(threads, 256), 256, 0, as_stream(stream)>>>(
        h->x32, h->dp8, h->dim, d_q, nq, k, d_rows, d_raw, d_count, row_offset, d_snap);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

int pr_merge_shards(const int64_t *d_rows, const double *d_raw, const uint8_t *d_snap, const int32_t *d_count,
                    int nshard, int64_t nq, int k, int64_t *d_out_rows, double *d_out_raw, double *d_out_reported,
                    int32_t *d_out_count, void *stream) {
    if (nshard < 1 || nshard > 64 || nq < 0 || k < 1) PR_FAIL(PR_ERR_BAD_ARG, "bad merge_shards");
    if (nq == 0) return PR_OK;
    ::pr::count_launch();
    merge_shards_kernel<<<(unsigned)ceil_div<int64_t>(nq, 128), 128, 0, as_stream(stream)>>>(
        d_rows, d_raw, d_snap, d_count, nshard, nq, k, d_out_rows, d_out_raw, d_out_reported, d_out_count);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

}  // extern "C"
