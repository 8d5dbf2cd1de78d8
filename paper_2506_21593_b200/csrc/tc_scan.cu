// Tensor-core score+select for FlatIndex.search (index.py:155-189), sm_100a.
//
// Stage 1 (tc_scan_kernel): S = Q16 · X16ᵀ on tcgen05 (kind::f16, fp32
//   accumulators in TMEM).  One CTA = 128 queries (TMEM lanes) × a split of
//   256-row store tiles (TMEM columns).  Warp 0 issues TMA loads of 64-column
//   (128 B, SWIZZLE_128B) K-slices into a 3-stage smem ring, warp 1 issues the
//   MMAs from one elected lane into a double-buffered TMEM accumulator, warps
//   4-7 drain TMEM with tcgen05.ld (thread i <-> query i) and keep, per query,
//   the top TC_KP approximate scores of the split.  The score matrix never
//   leaves the SM.
// Stage 2 (tc_rescore_kernel): per query, rescore in fp64 numpy-einsum order
//   (bit-exact) every candidate that can still reach the top-k, pick the exact
//   top-k and certify it against the largest score any non-candidate could
//   have (split floor + rigorous fp16 error bound).  Queries whose
//   certificate fails are listed for an exact fp64 rescan (index.cu).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "common.cuh"
#include "select.cuh"
#include "tc_scan.cuh"
#include "ptx.cuh"

namespace pr {

constexpr int TC_STAGES = 4;
constexpr int TC_THREADS = 256;
constexpr int TC_A_BYTES = TC_BLOCK_M * TC_BLOCK_K * 2;  // 16 KB
constexpr int TC_B_BYTES = TC_BLOCK_N * TC_BLOCK_K * 2;  // 32 KB
constexpr int TC_EPI_THREADS = 128;
constexpr int TC_TMEM_COLS = 512;

constexpr size_t tc_smem_bytes() {
    return 1024 /*alignment slack*/ + (size_t)TC_STAGES * (TC_A_BYTES + TC_B_BYTES) +
           (size_t)32 * TC_EPI_THREADS * 4 /*per-thread score spill for candidate chunks*/ + 256 /*barriers*/;
}

struct TcScanParams {
    int64_t n;
    int nkb;              // K blocks (dp64 / 64)
    int nsplit;
    int tiles_per_split;  // 256-row tiles per split
    int ntiles;
    int qtiles;
    uint64_t *cand;       // [nq_pad, nsplit, TC_KP] keys
    const int64_t *row_limit;  // nullable
    int64_t nq;
    // COLLECT mode (second pass for certificate failures): the query rows of the
    // tile are the compacted list qmap[0..*nlist); every row with approx >= thr[slot]
    // is appended to cbuf[slot][*] (ccount[slot] counts, capped at cap)
    const int32_t *qmap;
    const int32_t *nlist;
    const float *thr;
    int32_t *ccount;
    int32_t *cbuf;
    int cap;
};

template <bool COLLECT>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_scan_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tx, TcScanParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for SWIZZLE_128B, as an offset from the __shared__ array so
    // every derived pointer stays in the shared window (LDS/STS, not generic LD/ST)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *sA = smem;
    uint8_t *sB = sA + TC_STAGES * TC_A_BYTES;
    float *spill = reinterpret_cast<float *>(sB + TC_STAGES * TC_B_BYTES);  // [32][128]
    uint64_t *full = reinterpret_cast<uint64_t *>(spill + 32 * TC_EPI_THREADS);
    uint64_t *empty = full + TC_STAGES;
    uint64_t *tfull = empty + TC_STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // persistent static schedule: work item = (query tile, row split), query tile
    // fastest so CTAs running together stream the same store tiles through L2
    const int nitems = p.qtiles * p.nsplit;
    const int ntile_q = COLLECT ? (int)ceil_div<int64_t>(*p.nlist, TC_BLOCK_M) : p.qtiles;
    auto item_of = [&](int item, int &qtile, int &split, int &t0, int &nloc) {
        qtile = item % p.qtiles;
        split = item / p.qtiles;
        t0 = split * p.tiles_per_split;
        const int t1 = min(p.ntiles, t0 + p.tiles_per_split);
        nloc = (qtile < ntile_q) ? max(0, t1 - t0) : 0;  // COLLECT: tiles past the list do nothing
    };

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tq);
        tma_prefetch_desc(&tx);
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], TC_EPI_THREADS / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TC_TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                int qtile, split, t0, nloc;
                item_of(item, qtile, split, t0, nloc);
                for (int i = 0; i < nloc; ++i) {
                    const int t = t0 + i;
                    for (int kb = 0; kb < p.nkb; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        mbar_expect_tx(&full[stage], TC_A_BYTES + TC_B_BYTES);
                        tma_load_2d(sA + stage * TC_A_BYTES, &tq, &full[stage], kb * TC_BLOCK_K, qtile * TC_BLOCK_M);
                        tma_load_2d(sB + stage * TC_B_BYTES, &tx, &full[stage], kb * TC_BLOCK_K, t * TC_BLOCK_N);
                        if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (single thread) ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int tix = 0;  // running accumulator-tile counter across items
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                int qtile, split, t0, nloc;
                item_of(item, qtile, split, t0, nloc);
                for (int i = 0; i < nloc; ++i, ++tix) {
                    const int acc = tix & 1;
                    const uint32_t aphase = (tix >> 1) & 1;
                    mbar_wait(&tempty[acc], aphase ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem + acc * TC_BLOCK_N;
                    for (int kb = 0; kb < p.nkb; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint64_t ad = sw128_desc(smem_u32(sA + stage * TC_A_BYTES));
                        const uint64_t bd = sw128_desc(smem_u32(sB + stage * TC_B_BYTES));
#pragma unroll
                        for (int k = 0; k < TC_BLOCK_K / 16; ++k)  // +32 B per K=16 step inside the swizzle atom
                            mma_f16(d_tmem, ad + 2 * k, bd + 2 * k, (kb | k) != 0);
                        mma_commit(&empty[stage]);
                        if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
                    }
                    mma_commit(&tfull[acc]);
                }
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> top-K' ----------------
        const int et = threadIdx.x - 128;  // 0..127 == TMEM lane == query within tile
        const int ew = warp - 4;
        int tix = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
            int qtile, split, t0, nloc;
            item_of(item, qtile, split, t0, nloc);
            const int64_t my_slot = (int64_t)qtile * TC_BLOCK_M + et;
            int64_t my_q = my_slot;
            float cthr = INFINITY;
            if (COLLECT) {
                my_q = (my_slot < *p.nlist) ? p.qmap[my_slot] : -1;
                if (my_q >= 0) cthr = p.thr[my_slot];
            }
            int64_t my_lim = (p.row_limit && my_q >= 0 && my_q < p.nq) ? min(p.n, p.row_limit[my_q]) : p.n;
            if (my_q < 0) my_lim = 0;
            float ts[TC_KP];
            uint32_t tr[TC_KP];
#pragma unroll
            for (int i = 0; i < TC_KP; ++i) {
                ts[i] = -INFINITY;
                tr[i] = 0xFFFFFFFFu;
            }
            for (int i = 0; i < nloc; ++i, ++tix) {
                const int acc = tix & 1;
                const uint32_t aphase = (tix >> 1) & 1;
                mbar_wait(&tfull[acc], aphase);
                tc_fence_after();
                const int64_t rbase = (int64_t)(t0 + i) * TC_BLOCK_N;
#pragma unroll 1
                for (int c = 0; c < TC_BLOCK_N / 32; ++c) {
                    uint32_t v[32];
                    TMEM_LD32(tmem + ((uint32_t)(ew * 32) << 16) + acc * TC_BLOCK_N + c * 32, v);
                    tmem_wait_ld();
                    const int64_t rb = rbase + c * 32;
                    const int64_t rem_rows = my_lim - rb;
                    const int lim = rem_rows < 32 ? (int)rem_rows : 32;
                    const float thr = ts[TC_KP - 1];
                    uint32_t mask = 0;
                    if (COLLECT) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) mask |= (__uint_as_float(v[j]) >= cthr ? 1u : 0u) << j;
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) mask |= (__uint_as_float(v[j]) > thr ? 1u : 0u) << j;
                    }
                    if (lim < 32) mask &= (lim <= 0) ? 0u : (0xFFFFFFFFu >> (32 - lim));
                    if (COLLECT && mask) {
                        const int cnt = __popc(mask);
                        const int base = atomicAdd(&p.ccount[my_slot], cnt);
                        int o = base;
                        while (mask && o < p.cap) {
                            const int j = __ffs(mask) - 1;
                            mask &= mask - 1;
                            p.cbuf[my_slot * (int64_t)p.cap + o] = (int32_t)(rb + j);
                            ++o;
                        }
                        mask = 0;
                    }
                    if (mask) {
                        // rare: spill this chunk to smem so candidates can be indexed dynamically
#pragma unroll
                        for (int j = 0; j < 32; ++j) spill[j * TC_EPI_THREADS + et] = __uint_as_float(v[j]);
                        do {
                            const int j = __ffs(mask) - 1;
                            mask &= mask - 1;
                            const float s = spill[j * TC_EPI_THREADS + et];
                            if (s > ts[TC_KP - 1]) topk_insert(ts, tr, s, (uint32_t)(rb + j));
                        } while (mask);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
            }
            if (!COLLECT) {
                uint64_t *out = p.cand + (my_slot * p.nsplit + split) * TC_KP;
#pragma unroll
                for (int s = 0; s < TC_KP; ++s) out[s] = (tr[s] == 0xFFFFFFFFu) ? 0ull : cand_key(ts[s], tr[s]);
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_TMEM_COLS) : "memory");
    }
}

// ---------------------------------------------------------------------------
// queries fp32 (padded to dp8) -> fp16 [nq_pad, dp64], zero padding rows/cols
__global__ void queries_to_f16_kernel(const float *__restrict__ qp, int64_t nq, int dp8, int d, int64_t nq_pad, int dp64,
                                      __half *__restrict__ out) {
    int64_t total = nq_pad * (int64_t)dp64;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = t / dp64;
        int j = (int)(t - i * dp64);
        float v = (i < nq && j < d) ? qp[i * dp8 + j] : 0.0f;
        out[t] = __float2half_rn(v);
    }
}

// ---------------------------------------------------------------------------
// stage 2: certified exact rescoring, one CTA per query
constexpr int RS_THREADS = 128;
constexpr int RS_MAX = 512;  // rescored candidates per query before giving up

struct RescoreArgs {
    const uint64_t *cand;
    int nsplit;
    int64_t nq;
    int k;
    int64_t take;
    double err;  // E: |approx - exact| bound
    const float *x32;
    int dp8, d;
    const float *qp;
    int64_t *rows;
    double *raw, *rep;
    int32_t *count;
    int32_t *counters;
    int32_t *fallback;
    const int64_t *row_limit;
    int32_t *clist;  // certificate failures -> collect pass: query ids (counters[2] counts)
    float *cthr;     // ... and their collect thresholds (rounded down to fp32)
};

// hand a query whose certificate failed to the collect pass (or, without
// one, straight to the exact rescan)
__device__ __forceinline__ void defer_query(const RescoreArgs &a, int64_t q, double thr) {
    if (threadIdx.x == 0) {
        if (a.clist) {
            const int slot = atomicAdd(&a.counters[2], 1);
            a.clist[slot] = (int32_t)q;
            a.cthr[slot] = __double2float_rd(thr);
        } else {
            const int slot = atomicAdd(&a.counters[0], 1);
            a.fallback[slot] = (int32_t)q;
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(RS_THREADS) tc_rescore_kernel(RescoreArgs a) {
    extern __shared__ __align__(16) float rs_dyn[];  // [1 + RS_THREADS / 32][dp8]: query + per-warp row
    __shared__ int64_t r_row[RS_MAX];
    __shared__ double r_apx[RS_MAX];
    __shared__ double r_ex[RS_MAX];
    __shared__ double red_s[RS_THREADS / 32];
    __shared__ int64_t red_r[RS_THREADS / 32];
    __shared__ int r_n;
    const int M = a.nsplit * TC_KP;
    for (int64_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
        const uint64_t *cq = a.cand + q * (int64_t)M;
        const int64_t take = a.row_limit ? min(a.take, max((int64_t)0, a.row_limit[q])) : a.take;
        // F: the largest approximate score a non-candidate can have
        double F = -INFINITY;
        for (int sp = threadIdx.x; sp < a.nsplit; sp += RS_THREADS) {
            uint64_t last = cq[sp * TC_KP + TC_KP - 1];
            if (last) F = fmax(F, (double)key_score(last));
        }
        {
            double tmp = F;
            int64_t dummy = 0;
            // max-reduce via block_best on (score, row=0)
            int64_t rr = (tmp == -INFINITY) ? -1 : 0;
            block_best(tmp, rr, red_s, red_r);
            F = (rr < 0) ? -INFINITY : tmp;
            (void)dummy;
        }
        // a_k: take-th best approximate candidate (keys are unique)
        uint64_t last_key = ~0ull;
        for (int64_t j = 0; j < take; ++j) {
            uint64_t best = 0;
            for (int e = threadIdx.x; e < M; e += RS_THREADS) {
                uint64_t key = cq[e];
                if (key && key < last_key && key > best) best = key;
            }
            for (int o = 16; o; o >>= 1) {
                uint64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
                best = ob > best ? ob : best;
            }
            if ((threadIdx.x & 31) == 0) red_r[threadIdx.x >> 5] = (int64_t)best;
            __syncthreads();
            best = 0;
            for (int w = 0; w < RS_THREADS / 32; ++w) best = ((uint64_t)red_r[w] > best) ? (uint64_t)red_r[w] : best;
            __syncthreads();
            last_key = best;
        }
        const double ak = (last_key && last_key != ~0ull) ? (double)key_score(last_key) : -INFINITY;
        const double cut = ak - 2.0 * a.err;
        if (threadIdx.x == 0) r_n = 0;
        __syncthreads();
        for (int e = threadIdx.x; e < M; e += RS_THREADS) {
            uint64_t key = cq[e];
            if (!key) continue;
            double s = key_score(key);
            if (s >= cut) {
                int slot = atomicAdd(&r_n, 1);
                if (slot < RS_MAX) {
                    r_row[slot] = key_row(key);
                    r_apx[slot] = s;
                }
            }
        }
        __syncthreads();
        const int nr = r_n;
        if (nr > RS_MAX) {
            // every true top-k row has approx >= a_k - 2E
            defer_query(a, q, cut);
            continue;
        }
        const float *qv = a.qp + q * (int64_t)a.dp8;
        {
            // one warp per candidate row, staged through shared memory (warp_einsum_dot):
            // a thread streaming its own 4-KB row set this kernel's time
            float *qs = rs_dyn;
            float *xs = rs_dyn + a.dp8 * (1 + (threadIdx.x >> 5));
            for (int j = threadIdx.x * 4; j < a.dp8; j += RS_THREADS * 4)
                *reinterpret_cast<float4 *>(qs + j) = __ldg(reinterpret_cast<const float4 *>(qv + j));
            __syncthreads();
            for (int e = threadIdx.x >> 5; e < nr; e += RS_THREADS / 32) {
                const double ex = warp_einsum_dot(a.x32 + r_row[e] * (int64_t)a.dp8, xs, qs, a.dp8, a.d);
                if ((threadIdx.x & 31) == 0) r_ex[e] = ex;
            }
        }
        if (threadIdx.x == 0) atomicAdd(&a.counters[1], nr);
        __syncthreads();
        // exact top-take of R, certificate, outputs
        double last_s = INFINITY;
        int64_t last_r = -1;
        bool ok = true;
        for (int64_t j = 0; j < take; ++j) {
            double bs = -INFINITY;
            int64_t br = -1;
            for (int e = threadIdx.x; e < nr; e += RS_THREADS) {
                double s = r_ex[e];
                int64_t r = r_row[e];
                bool after = (last_r < 0) || ranks_before(last_s, last_r, s, r);
                if (after && (br < 0 || ranks_before(s, r, bs, br))) { bs = s; br = r; }
            }
            block_best(bs, br, red_s, red_r);
            if (br < 0) { ok = false; break; }
            last_s = bs;
            last_r = br;
        }
        // every non-candidate scores <= F + E exactly; candidates outside R
        // score < a_k - E <= e_k
        if (!ok) {
            defer_query(a, q, cut);
            continue;
        }
        if (!(last_s > F + a.err)) {
            // exact ties (or near-ties) at the boundary: e_k(R) <= true e_k, so every
            // true top-k row, incl. lower-row ties, has approx >= e_k(R) - E
            defer_query(a, q, last_s - a.err);
            continue;
        }
        last_s = INFINITY;
        last_r = -1;
        for (int64_t j = 0; j < a.k; ++j) {
            const int64_t o = q * a.k + j;
            if (j >= take) {
                if (threadIdx.x == 0) {
                    a.rows[o] = -1;
                    if (a.raw) a.raw[o] = 0.0;
                    if (a.rep) a.rep[o] = 0.0;
                }
                continue;
            }
            double bs = -INFINITY;
            int64_t br = -1;
            for (int e = threadIdx.x; e < nr; e += RS_THREADS) {
                double s = r_ex[e];
                int64_t r = r_row[e];
                bool after = (last_r < 0) || ranks_before(last_s, last_r, s, r);
                if (after && (br < 0 || ranks_before(s, r, bs, br))) { bs = s; br = r; }
            }
            block_best(bs, br, red_s, red_r);
            double rep;
            finalize_hit(a.x32, a.dp8, a.d, qv, br, bs, &rep);
            if (threadIdx.x == 0) {
                a.rows[o] = br;
                if (a.raw) a.raw[o] = bs;
                if (a.rep) a.rep[o] = rep;
            }
            last_s = bs;
            last_r = br;
        }
        if (threadIdx.x == 0) a.count[q] = (int32_t)take;
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// collect pass (certificate failures): exact rescoring of every collected row
constexpr int CL_THREADS = 256;
constexpr int CL_CAP = 8192;  // collected rows per query kept; more -> exact rescan

__global__ void gather_q16_kernel(const __half *__restrict__ q16, int dp64, const int32_t *__restrict__ list,
                                  const int32_t *__restrict__ nlist, __half *__restrict__ out) {
    const int n = *nlist;
    const int64_t total = (int64_t)n * dp64;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / dp64;
        out[t] = q16[(int64_t)list[i] * dp64 + (t - i * dp64)];
    }
}

struct CollectArgs {
    const int32_t *clist;
    const int32_t *nlist;
    const int32_t *ccount;
    const int32_t *cbuf;
    int cap;
    int k;
    int64_t take;
    const int64_t *row_limit;
    const float *x32;
    int dp8, d;
    const float *qp;
    int64_t *rows;
    double *raw, *rep;
    int32_t *count;
    int32_t *counters;
    int32_t *fallback;
};

__global__ void __launch_bounds__(CL_THREADS) tc_collect_rescore_kernel(CollectArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    double *ex = reinterpret_cast<double *>(smem);                // [cap]
    int32_t *rw = reinterpret_cast<int32_t *>(ex + a.cap);        // [cap]
    __shared__ double red_s[CL_THREADS / 32];
    __shared__ int64_t red_r[CL_THREADS / 32];
    const int n = *a.nlist;
    for (int slot = blockIdx.x; slot < n; slot += gridDim.x) {
        const int64_t q = a.clist[slot];
        const int cnt = a.ccount[slot];
        if (cnt > a.cap) {  // too many rows above the threshold: exact fp64 rescan
            if (threadIdx.x == 0) {
                const int f = atomicAdd(&a.counters[0], 1);
                a.fallback[f] = (int32_t)q;
            }
            continue;
        }
        const int64_t take = a.row_limit ? min(a.take, max((int64_t)0, a.row_limit[q])) : a.take;
        const float *qv = a.qp + q * (int64_t)a.dp8;
        const int32_t *src = a.cbuf + (int64_t)slot * a.cap;
        for (int e = threadIdx.x; e < cnt; e += CL_THREADS) {
            const int32_t r = src[e];
            rw[e] = r;
            ex[e] = einsum_dot_f32(a.x32 + (int64_t)r * a.dp8, qv, a.d);
        }
        if (threadIdx.x == 0) atomicAdd(&a.counters[1], cnt);
        __syncthreads();
        double last_s = INFINITY;
        int64_t last_r = -1;
        for (int64_t j = 0; j < a.k; ++j) {
            const int64_t o = q * a.k + j;
            double bs = -INFINITY;
            int64_t br = -1;
            if (j < take) {
                for (int e = threadIdx.x; e < cnt; e += CL_THREADS) {
                    const double s = ex[e];
                    const int64_t r = rw[e];
                    const bool after = (last_r < 0) || ranks_before(last_s, last_r, s, r);
                    if (after && (br < 0 || ranks_before(s, r, bs, br))) { bs = s; br = r; }
                }
            }
            block_best(bs, br, red_s, red_r);
            if (br < 0) {
                if (threadIdx.x == 0) {
                    a.rows[o] = -1;
                    if (a.raw) a.raw[o] = 0.0;
                    if (a.rep) a.rep[o] = 0.0;
                }
                continue;
            }
            double rep;
            finalize_hit(a.x32, a.dp8, a.d, qv, br, bs, &rep);
            if (threadIdx.x == 0) {
                a.rows[o] = br;
                if (a.raw) a.raw[o] = bs;
                if (a.rep) a.rep[o] = rep;
            }
            last_s = bs;
            last_r = br;
        }
        if (threadIdx.x == 0) a.count[q] = (int32_t)take;
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2-D K-major tile map: `cols` elements of `elem_bytes` per row, boxes of
// box_cols x box_rows, SWIZZLE_128B (box_cols * elem_bytes must be 128)
int make_map_2d(CUtensorMap *m, const void *base, int64_t rows, int cols, int elem_bytes, int box_cols,
                int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) PR_FAIL(PR_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * elem_bytes};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapDataType dt = elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8;
    CUresult r = fn(m, dt, 2, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) PR_FAIL(PR_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return PR_OK;
}

static int make_map(CUtensorMap *m, const void *base, int64_t rows, int cols, int box_rows) {
    return make_map_2d(m, base, rows, cols, 2, TC_BLOCK_K, box_rows);
}

bool tc_eligible(int d, int64_t n, int k) { return k <= TC_KP && n > 0 && n < (int64_t)0xFFFFFFF0ll && d <= 8192; }
// the fp64 CUDA-core scan costs ~n*nq*d / 5.5e12 s; the tensor path has ~50 us of
// fixed cost (five launches + TMA descriptors) but scans ~250x faster per row
bool tc_worthwhile(int64_t n, int64_t nq) { return n >= 4096 && n * nq >= ((int64_t)1 << 22); }

double tc_error_bound(int d, int dp64) {
    // |fp16(x) - x| <= u|x| + eta  (u = 2^-11 round-to-nearest, eta = 2^-25 half the
    // fp16 subnormal spacing).  For unit vectors within the 1e-4 norm tolerance
    // (index.py:46) S = sum|q_i v_i| <= (1 + 1e-4)^2 and sum|x_i| <= sqrt(d)(1 + 1e-4):
    //   product error   <= (2u + u^2) S + eta (2 + 2u) sqrt(d) (1 + 1e-4) + d eta^2
    //   fp32 accumulate <= dp64 * 2^-23 * (sum of |fp16 products|)   (any order, truncation)
    const double u = std::ldexp(1.0, -11), eta = std::ldexp(1.0, -25);
    const double S = (1 + 1e-4) * (1 + 1e-4);
    const double prod = (2 * u + u * u) * S + eta * (2 + 2 * u) * std::sqrt((double)d) * (1 + 1e-4) + d * eta * eta;
    const double sum_abs = S * (1 + u) * (1 + u) + prod;
    const double acc = dp64 * std::ldexp(1.0, -23) * sum_abs;
    return (prod + acc) * 1.01 + 1e-9;
}

size_t tc_scratch_bytes(int64_t nq, int dp64, int64_t n, int k) {
    (void)k;
    int64_t nq_pad = round_up<int64_t>(nq, TC_BLOCK_M);
    int64_t ntiles = ceil_div<int64_t>(n, TC_BLOCK_N);
    int64_t maxsplit = std::min<int64_t>(ntiles, 4 * 148);
    return (size_t)nq_pad * dp64 * 2 * 2 + (size_t)nq_pad * maxsplit * TC_KP * 8 + (size_t)nq * (4 * 4 + 4 * CL_CAP) +
           16384;
}

int tc_make_store_map(TcStoreMap *m, const __half *x16, int64_t rows, int dp64) {
    return make_map(&m->map, x16, rows, dp64, TC_BLOCK_N);
}

int choose_nsplit_waves(int64_t qtiles, int64_t ntiles) {
    const int sms = sm_count();
    int best = 1;
    double best_eff = -1;
    int64_t lo = std::max<int64_t>(1, ceil_div<int64_t>(sms, qtiles));
    int64_t hi = std::min<int64_t>(ntiles, std::max<int64_t>(lo, 8 * sms / std::max<int64_t>(1, qtiles)));
    for (int64_t ns = lo; ns <= std::max(lo, hi); ++ns) {
        int64_t tps = ceil_div<int64_t>(ntiles, ns);
        int64_t real_ns = ceil_div<int64_t>(ntiles, tps);
        int64_t waves = ceil_div<int64_t>(qtiles * real_ns, sms);
        double eff = (double)(qtiles * ntiles) / (double)(waves * sms * tps);
        if (eff > best_eff + 1e-3) {
            best_eff = eff;
            best = (int)real_ns;
        }
        if (ns > lo && eff > 0.97) break;
    }
    return ntiles < 1 ? 1 : std::max(1, best);
}

// the same for work units of which `slots` run at once (clusters of several CTA pairs)
int choose_nsplit_slots(int64_t units, int64_t ntiles, int slots) {
    slots = std::max(1, slots);
    int best = 1;
    double best_eff = -1;
    const int64_t lo = std::max<int64_t>(1, ceil_div<int64_t>(slots, units));
    const int64_t hi = std::min<int64_t>(ntiles, std::max<int64_t>(lo, 8 * (int64_t)slots / std::max<int64_t>(1, units)));
    for (int64_t ns = lo; ns <= std::max(lo, hi); ++ns) {
        const int64_t tps = ceil_div<int64_t>(ntiles, ns);
        const int64_t real_ns = ceil_div<int64_t>(ntiles, tps);
        const int64_t waves = ceil_div<int64_t>(units * real_ns, slots);
        const double eff = (double)(units * ntiles) / (double)(waves * slots * tps);
        if (eff > best_eff + 1e-3) {
            best_eff = eff;
            best = (int)real_ns;
        }
        if (ns > lo && eff > 0.97) break;
    }
    return ntiles < 1 ? 1 : std::max(1, best);
}

static int choose_nsplit(int64_t qtiles, int64_t ntiles) {
    // persistent CTAs take items (qtile, split) round-robin: the busiest CTA owns
    // ceil(items / sms) items of tps tiles; pick the split count that minimises it
    // (ties -> fewer splits = fewer candidates to rescore)
    const int sms = sm_count();
    if (ntiles < 1) return 1;
    int64_t best_ns = 1;
    double best_cost = 1e300;
    const int64_t hi = std::min<int64_t>(ntiles, std::max<int64_t>(1, (int64_t)16 * sms / std::max<int64_t>(1, qtiles)));
    for (int64_t ns = 1; ns <= hi; ++ns) {
        const int64_t tps = ceil_div<int64_t>(ntiles, ns);
        const int64_t real_ns = ceil_div<int64_t>(ntiles, tps);
        const int64_t items = qtiles * real_ns;
        const double cost = (double)ceil_div<int64_t>(items, sms) * tps + 0.02 * real_ns;  // tiles on the busiest CTA
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best_ns = real_ns;
        }
    }
    return (int)best_ns;
}

int tc_search(TcSearch &s, Carve &cv, cudaStream_t st, pr_search_stats *stats) {
    const int64_t nq_pad = round_up<int64_t>(s.nq, TC_BLOCK_M);
    const int64_t qtiles = nq_pad / TC_BLOCK_M;
    const int64_t ntiles = ceil_div<int64_t>(s.n, TC_BLOCK_N);
    // default: one CTA per (query tile, split) item in whole waves; PR_TC_SCHEDULE=persistent
    // runs one CTA per SM taking items round-robin (measured no faster: scripts/ab_sched.py)
    const char *sched_env = getenv("PR_TC_SCHEDULE");
    const bool waves = !(sched_env && sched_env[0] == 'p');
    const int nsplit = waves ? choose_nsplit_waves(qtiles, ntiles) : choose_nsplit(qtiles, ntiles);
    const int tps = (int)ceil_div<int64_t>(ntiles, nsplit);
    __half *q16 = cv.take<__half>((size_t)nq_pad * s.dp64);
    uint64_t *cand = cv.take<uint64_t>((size_t)nq_pad * nsplit * TC_KP);
    s.fallback_list = cv.take<int32_t>((size_t)s.nq);

    {
        int64_t total = nq_pad * s.dp64;
        int grid = (int)std::min<int64_t>(ceil_div<int64_t>(total, 256), (int64_t)sm_count() * 16);
        ::pr::count_launch();
        queries_to_f16_kernel<<<grid, 256, 0, st>>>(s.qp, s.nq, s.dp8, s.d, nq_pad, s.dp64, q16);
        PR_LAUNCH_CHECK();
    }
    TcStoreMap qmap;
    int rc = make_map(&qmap.map, q16, nq_pad, s.dp64, TC_BLOCK_M);
    if (rc) return rc;

    static bool attr = false;
    if (!attr) {
        PR_CUDA(cudaFuncSetAttribute(tc_scan_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)tc_smem_bytes()));
        PR_CUDA(cudaFuncSetAttribute(tc_scan_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)tc_smem_bytes()));
        PR_CUDA(cudaFuncSetAttribute(tc_collect_rescore_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     CL_CAP * 12 + 1024));
        attr = true;
    }
    TcScanParams p{s.n, s.dp64 / TC_BLOCK_K, nsplit, tps, (int)ntiles, (int)qtiles, cand, s.row_limit, s.nq,
                   nullptr, nullptr, nullptr, nullptr, nullptr, 0};
    // persistent: one CTA per SM (1 CTA/SM by smem + TMEM), items assigned round-robin
    dim3 grid((unsigned)(waves ? qtiles * nsplit : std::min<int64_t>(qtiles * nsplit, sm_count())));
    ::pr::count_launch();
    if (s.ev_begin) PR_CUDA(cudaEventRecord(s.ev_begin, st));
    tc_scan_kernel<false><<<grid, TC_THREADS, tc_smem_bytes(), st>>>(qmap.map, s.store_map->map, p);
    PR_LAUNCH_CHECK();
    if (s.ev_end) PR_CUDA(cudaEventRecord(s.ev_end, st));

    PR_CUDA(cudaMemsetAsync(s.counters, 0, 4 * sizeof(int32_t), st));
    int32_t *clist = cv.take<int32_t>((size_t)s.nq);
    float *cthr = cv.take<float>((size_t)s.nq);
    int32_t *ccount = cv.take<int32_t>((size_t)s.nq);
    int32_t *cbuf = cv.take<int32_t>((size_t)s.nq * CL_CAP);
    __half *q16c = cv.take<__half>((size_t)nq_pad * s.dp64);
    RescoreArgs ra{cand, nsplit, s.nq, s.k, std::min<int64_t>(s.k, s.n), tc_error_bound(s.d, s.dp64), s.x32,
                   s.dp8, s.d, s.qp, s.rows, s.raw, s.rep, s.count, s.counters, s.fallback_list, s.row_limit,
                   clist, cthr};
    int rgrid = (int)std::min<int64_t>(s.nq, (int64_t)sm_count() * 16);
    ::pr::count_launch();
    const size_t rs_smem = (size_t)(1 + RS_THREADS / 32) * s.dp8 * sizeof(float);
    static bool rs_attr = false;
    if (!rs_attr) {
        PR_CUDA(cudaFuncSetAttribute(tc_rescore_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        rs_attr = true;
    }
    tc_rescore_kernel<<<rgrid, RS_THREADS, rs_smem, st>>>(ra);
    PR_LAUNCH_CHECK();

    // collect pass for certificate failures (device-sized list; tiles past it exit at once)
    PR_CUDA(cudaMemsetAsync(ccount, 0, (size_t)s.nq * sizeof(int32_t), st));
    {
        int g = (int)std::min<int64_t>(ceil_div<int64_t>(nq_pad * s.dp64, 256), (int64_t)sm_count() * 8);
        ::pr::count_launch();
        gather_q16_kernel<<<g, 256, 0, st>>>(q16, s.dp64, clist, s.counters + 2, q16c);
        PR_LAUNCH_CHECK();
    }
    TcStoreMap cmap;
    rc = make_map(&cmap.map, q16c, nq_pad, s.dp64, TC_BLOCK_M);
    if (rc) return rc;
    TcScanParams pc = p;
    pc.qmap = clist;
    pc.nlist = s.counters + 2;
    pc.thr = cthr;
    pc.ccount = ccount;
    pc.cbuf = cbuf;
    pc.cap = CL_CAP;
    ::pr::count_launch();
    tc_scan_kernel<true><<<grid, TC_THREADS, tc_smem_bytes(), st>>>(cmap.map, s.store_map->map, pc);
    PR_LAUNCH_CHECK();
    CollectArgs ca{clist, s.counters + 2, ccount, cbuf, CL_CAP, s.k, std::min<int64_t>(s.k, s.n), s.row_limit,
                   s.x32, s.dp8, s.d, s.qp, s.rows, s.raw, s.rep, s.count, s.counters, s.fallback_list};
    ::pr::count_launch();
    tc_collect_rescore_kernel<<<(unsigned)std::min<int64_t>(s.nq, (int64_t)sm_count() * 4), CL_THREADS,
                                CL_CAP * 12, st>>>(ca);
    PR_LAUNCH_CHECK();
    stats->nsplit = nsplit;
    return PR_OK;
}

}  // namespace pr
