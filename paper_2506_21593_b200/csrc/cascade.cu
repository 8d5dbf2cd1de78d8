// On-device cascade of a routed batch (reference: router.py:227-273 _probe, :275-364 route).
//
// The router probes its layers in probe_order() and the first hit serves the query.  For a
// batch, the vector layers (L4 adaptive memory, L5 retrieval) only need the queries that
// neither fast layer answered, so the batch hands ONE compacted miss list from the fast
// layers to the scans, on the device:
//
//   pr_cascade_gate    L1 (fixed-KV probe result, OR an earlier in-window write of the same
//                      text) and L2 (semantic-cache top-1 >= threshold, caches.py:140) per
//                      query; a query blocked by a fast layer probed before the vector
//                      layers leaves the list; the survivors are compacted in query order
//                      (block-wide prefix sum) into list / count / slot — no host round trip.
//                      The knowledge-base scan then runs on the list (pr_index_search_list).
//   pr_recall_gate     L3 (memory recall, generation.py:203-224) when the backend's recall
//                      table is a device hash table: accept iff the question is in the table,
//                      its confidence >= the recall threshold and its answer is non-empty
//                      (the confidence array holds -1 for an empty answer).  Its output
//                      feeds pr_cascade_gate like the L1/L2 outcomes.
//   pr_cascade_seeds   the AKM-hit guard: the superset of seeds (top seed_k KB rows) every
//                      earlier listed query could settle into the AKM before a later query
//                      probes it (knowledge.py:217-228), deduplicated by KB row in first-
//                      occurrence order (a KB-sized mark array, atomicMin of positions), with
//                      each listed query's visible prefix length (row limit of the guard scan).
//
// Both run as one CTA (1024 threads) over the batch: the batch is a few thousand queries
// and tens of thousands of seed rows; the cost is a few microseconds, and one launch
// avoids any grid-wide synchronisation.
#include <algorithm>

#include "common.cuh"

namespace pr {

constexpr int CG_THREADS = 1024;

// exclusive block scan of one int per thread; returns the block total
__device__ __forceinline__ int block_exclusive_scan(int v, int *warp_sums, int &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < nwarp ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nwarp) warp_sums[lane] = w;
    }
    __syncthreads();
    const int base = warp > 0 ? warp_sums[warp - 1] : 0;
    total = warp_sums[nwarp - 1];
    __syncthreads();
    return base + x - v;
}

struct GateArgs {
    int64_t B;
    const uint8_t *kv_hit;    // [B] pre-batch fixed-KV probe (nullable: L1 absent)
    const uint8_t *rep;       // [B] text written earlier in the window (nullable)
    const int32_t *sc_count;  // [B] semantic-cache top-1 count (nullable: L2 absent)
    const double *sc_score;   // [B] reported top-1 score
    double sc_threshold;
    const uint8_t *l3_hit;     // [B] accepted recall (nullable: L3 absent or not on the device)
    int l1_blocks, l2_blocks, l3_blocks;  // the layer is probed before the vector layers
    uint8_t *l1, *l2;          // [B] out
    int32_t *list;             // [B] out: queries that reach the vector layers, in order
    int32_t *nlist;            // [1] out
    int32_t *slot;             // [B] out: position in list or -1
};

__global__ void __launch_bounds__(CG_THREADS) cascade_gate_kernel(GateArgs a) {
    __shared__ int warp_sums[32];
    int base = 0;
    for (int64_t c0 = 0; c0 < a.B; c0 += blockDim.x) {
        const int64_t j = c0 + threadIdx.x;
        int keep = 0;
        if (j < a.B) {
            const bool h1 = a.kv_hit && (a.kv_hit[j] || (a.rep && a.rep[j]));
            const bool h2 = a.sc_count && a.sc_count[j] > 0 && a.sc_score[j] >= a.sc_threshold;
            a.l1[j] = h1;
            a.l2[j] = h2;
            const bool h3 = a.l3_hit && a.l3_hit[j];
            keep = !((h1 && a.l1_blocks) || (h2 && a.l2_blocks) || (h3 && a.l3_blocks));
        }
        int total;
        const int pos = block_exclusive_scan(keep, warp_sums, total);
        if (j < a.B) {
            a.slot[j] = keep ? base + pos : -1;
            if (keep) a.list[base + pos] = (int32_t)j;
        }
        base += total;
    }
    if (threadIdx.x == 0) *a.nlist = base;
}

__global__ void recall_gate_kernel(int64_t n, const int64_t *__restrict__ vals, const uint8_t *__restrict__ hit,
                                   const double *__restrict__ conf, int64_t nconf, double threshold,
                                   uint8_t *__restrict__ out) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = vals[j];
        out[j] = hit[j] && v >= 0 && v < nconf && conf[v] >= threshold;
    }
}

struct SeedArgs {
    // previous span (its listed queries' seeds were not settled when this span was launched)
    const int64_t *prev_rows;  // [prev_max, sk] (nullable)
    const int32_t *prev_cnt;   // [prev_max]
    const int32_t *prev_n;     // [1] live listed queries
    // this span
    const int64_t *rows;  // [nq_max, sk]
    const int32_t *cnt;   // [nq_max]
    const int32_t *n;     // [1]
    int sk;
    int32_t *mark;       // [KB rows] INT_MAX between calls (restored on exit)
    int64_t *out_rows;   // [(prev_max + nq_max) * sk] deduplicated seed rows, junk (row 0) past *nout
    int64_t out_max;
    int32_t *nout;       // [1]
    int64_t *before;     // [nq_max] deduplicated seeds visible to listed query i
};

// sequence position p -> (row) over prev then cur, each listed query contributing cnt rows
__device__ __forceinline__ int64_t seq_row(const SeedArgs &a, int np, int64_t p) {
    const int64_t pp = (int64_t)np * a.sk;
    if (p < pp) return a.prev_rows[p];
    return a.rows[p - pp];
}
__device__ __forceinline__ bool seq_valid(const SeedArgs &a, int np, int64_t p) {
    const int64_t pp = (int64_t)np * a.sk;
    if (p < pp) return (p % a.sk) < a.prev_cnt[p / a.sk];
    const int64_t q = p - pp;
    return (q % a.sk) < a.cnt[q / a.sk];
}

__global__ void __launch_bounds__(CG_THREADS) cascade_seeds_kernel(SeedArgs a) {
    __shared__ int warp_sums[32];
    const int np = a.prev_rows ? max(0, *a.prev_n) : 0;
    const int nc = max(0, *a.n);
    const int64_t total = (int64_t)(np + nc) * a.sk;
    // 1) first occurrence of every KB row in sequence order
    for (int64_t p = threadIdx.x; p < total; p += blockDim.x)
        if (seq_valid(a, np, p)) atomicMin(&a.mark[seq_row(a, np, p)], (int32_t)p);
    __syncthreads();
    // 2) compact first occurrences; before[i] = firsts strictly before listed query i's seeds
    int base = 0;
    const int64_t cur0 = (int64_t)np * a.sk;
    for (int64_t c0 = 0; c0 < total; c0 += blockDim.x) {
        const int64_t p = c0 + threadIdx.x;
        int first = 0;
        int64_t r = 0;
        if (p < total && seq_valid(a, np, p)) {
            r = seq_row(a, np, p);
            first = a.mark[r] == (int32_t)p;
        }
        int tot;
        const int pos = block_exclusive_scan(first, warp_sums, tot);
        if (first) a.out_rows[base + pos] = r;
        if (p < total && p >= cur0 && (p - cur0) % a.sk == 0) a.before[(p - cur0) / a.sk] = base + pos;
        base += tot;
    }
    __syncthreads();
    // 3) restore the marks; pad the row list with a valid junk row (never visible)
    for (int64_t p = threadIdx.x; p < total; p += blockDim.x)
        if (seq_valid(a, np, p)) a.mark[seq_row(a, np, p)] = INT32_MAX;
    for (int64_t p = base + threadIdx.x; p < a.out_max; p += blockDim.x) a.out_rows[p] = 0;
    if (threadIdx.x == 0) *a.nout = base;
}

// L4 guard row limit of query j: the deduplicated seeds visible to its list position
__global__ void guard_limit_kernel(int64_t B, const int32_t *slot, const int64_t *before, int64_t *lim) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < B; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t s = slot[j];
        lim[j] = s >= 0 ? before[s] : 0;
    }
}

struct PackArgs {
    int64_t B;
    int seed_k;
    const uint8_t *l1, *l2;
    const int32_t *slot;
    const int64_t *sc_rows;  // [B] top-1 rows of L2 (NULL: not probed)
    const int64_t *kv_val;   // NULL: not probed
    const int32_t *kb_cnt;
    const uint8_t *l3;
    const int64_t *l3_val;
    const int32_t *nlist;
    const int64_t *kb_rows;
    int probe_l4;
    double thr;
    const int32_t *a_cnt;  // adaptive memory top-1 (NULL: empty)
    const double *a_rep;
    const int32_t *g_cnt;  // guard top-1
    const double *g_rep;
    int64_t *out;
};

// the span's packed read-back, and l4[j] = listed && (AKM top-1 >= thr || guard top-1 >= thr)
__global__ void cascade_pack_kernel(PackArgs a) {
    const int64_t B = a.B, nr = B * a.seed_k;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < B + nr; t += (int64_t)gridDim.x * blockDim.x) {
        if (t >= B) {
            a.out[9 * B + 1 + (t - B)] = a.kb_rows[t - B];
            continue;
        }
        const int64_t j = t;
        const int32_t s = a.slot[j];
        bool l4 = false;
        if (a.probe_l4 && s >= 0) {
            l4 = (a.a_cnt && a.a_cnt[j] > 0 && a.a_rep[j] >= a.thr) || (a.g_cnt[j] > 0 && a.g_rep[j] >= a.thr);
        }
        int64_t *o = a.out;
        o[j] = a.l1[j];
        o[B + j] = a.l2[j];
        o[2 * B + j] = s;
        o[3 * B + j] = l4;
        o[4 * B + j] = a.sc_rows ? a.sc_rows[j] : -1;
        o[5 * B + j] = a.kv_val ? a.kv_val[j] : -1;
        o[6 * B + j] = a.kb_cnt[j];
        o[7 * B + j] = a.l3 ? (int64_t)a.l3[j] : -1;
        o[8 * B + j] = a.l3_val ? a.l3_val[j] : -1;
        if (j == 0) o[9 * B] = *a.nlist;
    }
}

// carve of the composite call's scratch (256-byte aligned pieces)
struct RouteCarve {
    char *p;
    int64_t used = 0;
    template <class T>
    T *take(int64_t n) {
        T *r = reinterpret_cast<T *>(p ? p + used : nullptr);
        used += ((int64_t)sizeof(T) * std::max<int64_t>(n, 1) + 255) & ~(int64_t)255;
        return r;
    }
};

}  // namespace pr

using namespace pr;

extern "C" {

int pr_cascade_gate(int64_t B, const uint8_t *d_kv_hit, const uint8_t *d_rep, const int32_t *d_sc_count,
                    const double *d_sc_score, double sc_threshold, const uint8_t *d_l3_hit, int l1_blocks,
                    int l2_blocks, int l3_blocks, uint8_t *d_l1, uint8_t *d_l2, int32_t *d_list, int32_t *d_nlist,
                    int32_t *d_slot, void *stream) {
    if (B < 0 || !d_l1 || !d_l2 || !d_list || !d_nlist || !d_slot || (d_sc_count && !d_sc_score))
        PR_FAIL(PR_ERR_BAD_ARG, "bad cascade_gate");
    GateArgs a{B, d_kv_hit, d_rep, d_sc_count, d_sc_score, sc_threshold, d_l3_hit, l1_blocks, l2_blocks, l3_blocks,
               d_l1, d_l2, d_list, d_nlist, d_slot};
    ::pr::count_launch();
    cascade_gate_kernel<<<1, CG_THREADS, 0, as_stream(stream)>>>(a);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

int pr_recall_gate(int64_t n, const int64_t *d_vals, const uint8_t *d_hit, const double *d_conf, int64_t nconf,
                   double threshold, uint8_t *d_out, void *stream) {
    if (n < 0 || nconf < 0 || (n > 0 && (!d_vals || !d_hit || !d_out)) || (nconf > 0 && !d_conf))
        PR_FAIL(PR_ERR_BAD_ARG, "bad recall_gate");
    if (!(threshold >= 0.0 && threshold <= 1.0)) PR_FAIL(PR_ERR_BAD_ARG, "recall threshold outside [0, 1]");
    if (n == 0) return PR_OK;
    ::pr::count_launch();
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((n + threads - 1) / threads, 148 * 8);
    recall_gate_kernel<<<blocks, threads, 0, as_stream(stream)>>>(n, d_vals, d_hit, d_conf, nconf, threshold, d_out);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

int pr_cascade_mark_init(int32_t *d_mark, int64_t n, void *stream) {
    if (n < 0 || (n > 0 && !d_mark)) PR_FAIL(PR_ERR_BAD_ARG, "bad mark_init");
    if (n == 0) return PR_OK;
    PR_CUDA(cudaMemsetAsync(d_mark, 0x7f, (size_t)n * sizeof(int32_t), as_stream(stream)));  // >= INT32_MAX - 0x808080
    return PR_OK;
}

int pr_cascade_seeds(const int64_t *d_prev_rows, const int32_t *d_prev_cnt, const int32_t *d_prev_n,
                     const int64_t *d_rows, const int32_t *d_cnt, const int32_t *d_n, int seed_k, int32_t *d_mark,
                     int64_t *d_out_rows, int64_t out_max, int32_t *d_nout, int64_t *d_before, void *stream) {
    if (seed_k < 1 || !d_rows || !d_cnt || !d_n || !d_mark || !d_out_rows || !d_nout || !d_before ||
        (d_prev_rows && (!d_prev_cnt || !d_prev_n)))
        PR_FAIL(PR_ERR_BAD_ARG, "bad cascade_seeds");
    SeedArgs a{d_prev_rows, d_prev_cnt, d_prev_n, d_rows, d_cnt, d_n, seed_k, d_mark, d_out_rows, out_max, d_nout,
               d_before};
    ::pr::count_launch();
    cascade_seeds_kernel<<<1, CG_THREADS, 0, as_stream(stream)>>>(a);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

int64_t pr_cascade_route_scratch(int64_t B, int seed_k, int64_t prev_B) {
    if (B < 0 || seed_k < 1 || prev_B < 0) return -1;
    RouteCarve c{nullptr};
    c.take<uint8_t>(B), c.take<int64_t>(B);                    // kv hit / value
    c.take<uint8_t>(B), c.take<uint8_t>(B), c.take<int32_t>(B);  // l1, l2, list
    for (int r = 0; r < 3; ++r) c.take<int64_t>(B), c.take<double>(B), c.take<double>(B), c.take<int32_t>(B);
    c.take<int64_t>((prev_B + B) * seed_k), c.take<int32_t>(1), c.take<int64_t>(B), c.take<int64_t>(B);
    return c.used;
}

int pr_cascade_route(const pr_cascade_span *s, void *d_scratch, int64_t scratch_bytes, void *stream) {
    if (!s || s->B < 0 || s->seed_k < 1 || !s->kb || !s->d_rep || !s->d_kb_rows || !s->d_kb_raw || !s->d_kb_rep ||
        !s->d_kb_cnt || !s->d_nlist || !s->d_slot || !s->d_packed || (s->B > 0 && !s->d_vec) ||
        (s->kv && (!s->d_text || !s->d_text_off)) || (s->sc && !s->d_sc_limit) ||
        (s->probe_l4 && (!s->guard || !s->d_mark || (s->akm_rows > 0 && !s->akm))) ||
        (s->d_prev_rows && (!s->d_prev_cnt || !s->d_prev_n)))
        PR_FAIL(PR_ERR_BAD_ARG, "bad cascade_route");
    const int64_t B = s->B;
    const int sk = s->seed_k;
    const int64_t prev_B = s->d_prev_rows ? s->prev_B : 0;
    const int64_t need = pr_cascade_route_scratch(B, sk, prev_B);
    if (!d_scratch || scratch_bytes < need) PR_FAIL(PR_ERR_BAD_ARG, "cascade_route scratch too small");
    cudaStream_t st = as_stream(stream);
    RouteCarve c{static_cast<char *>(d_scratch)};
    uint8_t *kv_hit = c.take<uint8_t>(B);
    int64_t *kv_val = c.take<int64_t>(B);
    uint8_t *l1 = c.take<uint8_t>(B), *l2 = c.take<uint8_t>(B);
    int32_t *lst = c.take<int32_t>(B);
    int64_t *rows[3];
    double *raw[3], *rep[3];
    int32_t *cnt[3];  // 0: semantic cache, 1: adaptive memory, 2: guard
    for (int r = 0; r < 3; ++r)
        rows[r] = c.take<int64_t>(B), raw[r] = c.take<double>(B), rep[r] = c.take<double>(B), cnt[r] = c.take<int32_t>(B);
    const int64_t out_max = (prev_B + B) * sk;
    int64_t *out_rows = c.take<int64_t>(out_max);
    int32_t *nout = c.take<int32_t>(1);
    int64_t *before = c.take<int64_t>(B), *lim = c.take<int64_t>(B);
    int rc;
    if (B == 0) return PR_OK;
    // L1, L2: the fast layers' probes
    if (s->kv && (rc = pr_kv_get_text(s->kv, s->d_text, s->d_text_off, B, kv_val, kv_hit, stream)) != PR_OK) return rc;
    if (s->sc && (rc = pr_index_search_floor(s->sc, s->d_vec, B, 1, s->mode, s->d_sc_limit, s->sc_threshold, rows[0],
                                             raw[0], rep[0], cnt[0], stream)) != PR_OK)
        return rc;
    // gate + the compacted miss list, then the knowledge-base scan of the listed queries
    if ((rc = pr_cascade_gate(B, s->kv ? kv_hit : nullptr, s->d_rep, s->sc ? cnt[0] : nullptr, s->sc ? rep[0] : nullptr,
                              s->sc_threshold, s->d_l3_hit, s->l1_blocks, s->l2_blocks, s->l3_blocks, l1, l2, lst,
                              s->d_nlist, s->d_slot, stream)) != PR_OK)
        return rc;
    const int64_t hint = std::min<int64_t>(B, std::max<int64_t>(1, s->nlist_hint));
    if ((rc = pr_index_search_list(s->kb, s->d_vec, lst, s->d_nlist, B, hint, sk, s->mode, nullptr, s->d_kb_rows,
                                   s->d_kb_raw, s->d_kb_rep, s->d_kb_cnt, stream)) != PR_OK)
        return rc;
    // L4 guard: the adaptive memory as it is, and the seeds settled before each listed query
    const bool akm_on = s->probe_l4 && s->akm_rows > 0;
    if (s->probe_l4) {
        if (akm_on && (rc = pr_index_search_floor(s->akm, s->d_vec, B, 1, s->mode, nullptr, s->akm_threshold, rows[1],
                                                  raw[1], rep[1], cnt[1], stream)) != PR_OK)
            return rc;
        if ((rc = pr_cascade_seeds(s->d_prev_rows, s->d_prev_cnt, s->d_prev_n, s->d_kb_rows, s->d_kb_cnt, s->d_nlist, sk,
                                   s->d_mark, out_rows, out_max, nout, before, stream)) != PR_OK)
            return rc;
        if ((rc = pr_index_append_from(s->guard, s->kb, out_rows, out_max, stream)) != PR_OK) return rc;
        ::pr::count_launch();
        guard_limit_kernel<<<(unsigned)std::min<int64_t>((B + 255) / 256, 148 * 4), 256, 0, st>>>(B, s->d_slot, before,
                                                                                                 lim);
        PR_LAUNCH_CHECK();
        if ((rc = pr_index_search_floor(s->guard, s->d_vec, B, 1, s->mode, lim, s->akm_threshold, rows[2], raw[2],
                                        rep[2], cnt[2], stream)) != PR_OK)
            return rc;
    }
    PackArgs a{B, sk, l1, l2, s->d_slot, s->sc ? rows[0] : nullptr, s->kv ? kv_val : nullptr, s->d_kb_cnt,
               s->d_l3_hit, s->d_l3_val, s->d_nlist, s->d_kb_rows, s->probe_l4, s->akm_threshold,
               akm_on ? cnt[1] : nullptr, akm_on ? rep[1] : nullptr, cnt[2], rep[2], s->d_packed};
    ::pr::count_launch();
    cascade_pack_kernel<<<(unsigned)std::min<int64_t>((B * (1 + sk) + 255) / 256, 148 * 8), 256, 0, st>>>(a);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

}  // extern "C"
