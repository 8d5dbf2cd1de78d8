/*
 * pentarag.h — C ABI of the B200-native PentaRAG fast-routing hot path
 * (libpentarag.so, built from paper_2506_21593_b200/csrc).
 *
 * Plain pointers and sizes only: no torch, no C++ types.  Every `d_` pointer
 * is DEVICE memory owned by the caller; every call is ordered on the caller's
 * `stream` (a cudaStream_t passed as void*, NULL = legacy default stream).
 * Store buffers (the rows behind an index, the KV slot table) are owned by
 * the library and released by the matching *_destroy call.
 *
 * Each entry point names the reference interface it replaces; reference
 * paths are relative to /root/reference/pkg/src/ragcascade/.  The Python
 * host layer (paper_2506_21593_b200/) binds these with ctypes and keeps the
 * reference's duck-typed surface (FlatIndex, FixedKVCache, SemanticCache,
 * MainKnowledgeBase, AdaptiveKnowledgeMemory, CascadeRouter).
 *
 * Errors: every int-returning function returns PR_OK (0) or a negative
 * status; pr_last_error() gives a thread-local message.  The host layer maps
 * statuses onto the reference exceptions (errors.py:10-130).  No C++
 * exception crosses this boundary.  Handles are not thread-safe: the host
 * layer serialises calls per handle, as the reference serialises per index
 * (index.py:80 RLock).
 */
#ifndef PENTARAG_H
#define PENTARAG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define PR_OK 0
#define PR_ERR_BAD_ARG (-1)        /* ValueError (index.py:161-162, knowledge.py:77-80) */
#define PR_ERR_INVALID_VECTOR (-2) /* InvalidVector (errors.py:34-37) */
#define PR_ERR_EMPTY (-3)          /* EmptyKnowledgeBase (errors.py:46-49) */
#define PR_ERR_CUDA (-4)           /* CUDA runtime/driver failure */
#define PR_ERR_NOMEM (-5)          /* device allocation failed */
#define PR_ERR_UNSUPPORTED (-6)    /* not built for / not running on sm_100a */

/* ---- search modes ------------------------------------------------------ */
#define PR_SEARCH_AUTO 0   /* int8 tensor-core scan for stores >= 512k rows (dim <= 2048), fp16 tensor-core
                              scan for smaller stores that still pay for a scan, else exact */
#define PR_SEARCH_EXACT 1  /* fp64 einsum-order scan of every row          */
#define PR_SEARCH_TENSOR 2 /* tcgen05 fp16 scan + certified fp64 rescoring */
#define PR_SEARCH_TENSOR_I8 3 /* tcgen05 int8 scan with per-row error bounds + fp64 rescoring of the
                                 complete candidate set (same results, ~1.6x the scan rate) */

typedef struct pr_index pr_index;
typedef struct pr_kv pr_kv;

/* Per-call counters of the last pr_index_search on a handle (host-side copy;
 * reading them synchronises the handle's last search stream). */
typedef struct pr_search_stats {
    int64_t queries;        /* queries in the call                              */
    int64_t tensor_queries; /* went through the tcgen05 scan                    */
    int64_t fallback;       /* failed the certificate -> exact fp64 rescan      */
    int64_t candidates;     /* rows rescored in fp64 after the tensor scan      */
    int32_t nsplit;         /* row splits used by the scan grid                 */
    int32_t path;           /* PR_SEARCH_EXACT, PR_SEARCH_TENSOR or _TENSOR_I8  */
    int64_t collected;      /* failed the certificate -> tcgen05 collect pass   */
    int64_t appended;       /* int8 path: rows appended by the scan (pre-filter) */
} pr_search_stats;

/* ---- library ------------------------------------------------------------ */
const char *pr_last_error(void);
int pr_abi_version(void);
/* Device properties of the current device; fails with PR_ERR_UNSUPPORTED if
 * it is not compute capability 10.0 (the only target this library is built for). */
int pr_device_info(int *sm_count, int *cc_major, int *cc_minor);

/* ---- vector contract: index.py:58-70 (_coerce_vector), embedding.py:52-67 -
 * d_bad[i] = 1 if row i has a NaN/Inf or | ||v||_2 - 1 | > tol (fp64 norm). */
int pr_check_unit(const float *d_vecs, int64_t n, int dim, double tol, uint8_t *d_bad, void *stream);

/* ---- flat index store: index.py:73-153 (FlatIndex storage, insert/extend) --
 * Rows are kept three times: fp32 (the exact copy every score is computed
 * from, as _vectors32/_vectors64 at index.py:82-83,144-145), fp16 (the
 * certified tensor-core scan copy) and int8 with a per-row scale and a
 * rounded-up quantisation-error norm (the int8 tensor-core scan copy).  Row i is the i-th inserted entry id, so row order is the
 * reference's insertion (tie-break) order. */
int pr_index_create(int dim, int64_t capacity, uint32_t flags, pr_index **out);
int pr_index_destroy(pr_index *h);
int64_t pr_index_count(const pr_index *h);
int pr_index_dim(const pr_index *h);
int pr_index_reserve(pr_index *h, int64_t capacity, void *stream);
/* append n rows (d_vecs is [n, dim] fp32, row-major) — a new entry id (index.py:134-141) */
int pr_index_append(pr_index *h, const float *d_vecs, int64_t n, void *stream);
/* overwrite rows in place — an existing entry id keeps its row (index.py:142-145) */
int pr_index_update_rows(pr_index *h, const int64_t *d_rows, const float *d_vecs, int64_t n, void *stream);
/* FlatIndex.clear (index.py:191-196): forget every row, keep the buffers */
int pr_index_clear(pr_index *h);
/* keep only the first n rows (used by rebuild-style eviction, caches.py:166-181) */
int pr_index_truncate(pr_index *h, int64_t n);
/* copy rows [row0, row0+n) out as fp32 [n, dim] (FlatIndex.vector, index.py:111-114) */
int pr_index_read_rows(const pr_index *h, int64_t row0, int64_t n, float *d_out, void *stream);
/* append rows gathered from another index with the same dim (AKM settle from
 * KB rows, knowledge.py:217-228) */
int pr_index_append_from(pr_index *h, const pr_index *src, const int64_t *d_src_rows, int64_t n, void *stream);

/* ---- search: index.py:155-189 (FlatIndex.search) ------------------------
 * For each of nq queries (d_q is [nq, dim] fp32): top-min(k, count) rows by
 * (score desc, row asc), score = np.einsum("ij,j->i") in fp64 bit-for-bit.
 *   d_rows     int64 [nq, k]  row index, -1 past d_count
 *   d_raw      fp64  [nq, k]  einsum score (may be NULL)
 *   d_reported fp64  [nq, k]  SearchHit.score: self-snap + clamp (may be NULL)
 *   d_count    int32 [nq]     min(k, count)
 * k must be >= 1 (PR_ERR_BAD_ARG otherwise). An empty index gives count 0. */
int pr_index_search(pr_index *h, const float *d_q, int64_t nq, int k, uint32_t mode, int64_t *d_rows,
                    double *d_raw, double *d_reported, int32_t *d_count, void *stream);
/* As pr_index_search, with a per-query visibility limit: query q only sees
 * rows [0, d_row_limit[q]) (NULL = all rows).  This is the store "as of"
 * an earlier point of a sequential stream: the batched cascade uses it so
 * query j sees exactly the rows written back by queries i < j. */
int pr_index_search_ex(pr_index *h, const float *d_q, int64_t nq, int k, uint32_t mode, const int64_t *d_row_limit,
                       int64_t *d_rows, double *d_raw, double *d_reported, int32_t *d_count, void *stream);
/* As pr_index_search_ex for callers that only act on scores >= floor (the semantic-cache and
 * adaptive-memory thresholds, caches.py:140, knowledge.py:203-205): every result whose exact
 * score is >= min(floor, 1 - 1e-6) is exact and in its exact rank among such rows (self-snap and
 * clamp as pr_index_search); rows below that may be missing or out of order, and d_count
 * counts the rows reported.  A caller deciding `count > 0 && reported[0] >= floor` gets
 * exactly the full search's decision and, on a hit, its row and score.  The int8 scan then
 * starts from the floor as its bound (no pilot), so a threshold lookup is one scan. */
int pr_index_search_floor(pr_index *h, const float *d_q, int64_t nq, int k, uint32_t mode, const int64_t *d_row_limit,
                          double floor, int64_t *d_rows, double *d_raw, double *d_reported, int32_t *d_count,
                          void *stream);
/* The miss-list hand-off of the on-device cascade: search the queries a device-side
 * compaction selected, without reading the list back.  Listed position i searches
 * d_q[d_list[i]] (d_q is [*, dim] fp32) for i < *d_nlist (DEVICE int32); outputs are
 * [nq_max, k] in list order, positions past the live count are left undefined.
 * nq_hint (host) is the expected live count: the tensor-core grid is shaped for it (any
 * count <= nq_max is correct).  d_row_limit, if given, is per listed position.  The int8
 * and exact paths skip the dead positions; the fp16 path (small stores) scans nq_max. */
int pr_index_search_list(pr_index *h, const float *d_q, const int32_t *d_list, const int32_t *d_nlist, int64_t nq_max,
                         int64_t nq_hint, int k, uint32_t mode, const int64_t *d_row_limit, int64_t *d_rows,
                         double *d_raw, double *d_reported, int32_t *d_count, void *stream);
int pr_index_last_stats(pr_index *h, pr_search_stats *out);
/* Record CUDA events around the dominant scan kernel of every search (the
 * tcgen05 scan, or the exact scan on the exact path); pr_index_scan_time
 * synchronises, returns the summed kernel time and the number of timed
 * launches since the previous call, and resets. */
int pr_index_set_timing(pr_index *h, int enable);
int pr_index_scan_time(pr_index *h, double *total_ms, int64_t *launches);
/* number of kernels this library has launched in this process */
long long pr_launch_count(void);

/* Row-sharded stores (sharded.py): d_out[i] = the stored fp32 row d_rows[i] - row_offset
 * when this shard holds it (0 <= d_rows[i] - row_offset < count), else all zeros — a SUM
 * all-reduce of the int32 bit patterns over the shards assembles the exact rows (the AKM
 * settle and the cascade's seed guard copy knowledge-base rows, knowledge.py:217-228). */
int pr_index_gather_rows(const pr_index *h, const int64_t *d_rows, int64_t n, int64_t row_offset, float *d_out,
                         void *stream);
/* Merge per-shard top-k lists into the global top-k (the NCCL all-gather
 * merge of a row-sharded store).  d_rows/d_raw are [nshard, nq, k] with
 * global row ids; d_count is [nshard, nq].  Output as pr_index_search, with
 * d_snap [nshard, nq, k] (1 where the shard saw a bit-identical row) used to
 * produce d_reported. */
int pr_merge_shards(const int64_t *d_rows, const double *d_raw, const uint8_t *d_snap, const int32_t *d_count,
                    int nshard, int64_t nq, int k, int64_t *d_out_rows, double *d_out_raw,
                    double *d_out_reported, int32_t *d_out_count, void *stream);
/* d_snap[q, j] = 1 iff row d_rows[q, j] of h is element-wise equal to query q
 * and d_raw > 1 - 1e-6 (the self-snap predicate, index.py:180). */
int pr_index_snap_flags(const pr_index *h, const float *d_q, int64_t nq, int k, const int64_t *d_rows,
                        const double *d_raw, const int32_t *d_count, int64_t row_offset, uint8_t *d_snap,
                        void *stream);

/* ---- fixed KV cache: caches.py:45-101 (FixedKVCache) --------------------
 * Keys are the UTF-8 bytes of the query text, compared BYTE-EXACT like the
 * reference dict (caches.py:57-65): a linear-probing array of
 * 32-byte slots {16-byte key prefix, length|value, 32-bit tag, record index},
 * one 256-bit load per probe step, keys longer than 16 bytes completed by a
 * 32-byte aligned record; a hit is confirmed against the stored key bytes, so a
 * hash collision can never serve another key's answer.  Key batches are a UTF-8
 * arena d_bytes + int64 offsets d_off[n+1] (key i = d_bytes[d_off[i]..d_off[i+1])).
 * Values are non-negative int64 write sequence numbers: a larger value is a
 * later write, so puts of one key in one batch resolve last-write-wins
 * (caches.py:67-74).  The *_owned variants act only on the keys a shard owns
 * (owner = pr_kv_owner, bits disjoint from the slot index); the other keys
 * are skipped (get: value -1, hit 0) without touching the table. */
int pr_kv_create(int64_t capacity, pr_kv **out);
/* flags: PR_KV_WEAK_HASH keeps 2 tag bits and 4 home slots, so distinct keys collide
 * on purpose — a test hook for the byte-exact confirmation; never used by the product */
#define PR_KV_WEAK_HASH 1u
int pr_kv_create_ex(int64_t capacity, uint32_t flags, pr_kv **out);
int pr_kv_destroy(pr_kv *h);
/* hash n keys -> d_fp[2i] = tag (32-bit, top bit set; also picks the shard owner),
 * d_fp[2i+1] = home-slot hash (32-bit, independent chain) */
int pr_fingerprint(const uint8_t *d_bytes, const int64_t *d_off, int64_t n, uint64_t *d_fp, void *stream);
void pr_fingerprint_host(const uint8_t *bytes, int64_t len, uint64_t out[2]);
/* shard owner of each key for a table hash-partitioned over `world` ranks */
int pr_kv_owner(const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int world, int32_t *d_owner, void *stream);
/* upsert (caches.py:67-77); nbytes = d_off[n] - d_off[0] (reserves record space without a device read) */
int pr_kv_put_text(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int64_t nbytes,
                   const int64_t *d_vals, void *stream);
int pr_kv_put_text_owned(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int64_t nbytes,
                         const int64_t *d_vals, int rank, int world, void *stream);
/* d_vals[i] = value or -1; d_hit[i] = 1/0 (hit/miss, caches.py:57-65) */
int pr_kv_get_text(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int64_t *d_vals,
                   uint8_t *d_hit, void *stream);
int pr_kv_get_text_owned(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int rank, int world,
                         int64_t *d_vals, uint8_t *d_hit, void *stream);
/* remove keys (LRU eviction, caches.py:75-77) */
int pr_kv_erase_text(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, void *stream);
int pr_kv_clear(pr_kv *h, void *stream);
int64_t pr_kv_size(pr_kv *h, void *stream); /* live keys (synchronises `stream`) */
int64_t pr_kv_capacity(pr_kv *h);           /* slots */
/* device bytes: slot table, record arena in use, of which garbage (erased / lost-race records) */
int pr_kv_memory(pr_kv *h, int64_t *slot_bytes, int64_t *arena_bytes, int64_t *garbage_bytes, void *stream);
/* values of every live key (any order); returns the live count (> max: only max written) or < 0 */
int64_t pr_kv_export(pr_kv *h, int64_t *d_vals, int64_t max, void *stream);
/* value v -> d_map[v] for every live key with 0 <= v < nmap (host arena compaction) */
int pr_kv_remap(pr_kv *h, const int64_t *d_map, int64_t nmap, void *stream);
/* device L2 fetch granularity limit (cudaLimitMaxL2FetchGranularity, bytes; <= 0 only reads
 * it): random 32-byte probes waste DRAM bandwidth when L2 fetches whole 128-byte lines */
int pr_l2_fetch_granularity(int bytes, int *previous);

/* ---- on-device cascade: router.py:227-273 (_probe), :275-364 (route) ----------
 * The fast layers' outcome for a batch of B queries and the ONE compacted miss list the
 * vector layers consume (pr_index_search_list), without a host round trip:
 *   l1[j] = d_kv_hit[j] || d_rep[j]   (pre-batch KV probe, or an earlier in-window write)
 *   l2[j] = d_sc_count[j] > 0 && d_sc_score[j] >= sc_threshold   (caches.py:140, inclusive)
 *   l3[j] = d_l3_hit[j]               (accepted recall, pr_recall_gate)
 * A query hit by a fast layer probed before the vector layers (l1/l2/l3_blocks) is
 * dropped; the rest, in query order, form d_list[0..*d_nlist) and d_slot[j] = position or -1.
 * d_kv_hit NULL = L1 not probed; d_sc_count NULL = L2 not probed; d_l3_hit NULL = no recall
 * outcome on the device. */
int pr_cascade_gate(int64_t B, const uint8_t *d_kv_hit, const uint8_t *d_rep, const int32_t *d_sc_count,
                    const double *d_sc_score, double sc_threshold, const uint8_t *d_l3_hit, int l1_blocks,
                    int l2_blocks, int l3_blocks, uint8_t *d_l1, uint8_t *d_l2, int32_t *d_list, int32_t *d_nlist,
                    int32_t *d_slot, void *stream);
/* The L3 recall gate (generation.py:203-224 memory_recall over StubBackend.recall :110-115)
 * for a recall table kept in a pr_kv table (value = index into d_conf): d_out[j] = d_hit[j] &&
 * 0 <= d_vals[j] < nconf && d_conf[d_vals[j]] >= threshold.  d_conf holds -1 for an entry
 * whose answer is empty (never accepted).  threshold outside [0, 1] -> PR_ERR_BAD_ARG. */
int pr_recall_gate(int64_t n, const int64_t *d_vals, const uint8_t *d_hit, const double *d_conf, int64_t nconf,
                   double threshold, uint8_t *d_out, void *stream);
/* The adaptive-memory guard (knowledge.py:217-228: L5 seeds settle before the next query):
 * the seeds (top seed_k knowledge-base rows) of the previous span's listed queries, then of
 * this span's, deduplicated by KB row in first-occurrence order -> d_out_rows[0..*d_nout)
 * (padded with row 0 up to out_max), and d_before[i] = deduplicated seeds visible to this
 * span's listed query i.  d_mark is a KB-row-sized int32 scratch, initialised once with
 * pr_cascade_mark_init and restored by every call.  Previous span arguments may be NULL. */
int pr_cascade_mark_init(int32_t *d_mark, int64_t n, void *stream);
int pr_cascade_seeds(const int64_t *d_prev_rows, const int32_t *d_prev_cnt, const int32_t *d_prev_n,
                     const int64_t *d_rows, const int32_t *d_cnt, const int32_t *d_n, int seed_k, int32_t *d_mark,
                     int64_t *d_out_rows, int64_t out_max, int32_t *d_nout, int64_t *d_before, void *stream);

/* One span of the on-device cascade in ONE call (SURVEY §8(b) pr_cascade_route; router.py:227-273
 * _probe and :275-364 route for B queries): the L1 probe (pr_kv_get_text), the L2 top-1
 * threshold search over the rows each query may see (pr_index_search_floor, d_sc_limit),
 * pr_cascade_gate, the knowledge-base scan of the compacted miss list (pr_index_search_list),
 * the L4 guard (pr_cascade_seeds; the seeds appended to the scratch store `guard` with
 * pr_index_append_from; top-1 threshold searches over it, row-limited per listed query, and
 * over the adaptive memory), then ONE packed int64 record for the host's single read-back:
 *   d_packed[9B + 1 + B*seed_k] = l1[B] l2[B] slot[B] l4[B] sc_row[B] kv_val[B] kb_cnt[B]
 *                                  l3[B] l3_val[B] nlist kb_rows[B*seed_k]
 * (-1 in the columns of a layer not probed; kb_rows past nlist undefined).  The caller holds
 * the stores' locks, clears `guard` first, and keeps d_kb_rows / d_kb_cnt / d_nlist alive
 * for the next span (its d_prev_*).  d_scratch: pr_cascade_route_scratch(B, seed_k, prev_B)
 * bytes, free again once the stream has passed this call. */
typedef struct pr_cascade_span {
    int64_t B;
    const float *d_vec; /* [B, dim] fp32 query vectors */
    uint32_t mode;      /* PR_SEARCH_* for every search of the span */
    /* L1: kv NULL = not probed; keys are the UTF-8 arena of the span's texts */
    pr_kv *kv;
    const uint8_t *d_text;
    const int64_t *d_text_off;
    const uint8_t *d_rep; /* [B] an earlier in-window write of the same text (required) */
    /* L3 decided on the device (pr_recall_gate): NULL = none */
    const uint8_t *d_l3_hit;
    const int64_t *d_l3_val;
    /* L2: sc NULL = not probed */
    pr_index *sc;
    const int64_t *d_sc_limit; /* [B] rows of the semantic cache query j sees */
    double sc_threshold;
    int l1_blocks, l2_blocks, l3_blocks; /* fast layers probed before the vector layers */
    /* L5: the knowledge base, seeds per listed query, expected list length */
    pr_index *kb;
    int seed_k;
    int64_t nlist_hint;
    int64_t *d_kb_rows; /* [B, seed_k] */
    double *d_kb_raw;   /* [B, seed_k] */
    double *d_kb_rep;   /* [B, seed_k] */
    int32_t *d_kb_cnt;  /* [B] */
    int32_t *d_nlist;   /* [1] */
    int32_t *d_slot;    /* [B] list position of query j or -1 */
    /* L4: probe_l4 0 = not probed; akm_rows 0 = empty adaptive memory */
    int probe_l4;
    pr_index *akm;
    int64_t akm_rows;
    double akm_threshold;
    pr_index *guard; /* scratch store, cleared by the caller */
    int32_t *d_mark; /* pr_cascade_mark_init'ed, knowledge-base rows long */
    const int64_t *d_prev_rows;
    const int32_t *d_prev_cnt;
    const int32_t *d_prev_n;
    int64_t prev_B;
    int64_t *d_packed; /* [9B + 1 + B*seed_k] */
} pr_cascade_span;
int64_t pr_cascade_route_scratch(int64_t B, int seed_k, int64_t prev_B);
int pr_cascade_route(const pr_cascade_span *s, void *d_scratch, int64_t scratch_bytes, void *stream);

/* ---- device HashEmbedder: embedding.py:117-160 ------------
 * Texts are a UTF-8 arena + offsets as for pr_fingerprint; d_out is fp32
 * [n, dim], bit-identical to HashEmbedder(seed).embed(text).values for every
 * text the device handles.  d_host_flag[i] = 1 marks texts the device leaves
 * to the host (non-ASCII bytes, empty text, > 256 tokens). */
int pr_hash_embed(const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int dim, uint64_t seed, float *d_out,
                  uint8_t *d_host_flag, void *stream);
/* keyed blake2b (digest 8 bytes, key = seed big-endian) of prefix4 + data, as a
 * big-endian integer — the embedder's token hash, callable on the host */
uint64_t pr_blake2b64_host(uint64_t key, const char *prefix4, const uint8_t *data, int64_t len);

#ifdef __cplusplus
}
#endif
#endif /* PENTARAG_H */
