// Fixed KV cache on the GPU (reference: caches.py:45-101, FixedKVCache).
//
// The reference keys a dict by the raw query text: any one-byte difference is a
// different key (caches.py:57-65, tests/test_caches.py:36-45).  This table
// is byte-exact the same way: a hit is confirmed against the stored key bytes, so a
// fingerprint collision (accidental or constructed) can only cost a probe, never serve
// another key's answer.
//
// Layout (HBM):
//   slots  {u64 tag, u64 rec}[nslots]  nslots a power of two, grouped in 64-byte
//          buckets of 4 slots.  tag = first word of the key's 128-bit fingerprint with
//          the top bit forced (0 = EMPTY, 1 = TOMBSTONE); rec = byte offset of the key's
//          record in the arena.  Load factor <= 0.5.
//   arena  32-byte aligned records {i64 value, i32 len, i32 0, key bytes, zero pad}:
//          one 32-byte sector holds the header and the first 16 key bytes, so a hit on
//          a short key costs one bucket line plus one record sector.
// Home bucket = second fingerprint word & (nbuckets - 1); the shard owner of a key is
// taken from the first word's high half (disjoint from the bucket bits, sharded_kv.py).
//
// Probing is one thread per key: the thread hashes its key ONCE, loads its 64-byte
// bucket with two 256-bit loads (both in flight), compares the four tags in
// registers, confirms a tag match against the record (one more 256-bit load), and
// moves to the next bucket only when the bucket is full of other keys.  A warp keeps
// 32 independent probes in flight.  Values are int64 write sequence numbers supplied by
// the host; a put resolves with atomicMax on the record's value, so the largest (latest)
// write wins even when one batch writes a key twice (caches.py:67-74).
#include <algorithm>

#include "common.cuh"

struct pr_kv {
    ulonglong2 *slots = nullptr;            // [nslots] {tag, record offset}
    int64_t nslots = 0;
    uint8_t *arena = nullptr;               // records
    int64_t arena_cap = 0;                  // bytes
    unsigned long long *d_count = nullptr;  // [0] live [1] tombstones [2] arena cursor [3] garbage bytes
    int64_t upper = 0;                      // host bound on live + tombstones (no sync needed)
    int64_t arena_upper = 0;                // host bound on the arena cursor
    uint32_t flags = 0;                     // PR_KV_WEAK_HASH (tests only)
};

namespace pr {

constexpr uint64_t FP_SEED = 0x5EED1024CA5CADE5ull;  // same constant family as embedding.py:33
constexpr int KV_BUCKET = 4;
constexpr int KV_THREADS = 128;
constexpr int KV_REC_HDR = 16;
constexpr uint64_t TAG_EMPTY = 0, TAG_TOMB = 1;

__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

template <bool DEV>
__host__ __device__ __forceinline__ uint8_t ldb(const uint8_t *p) {
#ifdef __CUDA_ARCH__
    if (DEV) return __ldg(p);
#endif
    return *p;
}

// 128-bit fingerprint of the key bytes (Murmur3-x64-128 construction, fixed seed).
template <bool DEV = false>
__host__ __device__ inline void fingerprint128(const uint8_t *data, int64_t len, uint64_t *h_out, uint64_t *l_out) {
    const uint64_t c1 = 0x87c37b91114253d5ull, c2 = 0x4cf5ad432745937full;
    uint64_t h1 = FP_SEED, h2 = FP_SEED ^ 0x9E3779B97F4A7C15ull;
    const int64_t nblocks = len / 16;
    for (int64_t i = 0; i < nblocks; ++i) {
        uint64_t k1 = 0, k2 = 0;
        for (int b = 7; b >= 0; --b) k1 = (k1 << 8) | ldb<DEV>(data + 16 * i + b);
        for (int b = 7; b >= 0; --b) k2 = (k2 << 8) | ldb<DEV>(data + 16 * i + 8 + b);
        k1 *= c1; k1 = rotl64(k1, 31); k1 *= c2; h1 ^= k1;
        h1 = rotl64(h1, 27); h1 += h2; h1 = h1 * 5 + 0x52dce729;
        k2 *= c2; k2 = rotl64(k2, 33); k2 *= c1; h2 ^= k2;
        h2 = rotl64(h2, 31); h2 += h1; h2 = h2 * 5 + 0x38495ab5;
    }
    const uint8_t *tail = data + nblocks * 16;
    const int rem = (int)(len & 15);
    uint64_t k1 = 0, k2 = 0;
    for (int b = rem - 1; b >= 8; --b) k2 = (k2 << 8) | ldb<DEV>(tail + b);
    for (int b = std::min(rem, 8) - 1; b >= 0; --b) k1 = (k1 << 8) | ldb<DEV>(tail + b);
    if (rem > 8) { k2 *= c2; k2 = rotl64(k2, 33); k2 *= c1; h2 ^= k2; }
    if (rem > 0) { k1 *= c1; k1 = rotl64(k1, 31); k1 *= c2; h1 ^= k1; }
    h1 ^= (uint64_t)len;
    h2 ^= (uint64_t)len;
    h1 += h2; h2 += h1;
    h1 = fmix64(h1); h2 = fmix64(h2);
    h1 += h2; h2 += h1;
    *h_out = h1 | 0x8000000000000000ull;  // never EMPTY/TOMBSTONE
    *l_out = h2;
}

__host__ __device__ __forceinline__ int owner_of(uint64_t tag, int world) {
    return (int)((uint32_t)((tag >> 32) & 0x7fffffffu) % (uint32_t)world);
}

__host__ __device__ __forceinline__ int64_t rec_bytes(int64_t len) { return round_up<int64_t>(KV_REC_HDR + len, 32); }

// little-endian word of up to 8 key bytes (missing bytes read as zero)
__device__ __forceinline__ uint64_t key_word(const uint8_t *p, int n) {
    uint64_t w = 0;
    for (int b = (n < 8 ? n : 8) - 1; b >= 0; --b) w = (w << 8) | __ldg(p + b);
    return w;
}

template <bool STRONG>
__device__ __forceinline__ void ld256(const void *p, uint64_t &a, uint64_t &b, uint64_t &c, uint64_t &d) {
    if (STRONG)
        asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p) : "memory");
    else
        asm("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}

// Does the record at `rec` hold exactly the key bytes [key, key+len)?  The record's
// first sector (header + 16 key bytes) is one 256-bit load; the value comes with it.
template <bool STRONG>
__device__ __forceinline__ bool rec_matches(const uint8_t *rec, const uint8_t *key, int64_t len, int64_t *val_out) {
    uint64_t w0, w1, w2, w3;
    ld256<STRONG>(rec, w0, w1, w2, w3);
    if ((int64_t)(uint32_t)w1 != len) return false;
    if (w2 != key_word(key, (int)std::min<int64_t>(len, 8))) return false;
    if (len > 8 && w3 != key_word(key + 8, (int)std::min<int64_t>(len - 8, 8))) return false;
    for (int64_t o = 16; o < len; o += 8) {
        uint64_t r = STRONG ? *reinterpret_cast<const volatile uint64_t *>(rec + KV_REC_HDR + o)
                            : __ldcg(reinterpret_cast<const unsigned long long *>(rec + KV_REC_HDR + o));
        if (r != key_word(key + o, (int)std::min<int64_t>(len - o, 8))) return false;
    }
    *val_out = (int64_t)w0;
    return true;
}

__device__ __forceinline__ bool cas_slot(ulonglong2 *slot, uint64_t e0, uint64_t e1, uint64_t n0, uint64_t n1,
                                         uint64_t &o0, uint64_t &o1) {
    asm volatile(
        "{\n\t.reg .b128 d, c, v;\n\t"
        "mov.b128 c, {%2, %3};\n\t"
        "mov.b128 v, {%4, %5};\n\t"
        "atom.global.cas.b128 d, [%6], c, v;\n\t"
        "mov.b128 {%0, %1}, d;\n\t}"
        : "=l"(o0), "=l"(o1)
        : "l"(e0), "l"(e1), "l"(n0), "l"(n1), "l"(slot)
        : "memory");
    return o0 == e0 && o1 == e1;
}

// copy a key into a fresh record (header + bytes, zero padded to the 32-byte record size)
__device__ void write_record(uint8_t *rec, const uint8_t *key, int64_t len, int64_t val) {
    uint64_t *w = reinterpret_cast<uint64_t *>(rec);
    w[0] = (uint64_t)val;
    w[1] = (uint64_t)(uint32_t)len;
    const int64_t words = (rec_bytes(len) - KV_REC_HDR) / 8;
    for (int64_t i = 0; i < words; ++i) {
        const int64_t o = 8 * i;
        w[2 + i] = o < len ? key_word(key + o, (int)std::min<int64_t>(len - o, 8)) : 0;
    }
}

struct KvTable {
    ulonglong2 *slots;
    int64_t nb;  // buckets (power of two)
    uint8_t *arena;
    unsigned long long *counts;
    int weak;    // PR_KV_WEAK_HASH: 2-bit tags, 4 home buckets (forces collisions; tests only)
};

// tag + home-bucket hash of a key (the weak variant keeps 2 tag bits and 2 bucket bits)
__device__ __forceinline__ void key_hash(const KvTable &t, const uint8_t *key, int64_t len, uint64_t &tag,
                                         uint64_t &h2) {
    fingerprint128<true>(key, len, &tag, &h2);
    if (t.weak) {
        tag = (tag & 0x8000000000000003ull) | 0x8000000000000000ull;
        h2 &= 3;
    }
}

struct KeyBatch {
    const uint8_t *bytes;
    const int64_t *off;
    int64_t n;
};

// ---- get: one thread per key ------------------------------------------------
__global__ void __launch_bounds__(KV_THREADS) kv_get_kernel(KvTable t, KeyBatch kb, int rank, int world,
                                                             int64_t *__restrict__ out_vals,
                                                             uint8_t *__restrict__ out_hit) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= kb.n) return;
    const int64_t a = __ldg(kb.off + i), len = __ldg(kb.off + i + 1) - a;
    const uint8_t *key = kb.bytes + a;
    uint64_t tag, h2;
    key_hash(t, key, len, tag, h2);
    int64_t val = -1;
    if (world <= 1 || owner_of(tag, world) == rank) {
        int64_t b = (int64_t)(h2 & (uint64_t)(t.nb - 1));
        for (int64_t p = 0; p < t.nb; ++p) {
            uint64_t s[8];
            const ulonglong2 *bk = t.slots + b * KV_BUCKET;
            ld256<false>(bk, s[0], s[1], s[2], s[3]);
            ld256<false>(bk + 2, s[4], s[5], s[6], s[7]);
            bool done = false;
#pragma unroll
            for (int j = 0; j < KV_BUCKET; ++j) {
                if (done) break;
                if (s[2 * j] == tag) {
                    int64_t v;
                    if (rec_matches<false>(t.arena + s[2 * j + 1], key, len, &v)) {
                        val = v;
                        done = true;
                    }
                } else if (s[2 * j] == TAG_EMPTY) {
                    done = true;
                }
            }
            if (done) break;
            b = (b + 1) & (t.nb - 1);
        }
    }
    out_vals[i] = val;
    out_hit[i] = val >= 0;
}

// ---- put (upsert) / erase: one thread per key --------------------------------
template <bool ERASE>
__global__ void __launch_bounds__(KV_THREADS) kv_update_kernel(KvTable t, KeyBatch kb, int rank, int world,
                                                                const int64_t *__restrict__ in_vals) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= kb.n) return;
    const int64_t a = __ldg(kb.off + i), len = __ldg(kb.off + i + 1) - a;
    const uint8_t *key = kb.bytes + a;
    uint64_t tag, h2;
    key_hash(t, key, len, tag, h2);
    if (world > 1 && owner_of(tag, world) != rank) return;
    const int64_t v = ERASE ? -1 : in_vals[i];
    int64_t myrec = -1;  // record allocated for an insert (kept across lost CAS races)
    int64_t b = (int64_t)(h2 & (uint64_t)(t.nb - 1));
    bool done = false;
    for (int64_t p = 0; p < t.nb && !done; ++p) {
        uint64_t s[8];
        ulonglong2 *bk = t.slots + b * KV_BUCKET;
        ld256<true>(bk, s[0], s[1], s[2], s[3]);
        ld256<true>(bk + 2, s[4], s[5], s[6], s[7]);
        for (int j = 0; j < KV_BUCKET && !done; ++j) {
            uint64_t st = s[2 * j], sr = s[2 * j + 1];
            for (;;) {  // re-examines slot j after a lost CAS
                if (st == tag) {
                    __threadfence();  // the record was published before its slot (see insert)
                    int64_t old;
                    if (rec_matches<true>(t.arena + sr, key, len, &old)) {
                        if (ERASE) {
                            uint64_t o0, o1;
                            if (cas_slot(bk + j, st, sr, TAG_TOMB, 0, o0, o1)) {
                                atomicAdd(&t.counts[0], (unsigned long long)-1ll);
                                atomicAdd(&t.counts[1], 1ull);
                                atomicAdd(&t.counts[3], (unsigned long long)rec_bytes(len));
                            }
                        } else {
                            atomicMax(reinterpret_cast<long long *>(t.arena + sr), (long long)v);
                        }
                        done = true;
                    }
                    break;
                }
                if (st != TAG_EMPTY) break;  // another key or a tombstone: next slot
                if (ERASE) {                 // first empty slot: the key is absent
                    done = true;
                    break;
                }
                if (myrec < 0) {
                    myrec = (int64_t)atomicAdd(&t.counts[2], (unsigned long long)rec_bytes(len));
                    write_record(t.arena + myrec, key, len, v);
                    __threadfence();  // publish the record before the slot that points at it
                }
                uint64_t o0, o1;
                if (cas_slot(bk + j, TAG_EMPTY, 0, tag, (uint64_t)myrec, o0, o1)) {
                    atomicAdd(&t.counts[0], 1ull);
                    myrec = -1;
                    done = true;
                    break;
                }
                st = o0;  // lost the race: look at what was written there
                sr = o1;
            }
        }
        b = (b + 1) & (t.nb - 1);
    }
    if (myrec >= 0) atomicAdd(&t.counts[3], (unsigned long long)rec_bytes(len));  // lost every race
}

// ---- fingerprints / shard owners ---------------------------------------------
__global__ void fingerprint_kernel(KeyBatch kb, uint64_t *__restrict__ fp, int world, int32_t *__restrict__ owner) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < kb.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = kb.off[i];
        uint64_t h, l;
        fingerprint128<true>(kb.bytes + a, kb.off[i + 1] - a, &h, &l);
        if (fp) {
            fp[2 * i] = h;
            fp[2 * i + 1] = l;
        }
        if (owner) owner[i] = owner_of(h, world);
    }
}

// ---- maintenance ---------------------------------------------------------------
__global__ void kv_export_kernel(KvTable t, int64_t nslots, int64_t *val_out, int64_t max, unsigned long long *cursor) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots; s += (int64_t)gridDim.x * blockDim.x) {
        const ulonglong2 sl = t.slots[s];
        if (sl.x & 0x8000000000000000ull) {
            unsigned long long p = atomicAdd(cursor, 1ull);
            if ((int64_t)p < max) val_out[p] = *reinterpret_cast<const int64_t *>(t.arena + sl.y);
        }
    }
}

__global__ void kv_remap_kernel(KvTable t, int64_t nslots, const int64_t *__restrict__ map, int64_t nmap) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots; s += (int64_t)gridDim.x * blockDim.x) {
        const ulonglong2 sl = t.slots[s];
        if (sl.x & 0x8000000000000000ull) {
            int64_t *v = reinterpret_cast<int64_t *>(t.arena + sl.y);
            if (*v >= 0 && *v < nmap) *v = map[*v];
        }
    }
}

// rebuild: every live key of the old table is copied into a fresh arena (compacting away
// overwritten/erased records) and re-inserted by its fingerprint (no duplicates exist)
__global__ void kv_rebuild_kernel(const ulonglong2 *__restrict__ old_slots, int64_t old_n,
                                  const uint8_t *__restrict__ old_arena, KvTable t) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < old_n; s += (int64_t)gridDim.x * blockDim.x) {
        const ulonglong2 sl = old_slots[s];
        if (!(sl.x & 0x8000000000000000ull)) continue;
        const uint8_t *rec = old_arena + sl.y;
        const int64_t len = (int64_t)(uint32_t)reinterpret_cast<const uint64_t *>(rec)[1];
        const int64_t rb = rec_bytes(len);
        const int64_t dst = (int64_t)atomicAdd(&t.counts[2], (unsigned long long)rb);
        for (int64_t o = 0; o < rb; o += 8)
            *reinterpret_cast<uint64_t *>(t.arena + dst + o) = *reinterpret_cast<const uint64_t *>(rec + o);
        uint64_t tag, h2;
        key_hash(t, rec + KV_REC_HDR, len, tag, h2);
        int64_t b = (int64_t)(h2 & (uint64_t)(t.nb - 1));
        bool done = false;
        for (int64_t p = 0; p < t.nb && !done; ++p) {
            for (int j = 0; j < KV_BUCKET && !done; ++j) {
                uint64_t o0, o1;
                if (cas_slot(t.slots + b * KV_BUCKET + j, TAG_EMPTY, 0, tag, (uint64_t)dst, o0, o1)) {
                    atomicAdd(&t.counts[0], 1ull);
                    done = true;
                }
            }
            b = (b + 1) & (t.nb - 1);
        }
    }
}

static int64_t slots_for(int64_t keys) {
    int64_t s = 1024;
    while (s < 2 * keys) s *= 2;  // load factor <= 0.5
    return s;
}

static KvTable table_of(pr_kv *h) {
    return KvTable{h->slots, h->nslots / KV_BUCKET, h->arena, h->d_count, (h->flags & PR_KV_WEAK_HASH) ? 1 : 0};
}

static int read_counts(pr_kv *h, unsigned long long c[4], cudaStream_t st) {
    PR_CUDA(cudaMemcpyAsync(c, h->d_count, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    return PR_OK;
}

// Rebuild into a table for `need_keys` live keys and an arena of `need_bytes` live record
// bytes (drops tombstones and garbage records).  Synchronises the device: rare.
static int rebuild(pr_kv *h, int64_t need_keys, int64_t need_bytes, cudaStream_t st) {
    unsigned long long c[4];
    int rc = read_counts(h, c, st);
    if (rc) return rc;
    PR_CUDA(cudaDeviceSynchronize());
    const int64_t live = (int64_t)c[0];
    const int64_t live_bytes = (int64_t)c[2] - (int64_t)c[3];
    const int64_t nslots = slots_for(std::max<int64_t>(need_keys, live));
    const int64_t acap = std::max<int64_t>(4096, round_up<int64_t>(need_bytes + need_bytes / 2, 256));
    ulonglong2 *ns = nullptr;
    uint8_t *na = nullptr;
    PR_CUDA(cudaMalloc(&ns, (size_t)nslots * sizeof(ulonglong2)));
    if (cudaMalloc(&na, (size_t)acap) != cudaSuccess) {
        cudaFree(ns);
        PR_FAIL(PR_ERR_NOMEM, "kv arena: cannot allocate %lld bytes", (long long)acap);
    }
    PR_CUDA(cudaMemsetAsync(ns, 0, (size_t)nslots * sizeof(ulonglong2), st));
    PR_CUDA(cudaMemsetAsync(h->d_count, 0, 4 * sizeof(unsigned long long), st));
    ulonglong2 *os = h->slots;
    uint8_t *oa = h->arena;
    const int64_t on = h->nslots;
    h->slots = ns;
    h->nslots = nslots;
    h->arena = na;
    h->arena_cap = acap;
    if (live > 0) {
        const int g = (int)std::min<int64_t>(ceil_div<int64_t>(on, 256), (int64_t)sm_count() * 16);
        ::pr::count_launch();
        kv_rebuild_kernel<<<g, 256, 0, st>>>(os, on, oa, table_of(h));
        PR_LAUNCH_CHECK();
    }
    PR_CUDA(cudaStreamSynchronize(st));
    cudaFree(os);
    cudaFree(oa);
    h->upper = live;
    h->arena_upper = live_bytes;
    return PR_OK;
}

static unsigned kv_grid(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div<int64_t>(n, KV_THREADS)); }

static int check_batch(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int rank, int world) {
    if (!h || n < 0 || (n > 0 && (!d_bytes || !d_off))) PR_FAIL(PR_ERR_BAD_ARG, "bad kv key batch");
    if (world < 1 || rank < 0 || rank >= world) PR_FAIL(PR_ERR_BAD_ARG, "bad shard rank/world");
    return PR_OK;
}

static int put_impl(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int64_t nbytes,
                    const int64_t *d_vals, int rank, int world, void *stream) {
    int rc = check_batch(h, d_bytes, d_off, n, rank, world);
    if (rc) return rc;
    if (nbytes < 0 || !d_vals) PR_FAIL(PR_ERR_BAD_ARG, "bad kv_put");
    if (n == 0) return PR_OK;
    cudaStream_t st = as_stream(stream);
    const int64_t rec_need = n * (KV_REC_HDR + 31) + nbytes;  // >= sum of rec_bytes over the batch
    if (2 * (h->upper + n) > h->nslots || h->arena_upper + rec_need > h->arena_cap) {
        unsigned long long c[4];
        rc = read_counts(h, c, st);
        if (rc) return rc;
        h->upper = (int64_t)(c[0] + c[1]);
        h->arena_upper = (int64_t)c[2];
        const bool slots_short = 2 * (h->upper + n) > h->nslots;
        const bool arena_short = h->arena_upper + rec_need > h->arena_cap;
        if (slots_short || arena_short) {
            rc = rebuild(h, (int64_t)c[0] + n, (int64_t)(c[2] - c[3]) + rec_need, st);
            if (rc) return rc;
        }
    }
    ::pr::count_launch();
    kv_update_kernel<false><<<kv_grid(n), KV_THREADS, 0, st>>>(table_of(h), KeyBatch{d_bytes, d_off, n}, rank,
                                                                world, d_vals);
    PR_LAUNCH_CHECK();
    h->upper += n;
    h->arena_upper += rec_need;
    return PR_OK;
}

static int get_impl(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int rank, int world,
                    int64_t *d_vals, uint8_t *d_hit, void *stream) {
    int rc = check_batch(h, d_bytes, d_off, n, rank, world);
    if (rc) return rc;
    if (n == 0) return PR_OK;
    if (!d_vals || !d_hit) PR_FAIL(PR_ERR_BAD_ARG, "bad kv_get outputs");
    ::pr::count_launch();
    kv_get_kernel<<<kv_grid(n), KV_THREADS, 0, as_stream(stream)>>>(table_of(h), KeyBatch{d_bytes, d_off, n}, rank,
                                                                      world, d_vals, d_hit);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

}  // namespace pr

using namespace pr;

extern "C" {

void pr_fingerprint_host(const uint8_t *bytes, int64_t len, uint64_t out[2]) {
    fingerprint128<false>(bytes, len, &out[0], &out[1]);
}

int pr_fingerprint(const uint8_t *d_bytes, const int64_t *d_off, int64_t n, uint64_t *d_fp, void *stream) {
    if (n < 0) PR_FAIL(PR_ERR_BAD_ARG, "n < 0");
    if (n == 0) return PR_OK;
    int g = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), (int64_t)sm_count() * 16);
    ::pr::count_launch();
    fingerprint_kernel<<<g, 256, 0, as_stream(stream)>>>(KeyBatch{d_bytes, d_off, n}, d_fp, 1, nullptr);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

int pr_kv_owner(const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int world, int32_t *d_owner, void *stream) {
    if (n < 0 || world < 1 || (n > 0 && !d_owner)) PR_FAIL(PR_ERR_BAD_ARG, "bad kv_owner");
    if (n == 0) return PR_OK;
    int g = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), (int64_t)sm_count() * 16);
    ::pr::count_launch();
    fingerprint_kernel<<<g, 256, 0, as_stream(stream)>>>(KeyBatch{d_bytes, d_off, n}, nullptr, world, d_owner);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

int pr_kv_create(int64_t capacity, pr_kv **out) { return pr_kv_create_ex(capacity, 0, out); }

int pr_kv_create_ex(int64_t capacity, uint32_t flags, pr_kv **out) {
    if (!out || capacity < 0 || (flags & ~PR_KV_WEAK_HASH)) PR_FAIL(PR_ERR_BAD_ARG, "bad kv_create");
    pr_kv *h = new pr_kv();
    h->flags = flags;
    h->nslots = slots_for(capacity);
    h->arena_cap = std::max<int64_t>(4096, capacity * 48);
    if (cudaMalloc(&h->slots, (size_t)h->nslots * sizeof(ulonglong2)) != cudaSuccess ||
        cudaMalloc(&h->arena, (size_t)h->arena_cap) != cudaSuccess ||
        cudaMalloc(&h->d_count, 4 * sizeof(unsigned long long)) != cudaSuccess) {
        cudaFree(h->slots);
        cudaFree(h->arena);
        delete h;
        cudaGetLastError();
        PR_FAIL(PR_ERR_NOMEM, "kv_create: device allocation failed");
    }
    PR_CUDA(cudaMemset(h->slots, 0, (size_t)h->nslots * sizeof(ulonglong2)));
    PR_CUDA(cudaMemset(h->d_count, 0, 4 * sizeof(unsigned long long)));
    PR_CUDA(cudaDeviceSynchronize());
    *out = h;
    return PR_OK;
}

int pr_kv_destroy(pr_kv *h) {
    if (!h) return PR_OK;
    cudaDeviceSynchronize();
    cudaFree(h->slots);
    cudaFree(h->arena);
    cudaFree(h->d_count);
    delete h;
    return PR_OK;
}

int pr_kv_put_text(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int64_t nbytes,
                   const int64_t *d_vals, void *stream) {
    return put_impl(h, d_bytes, d_off, n, nbytes, d_vals, 0, 1, stream);
}

int pr_kv_put_text_owned(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int64_t nbytes,
                         const int64_t *d_vals, int rank, int world, void *stream) {
    return put_impl(h, d_bytes, d_off, n, nbytes, d_vals, rank, world, stream);
}

int pr_kv_get_text(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int64_t *d_vals, uint8_t *d_hit,
                   void *stream) {
    return get_impl(h, d_bytes, d_off, n, 0, 1, d_vals, d_hit, stream);
}

int pr_kv_get_text_owned(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int rank, int world,
                         int64_t *d_vals, uint8_t *d_hit, void *stream) {
    return get_impl(h, d_bytes, d_off, n, rank, world, d_vals, d_hit, stream);
}

int pr_kv_erase_text(pr_kv *h, const uint8_t *d_bytes, const int64_t *d_off, int64_t n, void *stream) {
    int rc = check_batch(h, d_bytes, d_off, n, 0, 1);
    if (rc) return rc;
    if (n == 0) return PR_OK;
    ::pr::count_launch();
    kv_update_kernel<true><<<kv_grid(n), KV_THREADS, 0, as_stream(stream)>>>(table_of(h), KeyBatch{d_bytes, d_off, n},
                                                                             0, 1, nullptr);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

int pr_kv_clear(pr_kv *h, void *stream) {
    if (!h) PR_FAIL(PR_ERR_BAD_ARG, "null kv");
    cudaStream_t st = as_stream(stream);
    PR_CUDA(cudaMemsetAsync(h->slots, 0, (size_t)h->nslots * sizeof(ulonglong2), st));
    PR_CUDA(cudaMemsetAsync(h->d_count, 0, 4 * sizeof(unsigned long long), st));
    h->upper = 0;
    h->arena_upper = 0;
    return PR_OK;
}

int64_t pr_kv_size(pr_kv *h, void *stream) {
    if (!h) return -1;
    unsigned long long c[4];
    if (read_counts(h, c, as_stream(stream)) != PR_OK) return -1;
    return (int64_t)c[0];
}

int64_t pr_kv_capacity(pr_kv *h) { return h ? h->nslots : -1; }

int pr_kv_memory(pr_kv *h, int64_t *slot_bytes, int64_t *arena_bytes, int64_t *garbage_bytes, void *stream) {
    if (!h) PR_FAIL(PR_ERR_BAD_ARG, "null kv");
    unsigned long long c[4];
    int rc = read_counts(h, c, as_stream(stream));
    if (rc) return rc;
    if (slot_bytes) *slot_bytes = h->nslots * (int64_t)sizeof(ulonglong2);
    if (arena_bytes) *arena_bytes = (int64_t)c[2];
    if (garbage_bytes) *garbage_bytes = (int64_t)c[3];
    return PR_OK;
}

int64_t pr_kv_export(pr_kv *h, int64_t *d_vals, int64_t max, void *stream) {
    if (!h || max < 0) PR_FAIL(PR_ERR_BAD_ARG, "bad kv_export");
    cudaStream_t st = as_stream(stream);
    unsigned long long *cur = nullptr;
    PR_CUDA(cudaMallocAsync(&cur, sizeof(unsigned long long), st));
    PR_CUDA(cudaMemsetAsync(cur, 0, sizeof(unsigned long long), st));
    int g = (int)std::min<int64_t>(ceil_div<int64_t>(h->nslots, 256), (int64_t)sm_count() * 16);
    ::pr::count_launch();
    kv_export_kernel<<<g, 256, 0, st>>>(table_of(h), h->nslots, d_vals, max, cur);
    PR_LAUNCH_CHECK();
    unsigned long long c = 0;
    PR_CUDA(cudaMemcpyAsync(&c, cur, sizeof(c), cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaFreeAsync(cur, st));
    PR_CUDA(cudaStreamSynchronize(st));
    return (int64_t)c;  // may exceed max: the caller retries with a larger buffer
}

int pr_kv_remap(pr_kv *h, const int64_t *d_map, int64_t nmap, void *stream) {
    if (!h || nmap < 0 || (nmap > 0 && !d_map)) PR_FAIL(PR_ERR_BAD_ARG, "bad kv_remap");
    if (nmap == 0) return PR_OK;
    int g = (int)std::min<int64_t>(ceil_div<int64_t>(h->nslots, 256), (int64_t)sm_count() * 16);
    ::pr::count_launch();
    kv_remap_kernel<<<g, 256, 0, as_stream(stream)>>>(table_of(h), h->nslots, d_map, nmap);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

}  // extern "C"
