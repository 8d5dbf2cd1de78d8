// Fixed KV cache on the GPU (reference: caches.py:45-101, FixedKVCache).
//
// The reference keys a dict by the raw query text: any one-byte difference is a
// different key (caches.py:57-65, tests/test_caches.py:36-45).  This table
// is byte-exact the same way: a hit is confirmed against the stored key bytes, so a hash
// collision (accidental or constructed) can only cost a probe, never serve another key's
// answer.
//
// Layout (HBM):
//   slots  u64[nslots] = {u32 tag | u32 rec << 32}, nslots a power of two, grouped in
//          32-byte buckets of 4 slots (ONE DRAM sector per bucket).  tag = 32-bit key hash
//          with the top bit forced (0 = EMPTY, 1 = TOMBSTONE); rec = the key's record in
//          32-byte units.  Load factor <= 0.5.
//   arena  32-byte aligned records {i64 value, u32 len, u32 0, key bytes, zero pad}: one
//          sector holds the header and the first 16 key bytes, so a hit on a short key
//          costs one bucket sector plus one record sector.
// Hash: two 32-bit multiply-rotate chains over the key's little-endian words (murmur3_32
// round function, two seeds).  hA -> tag (and shard owner), hB -> home bucket: the
// ownership bits and the bucket bits come from independent chains.  Only 32-bit integer
// multiplies (no 64-bit emulation): the hash is a short dependency chain per key.
//
// Probing is one thread per key: it hashes its key ONCE (aligned 32-bit loads + funnel
// shifts, not byte loads), reads its bucket with one 256-bit load, compares the four tags
// in registers, confirms a tag match against the record (one more 256-bit load, which
// also carries the value), and moves to the next bucket only when the bucket is full of
// other keys.  A warp keeps 32 independent probes in flight.  Values are non-negative
// int64 write sequence numbers supplied by the host; a put resolves with atomicMax on the
// record's value, so the largest (latest) write wins even when one batch writes a key
// twice (caches.py:67-74).
#include <algorithm>

#include "common.cuh"

struct pr_kv {
    unsigned long long *slots = nullptr;    // [nslots] {tag, record index}
    int64_t nslots = 0;
    uint8_t *arena = nullptr;               // records
    int64_t arena_cap = 0;                  // bytes
    unsigned long long *d_count = nullptr;  // [0] live [1] tombstones [2] arena cursor [3] garbage bytes
    int64_t upper = 0;                      // host bound on live + tombstones (no sync needed)
    int64_t arena_upper = 0;                // host bound on the arena cursor
    uint32_t flags = 0;                     // PR_KV_WEAK_HASH (tests only)
};

namespace pr {

constexpr int KV_BUCKET = 4;  // slots per 32-byte bucket
constexpr int KV_THREADS = 128;
constexpr int KV_REC_HDR = 16;
constexpr uint32_t TAG_EMPTY = 0, TAG_TOMB = 1;
constexpr uint32_t SEED_A = 0x5EED1024u, SEED_B = 0xCA5CADE5u;  // the HASH_SEED family (embedding.py:33)
constexpr int64_t KV_MAX_ARENA = (int64_t)32 << 32;              // 32-bit record index x 32 bytes

__host__ __device__ __forceinline__ uint32_t rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }
__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    return h;
}
__host__ __device__ __forceinline__ uint32_t mix32(uint32_t h, uint32_t k) {
    k *= 0xcc9e2d51u;
    k = rotl32(k, 15);
    k *= 0x1b873593u;
    h ^= k;
    h = rotl32(h, 13);
    return h * 5u + 0xe6546b64u;
}

// The two hash chains over little-endian 32-bit key words (the last one zero padded).
struct KeyHash {
    uint32_t a, b;
    __host__ __device__ __forceinline__ void init(int64_t len) {
        a = SEED_A ^ (uint32_t)len;
        b = SEED_B ^ (uint32_t)(len * 0x9E3779B1u);
    }
    __host__ __device__ __forceinline__ void word(uint32_t w) {
        a = mix32(a, w);
        b = mix32(b, w * 0x9E3779B1u + 0x7F4A7C15u);
    }
    __host__ __device__ __forceinline__ void fin(int64_t len, uint32_t &tag, uint32_t &hb) {
        tag = fmix32(a ^ (uint32_t)len) | 0x80000000u;  // never EMPTY/TOMBSTONE
        hb = fmix32(b ^ (uint32_t)(len >> 32) ^ 0x2545F491u);
    }
};

__host__ __device__ __forceinline__ int owner_of(uint32_t tag, int world) {
    return (int)((tag & 0x7fffffffu) % (uint32_t)world);
}

__host__ __device__ __forceinline__ int64_t rec_bytes(int64_t len) { return round_up<int64_t>(KV_REC_HDR + len, 32); }

// A key in device memory, read as aligned 32-bit words: word j = bytes [4j, 4j+4) of the
// key (little-endian, zero beyond len).  Only words that hold key bytes are loaded.
struct KeyRef {
    const uint32_t *w;  // aligned base
    int sh;             // misalignment in bits
    int64_t len;
    int64_t last;       // index (from w) of the aligned word holding the last key byte
    __device__ __forceinline__ KeyRef(const uint8_t *p, int64_t n) {
        const uintptr_t u = reinterpret_cast<uintptr_t>(p);
        w = reinterpret_cast<const uint32_t *>(u & ~(uintptr_t)3);
        sh = (int)(u & 3) * 8;
        len = n;
        last = n > 0 ? ((u & 3) + n - 1) >> 2 : -1;
    }
    __device__ __forceinline__ uint32_t ld(int64_t j) const { return j <= last ? __ldg(w + j) : 0u; }
    // word j given the aligned words j and j+1 already loaded
    __device__ __forceinline__ uint32_t join(uint32_t lo, uint32_t hi, int64_t j) const {
        uint32_t v = sh ? __funnelshift_r(lo, hi, sh) : lo;
        const int64_t rem = len - 4 * j;
        return rem >= 4 ? v : (rem <= 0 ? 0u : v & ((1u << (8 * rem)) - 1u));
    }
    __device__ __forceinline__ uint32_t word(int64_t j) const { return join(ld(j), sh ? ld(j + 1) : 0u, j); }
};

__device__ __forceinline__ void hash_key(const KeyRef &k, int weak, uint32_t &tag, uint32_t &hb) {
    KeyHash h;
    h.init(k.len);
    const int64_t nw = (k.len + 3) >> 2;
    uint32_t lo = k.ld(0);
    for (int64_t j = 0; j < nw; ++j) {
        const uint32_t hi = k.sh ? k.ld(j + 1) : 0u;
        h.word(k.join(lo, hi, j));
        lo = k.sh ? hi : k.ld(j + 1);
    }
    h.fin(k.len, tag, hb);
    if (weak) {  // PR_KV_WEAK_HASH: 2 tag bits, 4 home buckets
        tag = (tag & 3u) | 0x80000000u;
        hb &= 3u;
    }
}

static inline void hash_host(const uint8_t *p, int64_t len, uint32_t &tag, uint32_t &hb) {
    KeyHash h;
    h.init(len);
    for (int64_t o = 0; o < len; o += 4) {
        uint32_t v = 0;
        for (int b = (int)std::min<int64_t>(4, len - o) - 1; b >= 0; --b) v = (v << 8) | p[o + b];
        h.word(v);
    }
    h.fin(len, tag, hb);
}

template <bool STRONG>
__device__ __forceinline__ void ld256(const void *p, uint64_t &a, uint64_t &b, uint64_t &c, uint64_t &d) {
    if (STRONG)
        asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p) : "memory");
    else
        asm("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}

template <bool STRONG>
__device__ __forceinline__ void ld128(const void *p, uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d) {
    if (STRONG)
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p) : "memory");
    else
        asm("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
}

// Does the record at `rec` hold exactly the key's bytes?  The record's first sector
// (header + key words 0..3) is one 256-bit load; the value comes with it.
template <bool STRONG>
__device__ __forceinline__ bool rec_matches(const uint8_t *rec, const KeyRef &k, int64_t *val_out) {
    uint64_t w0, w1, w2, w3;
    ld256<STRONG>(rec, w0, w1, w2, w3);
    if ((int64_t)(uint32_t)w1 != k.len) return false;
    if ((uint32_t)w2 != k.word(0) || (uint32_t)(w2 >> 32) != k.word(1) || (uint32_t)w3 != k.word(2) ||
        (uint32_t)(w3 >> 32) != k.word(3))
        return false;
    for (int64_t g = 1; 16 * g < k.len; ++g) {
        uint32_t r[4];
        ld128<STRONG>(rec + KV_REC_HDR + 16 * g, r[0], r[1], r[2], r[3]);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (r[q] != k.word(4 * g + q)) return false;
    }
    *val_out = (int64_t)w0;
    return true;
}

// copy a key into a fresh record (header + bytes, zero padded to the 32-byte record size)
__device__ void write_record(uint8_t *rec, const KeyRef &k, int64_t val) {
    uint64_t *h = reinterpret_cast<uint64_t *>(rec);
    h[0] = (uint64_t)val;
    h[1] = (uint64_t)(uint32_t)k.len;
    uint32_t *w = reinterpret_cast<uint32_t *>(rec + KV_REC_HDR);
    const int64_t words = (rec_bytes(k.len) - KV_REC_HDR) / 4;
    for (int64_t j = 0; j < words; ++j) w[j] = k.word(j);
}

struct KvTable {
    unsigned long long *slots;
    int64_t nb;  // buckets (power of two)
    uint8_t *arena;
    unsigned long long *counts;
    int weak;  // PR_KV_WEAK_HASH: 2-bit tags, 4 home buckets (forces collisions; tests only)
};

struct KeyBatch {
    const uint8_t *bytes;
    const int64_t *off;
    int64_t n;
};

__device__ __forceinline__ uint64_t slot_of(uint32_t tag, int64_t rec_off) {
    return (uint64_t)tag | ((uint64_t)(rec_off >> 5) << 32);
}
__device__ __forceinline__ int64_t rec_off_of(uint64_t s) { return (int64_t)(s >> 32) << 5; }

// ---- get: one thread per key ------------------------------------------------
__global__ void __launch_bounds__(KV_THREADS) kv_get_kernel(KvTable t, KeyBatch kb, int rank, int world,
                                                             int64_t *__restrict__ out_vals,
                                                             uint8_t *__restrict__ out_hit) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= kb.n) return;
    const int64_t a = __ldg(kb.off + i);
    const KeyRef k(kb.bytes + a, __ldg(kb.off + i + 1) - a);
    uint32_t tag, hb;
    hash_key(k, t.weak, tag, hb);
    int64_t val = -1;
    if (world <= 1 || owner_of(tag, world) == rank) {
        int64_t b = (int64_t)(hb & (uint32_t)(t.nb - 1));
        for (int64_t p = 0; p < t.nb; ++p) {
            uint64_t s[4];
            ld256<false>(t.slots + b * KV_BUCKET, s[0], s[1], s[2], s[3]);
            bool done = false;
#pragma unroll
            for (int j = 0; j < KV_BUCKET; ++j) {
                if (done) break;
                const uint32_t st = (uint32_t)s[j];
                if (st == tag) {
                    int64_t v;
                    if (rec_matches<false>(t.arena + rec_off_of(s[j]), k, &v)) {
                        val = v;
                        done = true;
                    }
                } else if (st == TAG_EMPTY) {
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
    const int64_t a = __ldg(kb.off + i);
    const KeyRef k(kb.bytes + a, __ldg(kb.off + i + 1) - a);
    uint32_t tag, hb;
    hash_key(k, t.weak, tag, hb);
    if (world > 1 && owner_of(tag, world) != rank) return;
    const int64_t v = ERASE ? -1 : in_vals[i];
    int64_t myrec = -1;  // record allocated for an insert (kept across lost CAS races)
    int64_t b = (int64_t)(hb & (uint32_t)(t.nb - 1));
    bool done = false;
    for (int64_t p = 0; p < t.nb && !done; ++p) {
        uint64_t s[4];
        unsigned long long *bk = t.slots + b * KV_BUCKET;
        ld256<true>(bk, s[0], s[1], s[2], s[3]);
        for (int j = 0; j < KV_BUCKET && !done; ++j) {
            uint64_t cur = s[j];
            for (;;) {  // re-examines slot j after a lost CAS
                const uint32_t st = (uint32_t)cur;
                if (st == tag) {
                    __threadfence();  // the record was published before its slot (see insert)
                    int64_t old;
                    const int64_t ro = rec_off_of(cur);
                    if (rec_matches<true>(t.arena + ro, k, &old)) {
                        if (ERASE) {
                            if (atomicCAS(bk + j, cur, (unsigned long long)TAG_TOMB) == cur) {
                                atomicAdd(&t.counts[0], (unsigned long long)-1ll);
                                atomicAdd(&t.counts[1], 1ull);
                                atomicAdd(&t.counts[3], (unsigned long long)rec_bytes(k.len));
                            }
                        } else {
                            atomicMax(reinterpret_cast<long long *>(t.arena + ro), (long long)v);
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
                    myrec = (int64_t)atomicAdd(&t.counts[2], (unsigned long long)rec_bytes(k.len));
                    write_record(t.arena + myrec, k, v);
                    __threadfence();  // publish the record before the slot that points at it
                }
                const unsigned long long want = slot_of(tag, myrec);
                const unsigned long long got = atomicCAS(bk + j, 0ull, want);
                if (got == 0ull) {
                    atomicAdd(&t.counts[0], 1ull);
                    myrec = -1;
                    done = true;
                    break;
                }
                cur = got;  // lost the race: look at what was written there
            }
        }
        b = (b + 1) & (t.nb - 1);
    }
    if (myrec >= 0) atomicAdd(&t.counts[3], (unsigned long long)rec_bytes(k.len));  // lost every race
}

// ---- hashes / shard owners ---------------------------------------------------
__global__ void fingerprint_kernel(KeyBatch kb, uint64_t *__restrict__ fp, int world, int32_t *__restrict__ owner) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < kb.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = kb.off[i];
        const KeyRef k(kb.bytes + a, kb.off[i + 1] - a);
        uint32_t tag, hb;
        hash_key(k, 0, tag, hb);
        if (fp) {
            fp[2 * i] = tag;
            fp[2 * i + 1] = hb;
        }
        if (owner) owner[i] = owner_of(tag, world);
    }
}

// ---- maintenance ---------------------------------------------------------------
__device__ __forceinline__ bool live_slot(uint64_t s) { return ((uint32_t)s & 0x80000000u) != 0; }

__global__ void kv_export_kernel(KvTable t, int64_t nslots, int64_t *val_out, int64_t max, unsigned long long *cursor) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots; s += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t sl = t.slots[s];
        if (live_slot(sl)) {
            unsigned long long p = atomicAdd(cursor, 1ull);
            if ((int64_t)p < max) val_out[p] = *reinterpret_cast<const int64_t *>(t.arena + rec_off_of(sl));
        }
    }
}

__global__ void kv_remap_kernel(KvTable t, int64_t nslots, const int64_t *__restrict__ map, int64_t nmap) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots; s += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t sl = t.slots[s];
        if (live_slot(sl)) {
            int64_t *v = reinterpret_cast<int64_t *>(t.arena + rec_off_of(sl));
            if (*v >= 0 && *v < nmap) *v = map[*v];
        }
    }
}

// rebuild: every live key of the old table is copied into a fresh arena (compacting away
// overwritten/erased records) and re-inserted by its hash (no duplicates exist)
__global__ void kv_rebuild_kernel(const unsigned long long *__restrict__ old_slots, int64_t old_n,
                                  const uint8_t *__restrict__ old_arena, KvTable t) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < old_n; s += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t sl = old_slots[s];
        if (!live_slot(sl)) continue;
        const uint8_t *rec = old_arena + rec_off_of(sl);
        const int64_t len = (int64_t)(uint32_t)reinterpret_cast<const uint64_t *>(rec)[1];
        const int64_t rb = rec_bytes(len);
        const int64_t dst = (int64_t)atomicAdd(&t.counts[2], (unsigned long long)rb);
        for (int64_t o = 0; o < rb; o += 8)
            *reinterpret_cast<uint64_t *>(t.arena + dst + o) = *reinterpret_cast<const uint64_t *>(rec + o);
        const KeyRef k(rec + KV_REC_HDR, len);
        uint32_t tag, hb;
        hash_key(k, t.weak, tag, hb);
        int64_t b = (int64_t)(hb & (uint32_t)(t.nb - 1));
        bool done = false;
        for (int64_t p = 0; p < t.nb && !done; ++p) {
            for (int j = 0; j < KV_BUCKET && !done; ++j) {
                if (atomicCAS(t.slots + b * KV_BUCKET + j, 0ull, slot_of(tag, dst)) == 0ull) {
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
    const int64_t acap = std::min<int64_t>(KV_MAX_ARENA,
                                           std::max<int64_t>(4096, round_up<int64_t>(need_bytes + need_bytes / 2, 256)));
    if (need_bytes > acap) PR_FAIL(PR_ERR_NOMEM, "kv arena: %lld bytes exceed the 128 GiB record space",
                                   (long long)need_bytes);
    unsigned long long *ns = nullptr;
    uint8_t *na = nullptr;
    PR_CUDA(cudaMalloc(&ns, (size_t)nslots * sizeof(unsigned long long)));
    if (cudaMalloc(&na, (size_t)acap) != cudaSuccess) {
        cudaFree(ns);
        cudaGetLastError();
        PR_FAIL(PR_ERR_NOMEM, "kv arena: cannot allocate %lld bytes", (long long)acap);
    }
    PR_CUDA(cudaMemsetAsync(ns, 0, (size_t)nslots * sizeof(unsigned long long), st));
    PR_CUDA(cudaMemsetAsync(h->d_count, 0, 4 * sizeof(unsigned long long), st));
    unsigned long long *os = h->slots;
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
    uint32_t tag, hb;
    hash_host(bytes, len, tag, hb);
    out[0] = tag;
    out[1] = hb;
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

int pr_l2_fetch_granularity(int bytes, int *previous) {
    size_t prev = 0;
    PR_CUDA(cudaDeviceGetLimit(&prev, cudaLimitMaxL2FetchGranularity));
    if (previous) *previous = (int)prev;
    if (bytes > 0) PR_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes));
    return PR_OK;
}

int pr_kv_create(int64_t capacity, pr_kv **out) { return pr_kv_create_ex(capacity, 0, out); }

int pr_kv_create_ex(int64_t capacity, uint32_t flags, pr_kv **out) {
    if (!out || capacity < 0 || (flags & ~PR_KV_WEAK_HASH)) PR_FAIL(PR_ERR_BAD_ARG, "bad kv_create");
    pr_kv *h = new pr_kv();
    h->flags = flags;
    h->nslots = slots_for(capacity);
    h->arena_cap = std::max<int64_t>(4096, capacity * 48);
    if (cudaMalloc(&h->slots, (size_t)h->nslots * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&h->arena, (size_t)h->arena_cap) != cudaSuccess ||
        cudaMalloc(&h->d_count, 4 * sizeof(unsigned long long)) != cudaSuccess) {
        cudaFree(h->slots);
        cudaFree(h->arena);
        delete h;
        cudaGetLastError();
        PR_FAIL(PR_ERR_NOMEM, "kv_create: device allocation failed");
    }
    PR_CUDA(cudaMemset(h->slots, 0, (size_t)h->nslots * sizeof(unsigned long long)));
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
    PR_CUDA(cudaMemsetAsync(h->slots, 0, (size_t)h->nslots * sizeof(unsigned long long), st));
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
    if (slot_bytes) *slot_bytes = h->nslots * (int64_t)sizeof(unsigned long long);
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
