// Fixed KV cache on the GPU (reference: caches.py:45-101, FixedKVCache).
//
// The reference keys a dict by the raw query text: any one-byte difference is a
// different key (caches.py:57-65, tests/test_caches.py:36-45).  This table
// is byte-exact the same way: a hit is confirmed against the stored key bytes, so a hash
// collision (accidental or constructed) can only cost a probe, never serve another key's
// answer.
//
// Why the layout is what it is (measured on B200, scripts/micro/{randline,kvbench,kvslot}.cu):
// * a random read costs one 128-byte line of DRAM whatever its width, and HBM3e serves
//   ~45 G random lines/s (5.8 TB/s) — random lines are NOT the problem;
// * two or more loads in flight to the same missing line are far slower than one (three
//   16-byte loads of one line: 12 G lookups/s vs 24), and a dependent second access to a
//   line just fetched (an L2 hit) still costs a full L2 round trip per lookup;
// so a lookup should be ONE load of ONE sector.  The table is an array of 32-byte SLOTS
// (one sector each, nslots a power of two, load <= 3/8), probed with one 256-bit load:
//
//   slot   [0,16) key prefix (zero padded; keys <= 16 bytes live here whole)
//          [16,24) u64 len (24 bits) | value << 24
//          [24,28) u32 tag: 0 = EMPTY, 1 = TOMBSTONE, 2 = BUSY (claimed, being written),
//                  else the 32-bit key hash with its top bit set
//          [28,32) u32 record index of a key longer than 16 bytes, in 32-byte units
//   arena  32-byte aligned records: the full bytes of keys longer than 16 bytes.
//
// A key of <= 16 bytes is confirmed byte for byte from the slot it loaded (tag, length and
// the 16 bytes); a longer key also compares its tail against its record.  Linear probing by
// slot: at load <= 3/8 most keys are found (or proven absent by an EMPTY slot) in the home
// slot, and the next slot is the adjacent sector of the same line.  Round 2's 128-byte
// bucket lines (tag vector first, slot body on a match) ran 24 G lookups/s at 4M-key
// batches; one 32-byte slot per load runs ~32 G at this load (kvslot.cu).
// Hash: two 32-bit multiply-rotate chains over the key's little-endian words (murmur3_32
// round function, two seeds).  hA -> tag (and shard owner), hB -> home slot: the
// ownership bits and the slot bits come from independent chains.  Only 32-bit integer
// multiplies: the hash is a short dependency chain per key.
//
// One thread per key: it hashes its key ONCE (aligned 32-bit loads + funnel shifts, not
// byte loads), so a warp keeps 32 independent slots in flight.  Values are write sequence
// numbers supplied by the host; a put resolves an existing key with atomicMax on len|value,
// so the largest (latest) write wins even when one batch writes a key twice
// (caches.py:67-74).
#include <algorithm>

#include "common.cuh"

struct pr_kv {
    uint8_t *lines = nullptr;               // [nslots] 32-byte slots
    int64_t nslots = 0;
    uint8_t *arena = nullptr;               // records
    int64_t arena_cap = 0;                  // bytes
    unsigned long long *d_count = nullptr;  // [0] live [1] tombstones [2] arena cursor [3] garbage bytes
    int64_t upper = 0;                      // host bound on live + tombstones (no sync needed)
    int64_t arena_upper = 0;                // host bound on the arena cursor
    uint32_t flags = 0;                     // PR_KV_WEAK_HASH (tests only)
};

namespace pr {

constexpr int KV_THREADS = 128;
constexpr int KV_INLINE = 16;                        // key bytes held in the slot
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

// record bytes of a key (keys <= 16 bytes live entirely in their slot)
__host__ __device__ __forceinline__ int64_t rec_bytes(int64_t len) {
    return len > KV_INLINE ? round_up<int64_t>(len, 32) : 0;
}

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
        last = n > 0 ? ((int64_t)(u & 3) + n - 1) >> 2 : -1;
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

// Hash a key and return its first four words (the slot's inline prefix).
__device__ __forceinline__ void hash_key(const KeyRef &k, int weak, uint32_t &tag, uint32_t &hb, uint32_t pw[4]) {
    KeyHash h;
    h.init(k.len);
    const int64_t nw = (k.len + 3) >> 2;
    uint32_t lo = k.ld(0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t hi = k.ld(j + 1);
        pw[j] = k.join(lo, hi, j);
        if (j < nw) h.word(pw[j]);
        lo = hi;
    }
    for (int64_t j = 4; j < nw; ++j) {
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

// hash of a key held inline in a slot (<= 16 bytes: words w2 | w3, zero padded)
__device__ __forceinline__ void hash_inline(uint64_t w2, uint64_t w3, int64_t len, int weak, uint32_t &tag,
                                            uint32_t &hb) {
    const uint32_t w[4] = {(uint32_t)w2, (uint32_t)(w2 >> 32), (uint32_t)w3, (uint32_t)(w3 >> 32)};
    KeyHash h;
    h.init(len);
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (4 * j < len) h.word(w[j]);
    h.fin(len, tag, hb);
    if (weak) {
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

// One 32-byte slot (see the file comment): prefix | len|value | tag | record index.
constexpr uint32_t TAG_BUSY = 2;
constexpr int64_t KV_SLOT = 32;

__host__ __device__ __forceinline__ uint64_t pack_lv(int64_t len, int64_t val) {
    return (uint64_t)len | ((uint64_t)val << 24);
}

struct KvTable {
    uint8_t *slots;  // [ns][32]
    int64_t ns;      // slots (power of two)
    uint8_t *arena;
    unsigned long long *counts;
    int weak;  // PR_KV_WEAK_HASH: 2-bit tags, 4 home slots (forces collisions; tests only)
    __device__ __forceinline__ uint8_t *slot(int64_t s) const { return slots + s * KV_SLOT; }
    __device__ __forceinline__ uint4 *prefix(int64_t s) const { return reinterpret_cast<uint4 *>(slot(s)); }
    __device__ __forceinline__ unsigned long long *lv(int64_t s) const {
        return reinterpret_cast<unsigned long long *>(slot(s) + 16);
    }
    __device__ __forceinline__ uint32_t *tag(int64_t s) const { return reinterpret_cast<uint32_t *>(slot(s) + 24); }
    __device__ __forceinline__ uint32_t *rec(int64_t s) const { return reinterpret_cast<uint32_t *>(slot(s) + 28); }
};

struct KeyBatch {
    const uint8_t *bytes;
    const int64_t *off;
    int64_t n;
};

template <bool STRONG>
__device__ __forceinline__ uint4 ld4(const void *p) {
    uint4 v;
    if (STRONG)
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    else
        asm("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
template <bool STRONG>
__device__ __forceinline__ uint64_t ld8(const void *p) {
    uint64_t v;
    if (STRONG)
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else
        asm("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
template <bool STRONG>
__device__ __forceinline__ uint32_t ld4b(const void *p) {
    uint32_t v;
    if (STRONG)
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    else
        asm("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// bytes [16, len) of a long key against its record (the record holds the whole key)
template <bool STRONG>
__device__ __forceinline__ bool tail_matches(const uint8_t *rec, const KeyRef &k) {
    for (int64_t g = 1; 16 * g < k.len; ++g) {
        const uint4 r = ld4<STRONG>(rec + 16 * g);
        if (r.x != k.word(4 * g) || r.y != k.word(4 * g + 1) || r.z != k.word(4 * g + 2) || r.w != k.word(4 * g + 3))
            return false;
    }
    return true;
}

// slot s carries the key's tag: does it hold the key?  *val = its value if so.
template <bool STRONG>
__device__ __forceinline__ bool slot_holds(const KvTable &t, int64_t s, const KeyRef &k, const uint32_t pw[4],
                                           int64_t *val) {
    const uint64_t lv = ld8<STRONG>(t.lv(s));
    const uint4 pre = ld4<STRONG>(t.prefix(s));
    if ((int64_t)(lv & 0xffffffull) != k.len || pre.x != pw[0] || pre.y != pw[1] || pre.z != pw[2] || pre.w != pw[3])
        return false;
    if (k.len > KV_INLINE && !tail_matches<STRONG>(t.arena + ((int64_t)ld4b<STRONG>(t.rec(s)) << 5), k))
        return false;
    *val = (int64_t)(lv >> 24);
    return true;
}

// the whole slot in one 256-bit load (one sector)
__device__ __forceinline__ void ld_slot(const uint8_t *p, uint64_t &w0, uint64_t &w1, uint64_t &w2, uint64_t &w3) {
    asm("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3) : "l"(p));
}

// ---- get: one thread per key, one 32-byte slot per probe step ----------------
__global__ void __launch_bounds__(KV_THREADS) kv_get_kernel(KvTable t, KeyBatch kb, int rank, int world,
                                                             int64_t *__restrict__ out_vals,
                                                             uint8_t *__restrict__ out_hit) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= kb.n) return;
    const int64_t a = __ldg(kb.off + i);
    const KeyRef k(kb.bytes + a, __ldg(kb.off + i + 1) - a);
    uint32_t tag, hb, pw[4];
    hash_key(k, t.weak, tag, hb, pw);
    int64_t val = -1;
    if (world <= 1 || owner_of(tag, world) == rank) {
        const uint64_t k0 = ((uint64_t)pw[1] << 32) | pw[0], k1 = ((uint64_t)pw[3] << 32) | pw[2];
        int64_t s = (int64_t)(hb & (uint32_t)(t.ns - 1));
        for (int64_t p = 0; p < t.ns; ++p) {
            uint64_t w0, w1, w2, w3;
            ld_slot(t.slot(s), w0, w1, w2, w3);
            const uint32_t st = (uint32_t)w3;
            if (st == TAG_EMPTY) break;
            if (st == tag && w0 == k0 && w1 == k1 && (int64_t)(w2 & 0xffffffull) == k.len &&
                (k.len <= KV_INLINE || tail_matches<false>(t.arena + ((int64_t)(uint32_t)(w3 >> 32) << 5), k))) {
                val = (int64_t)(w2 >> 24);
                break;
            }
            s = (s + 1) & (t.ns - 1);
        }
    }
    out_vals[i] = val;
    out_hit[i] = val >= 0;
}

// copy a long key into a fresh record (zero padded to its 32-byte record size)
__device__ void write_record(uint8_t *rec, const KeyRef &k) {
    uint32_t *w = reinterpret_cast<uint32_t *>(rec);
    const int64_t words = rec_bytes(k.len) / 4;
    for (int64_t j = 0; j < words; ++j) w[j] = k.word(j);
}

// fill a claimed slot and publish its tag (the slot's other fields become visible first)
__device__ __forceinline__ void publish(const KvTable &t, int64_t s, uint32_t tag, uint32_t rec, uint64_t lv,
                                        uint4 pre) {
    *t.rec(s) = rec;
    *t.lv(s) = lv;
    *t.prefix(s) = pre;
    __threadfence();
    atomicExch(t.tag(s), tag);
}

// ---- put (upsert) / erase: one thread per key --------------------------------
// Insert protocol: CAS tag EMPTY -> BUSY; write rec, lv, prefix (+ the record of a long
// key); fence; publish the tag.  A thread that meets a BUSY slot waits for its
// publication before comparing (duplicates of one new key inside one batch).
template <bool ERASE>
__global__ void __launch_bounds__(KV_THREADS) kv_update_kernel(KvTable t, KeyBatch kb, int rank, int world,
                                                                const int64_t *__restrict__ in_vals) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= kb.n) return;
    const int64_t a = __ldg(kb.off + i);
    const KeyRef k(kb.bytes + a, __ldg(kb.off + i + 1) - a);
    uint32_t tag, hb, pw[4];
    hash_key(k, t.weak, tag, hb, pw);
    if (world > 1 && owner_of(tag, world) != rank) return;
    const int64_t v = ERASE ? -1 : in_vals[i];
    int64_t s = (int64_t)(hb & (uint32_t)(t.ns - 1));
    for (int64_t p = 0; p < t.ns; ++p) {
        uint32_t cur = ld4b<true>(t.tag(s));
        for (;;) {  // re-examines slot s after a lost CAS / a pending publication
            if (cur == TAG_BUSY) {
                do {
                    __nanosleep(32);
                    cur = ld4b<true>(t.tag(s));
                } while (cur == TAG_BUSY);
                continue;
            }
            if (cur == tag) {
                __threadfence();  // pairs with publish(): the slot's fields are visible
                int64_t old;
                if (slot_holds<true>(t, s, k, pw, &old)) {
                    if (ERASE) {
                        if (atomicCAS(t.tag(s), tag, TAG_TOMB) == tag) {
                            atomicAdd(&t.counts[0], (unsigned long long)-1ll);
                            atomicAdd(&t.counts[1], 1ull);
                            atomicAdd(&t.counts[3], (unsigned long long)rec_bytes(k.len));
                        }
                    } else {
                        atomicMax(t.lv(s), (unsigned long long)pack_lv(k.len, v));
                    }
                    return;
                }
                break;  // same tag, another key
            }
            if (cur != TAG_EMPTY) break;  // another key or a tombstone: next slot
            if (ERASE) return;            // first empty slot: the key is absent
            const uint32_t got = atomicCAS(t.tag(s), TAG_EMPTY, TAG_BUSY);
            if (got != TAG_EMPTY) {  // lost the race: look at what was claimed there
                cur = got;
                continue;
            }
            int64_t rec = 0;
            if (k.len > KV_INLINE) {
                rec = (int64_t)atomicAdd(&t.counts[2], (unsigned long long)rec_bytes(k.len));
                write_record(t.arena + rec, k);
            }
            publish(t, s, tag, (uint32_t)(rec >> 5), pack_lv(k.len, v), make_uint4(pw[0], pw[1], pw[2], pw[3]));
            atomicAdd(&t.counts[0], 1ull);
            return;
        }
        s = (s + 1) & (t.ns - 1);
    }
}

// ---- hashes / shard owners ---------------------------------------------------
__global__ void fingerprint_kernel(KeyBatch kb, uint64_t *__restrict__ fp, int world, int32_t *__restrict__ owner) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < kb.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = kb.off[i];
        const KeyRef k(kb.bytes + a, kb.off[i + 1] - a);
        uint32_t tag, hb, pw[4];
        hash_key(k, 0, tag, hb, pw);
        if (fp) {
            fp[2 * i] = tag;
            fp[2 * i + 1] = hb;
        }
        if (owner) owner[i] = owner_of(tag, world);
    }
}

// ---- maintenance (one thread per slot) -------------------------------------------
__device__ __forceinline__ bool live_tag(uint32_t tag) { return (tag & 0x80000000u) != 0; }

__global__ void kv_export_kernel(KvTable t, int64_t nslots, int64_t *val_out, int64_t max, unsigned long long *cursor) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots; s += (int64_t)gridDim.x * blockDim.x) {
        if (live_tag(*t.tag(s))) {
            unsigned long long p = atomicAdd(cursor, 1ull);
            if ((int64_t)p < max) val_out[p] = (int64_t)(*t.lv(s) >> 24);
        }
    }
}

__global__ void kv_remap_kernel(KvTable t, int64_t nslots, const int64_t *__restrict__ map, int64_t nmap) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots; s += (int64_t)gridDim.x * blockDim.x) {
        if (live_tag(*t.tag(s))) {
            const uint64_t lv = *t.lv(s);
            const int64_t v = (int64_t)(lv >> 24);
            if (v >= 0 && v < nmap) *t.lv(s) = pack_lv((int64_t)(lv & 0xffffffull), map[v]);
        }
    }
}

// rebuild: every live key of the old table is re-inserted by its hash into a fresh table
// (no duplicates exist); long keys' records move into a fresh, compacted arena
__global__ void kv_rebuild_kernel(KvTable o, int64_t old_slots, KvTable t) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < old_slots; s += (int64_t)gridDim.x * blockDim.x) {
        if (!live_tag(*o.tag(s))) continue;
        const uint64_t lv = *o.lv(s);
        const uint4 pre = *o.prefix(s);
        const int64_t len = (int64_t)(lv & 0xffffffull);
        int64_t rec = 0;
        uint32_t tag, hb, pw[4];
        if (len > KV_INLINE) {
            const uint8_t *src = o.arena + ((int64_t)*o.rec(s) << 5);
            const int64_t rb = rec_bytes(len);
            rec = (int64_t)atomicAdd(&t.counts[2], (unsigned long long)rb);
            for (int64_t x = 0; x < rb; x += 8)
                *reinterpret_cast<uint64_t *>(t.arena + rec + x) = *reinterpret_cast<const uint64_t *>(src + x);
            hash_key(KeyRef(src, len), t.weak, tag, hb, pw);
        } else {
            hash_inline((uint64_t)pre.x | ((uint64_t)pre.y << 32), (uint64_t)pre.z | ((uint64_t)pre.w << 32), len,
                        t.weak, tag, hb);
        }
        int64_t q = (int64_t)(hb & (uint32_t)(t.ns - 1));
        for (int64_t p = 0; p < t.ns; ++p) {
            if (atomicCAS(t.tag(q), TAG_EMPTY, TAG_BUSY) == TAG_EMPTY) {
                publish(t, q, tag, (uint32_t)(rec >> 5), lv, pre);
                atomicAdd(&t.counts[0], 1ull);
                break;
            }
            q = (q + 1) & (t.ns - 1);
        }
    }
}

// sizing: at most 3/16 full when built for `keys` (100M keys -> 2^29 slots, 17 GB); a put
// that would pass 3/8 (live + tombstones) rebuilds at twice the size
static int64_t slots_for(int64_t keys) {
    int64_t s = 1024;
    while (3 * s < 16 * keys) s *= 2;
    return s;
}
static bool over_load(int64_t used, int64_t nslots) { return 8 * used > 3 * nslots; }

static KvTable table_of(pr_kv *h) {
    return KvTable{h->lines, h->nslots, h->arena, h->d_count, (h->flags & PR_KV_WEAK_HASH) ? 1 : 0};
}

static int read_counts(pr_kv *h, unsigned long long c[4], cudaStream_t st) {
    PR_CUDA(cudaMemcpyAsync(c, h->d_count, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    PR_CUDA(cudaStreamSynchronize(st));
    return PR_OK;
}

constexpr int64_t KV_SLOT_BYTES = 32;
constexpr int64_t KV_ARENA_BASE = 32;  // record index 0 means "no record"

// Rebuild into a table for `need_keys` live keys and an arena of `need_bytes` live record
// bytes (drops tombstones and garbage records).  Synchronises the device: rare.
static int rebuild(pr_kv *h, int64_t need_keys, int64_t need_bytes, cudaStream_t st) {
    unsigned long long c[4];
    int rc = read_counts(h, c, st);
    if (rc) return rc;
    PR_CUDA(cudaDeviceSynchronize());
    const int64_t live = (int64_t)c[0];
    const int64_t live_bytes = (int64_t)c[2] - KV_ARENA_BASE - (int64_t)c[3];
    const int64_t nslots = slots_for(std::max<int64_t>(need_keys, live));
    const int64_t acap = std::min<int64_t>(KV_MAX_ARENA, std::max<int64_t>(
                                                             4096, round_up<int64_t>(need_bytes + need_bytes / 2, 256)));
    if (need_bytes > acap) PR_FAIL(PR_ERR_NOMEM, "kv arena: %lld bytes exceed the 128 GiB record space",
                                   (long long)need_bytes);
    uint8_t *ns = nullptr;
    uint8_t *na = nullptr;
    PR_CUDA(cudaMalloc(&ns, (size_t)nslots * KV_SLOT_BYTES));
    if (cudaMalloc(&na, (size_t)acap) != cudaSuccess) {
        cudaFree(ns);
        cudaGetLastError();
        PR_FAIL(PR_ERR_NOMEM, "kv arena: cannot allocate %lld bytes", (long long)acap);
    }
    PR_CUDA(cudaMemsetAsync(ns, 0, (size_t)nslots * KV_SLOT_BYTES, st));
    const unsigned long long c0[4] = {0, 0, (unsigned long long)KV_ARENA_BASE, 0};
    PR_CUDA(cudaMemcpyAsync(h->d_count, c0, sizeof(c0), cudaMemcpyHostToDevice, st));
    const KvTable old = table_of(h);
    uint8_t *os = h->lines;
    uint8_t *oa = h->arena;
    const int64_t on = h->nslots;
    h->lines = ns;
    h->nslots = nslots;
    h->arena = na;
    h->arena_cap = acap;
    if (live > 0) {
        const int g = (int)std::min<int64_t>(ceil_div<int64_t>(on, 256), (int64_t)sm_count() * 16);
        ::pr::count_launch();
        kv_rebuild_kernel<<<g, 256, 0, st>>>(old, on, table_of(h));
        PR_LAUNCH_CHECK();
    }
    PR_CUDA(cudaStreamSynchronize(st));
    cudaFree(os);
    cudaFree(oa);
    h->upper = live;
    h->arena_upper = KV_ARENA_BASE + live_bytes;
    return PR_OK;
}

// a larger record arena; record indices stay valid (the used prefix is copied)
static int grow_arena(pr_kv *h, int64_t need, cudaStream_t st) {
    const int64_t cap = std::min<int64_t>(KV_MAX_ARENA, round_up<int64_t>(std::max<int64_t>(need + need / 2, 1 << 16), 256));
    if (need > cap) PR_FAIL(PR_ERR_NOMEM, "kv arena: %lld bytes exceed the 128 GiB record space", (long long)need);
    uint8_t *na = nullptr;
    if (cudaMalloc(&na, (size_t)cap) != cudaSuccess) {
        cudaGetLastError();
        PR_FAIL(PR_ERR_NOMEM, "kv arena: cannot allocate %lld bytes", (long long)cap);
    }
    PR_CUDA(cudaMemcpyAsync(na, h->arena, (size_t)h->arena_upper, cudaMemcpyDeviceToDevice, st));
    PR_CUDA(cudaStreamSynchronize(st));
    PR_CUDA(cudaDeviceSynchronize());  // no other stream may still read the old arena
    cudaFree(h->arena);
    h->arena = na;
    h->arena_cap = cap;
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
    const int64_t rec_need = n * 31 + nbytes;  // >= sum of rec_bytes over the batch
    if (over_load(h->upper + n, h->nslots) || h->arena_upper + rec_need > h->arena_cap) {
        unsigned long long c[4];
        rc = read_counts(h, c, st);
        if (rc) return rc;
        h->upper = (int64_t)(c[0] + c[1]);
        h->arena_upper = (int64_t)c[2];
        const bool slots_short = over_load(h->upper + n, h->nslots);
        const bool arena_short = h->arena_upper + rec_need > h->arena_cap;
        if (slots_short) {
            rc = rebuild(h, (int64_t)c[0] + n, (int64_t)(c[2] - c[3]) - KV_ARENA_BASE + rec_need, st);
            if (rc) return rc;
        } else if (arena_short) {
            rc = grow_arena(h, h->arena_upper + rec_need, st);
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
    h->arena_cap = 1 << 16;  // records exist only for keys longer than 16 bytes; grown on demand
    if (cudaMalloc(&h->lines, (size_t)h->nslots * KV_SLOT_BYTES) != cudaSuccess ||
        cudaMalloc(&h->arena, (size_t)h->arena_cap) != cudaSuccess ||
        cudaMalloc(&h->d_count, 4 * sizeof(unsigned long long)) != cudaSuccess) {
        cudaFree(h->lines);
        cudaFree(h->arena);
        delete h;
        cudaGetLastError();
        PR_FAIL(PR_ERR_NOMEM, "kv_create: device allocation failed");
    }
    PR_CUDA(cudaMemset(h->lines, 0, (size_t)h->nslots * KV_SLOT_BYTES));
    const unsigned long long c0[4] = {0, 0, (unsigned long long)KV_ARENA_BASE, 0};
    PR_CUDA(cudaMemcpy(h->d_count, c0, sizeof(c0), cudaMemcpyHostToDevice));
    h->arena_upper = KV_ARENA_BASE;
    PR_CUDA(cudaDeviceSynchronize());
    *out = h;
    return PR_OK;
}

int pr_kv_destroy(pr_kv *h) {
    if (!h) return PR_OK;
    cudaDeviceSynchronize();
    cudaFree(h->lines);
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
    PR_CUDA(cudaMemsetAsync(h->lines, 0, (size_t)h->nslots * KV_SLOT_BYTES, st));
    // the counts are reset by a tiny kernel-free copy from a static host block (stream ordered)
    static const unsigned long long c0[4] = {0, 0, (unsigned long long)KV_ARENA_BASE, 0};
    PR_CUDA(cudaMemcpyAsync(h->d_count, c0, sizeof(c0), cudaMemcpyHostToDevice, st));
    h->upper = 0;
    h->arena_upper = KV_ARENA_BASE;
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
    if (slot_bytes) *slot_bytes = h->nslots * KV_SLOT_BYTES;
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
