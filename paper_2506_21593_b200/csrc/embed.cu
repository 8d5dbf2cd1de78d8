// Device HashEmbedder (reference: embedding.py:117-160).
//
// embed(text): tokens = re.findall(r"\w+", text); per token
//   h = int.from_bytes(blake2b(b"tok:" + token, digest_size=8, key=HASH_SEED.to_bytes(8, "big")), "big")
//   acc[h % dim] += +1.0 if h >> 63 else -1.0      (fp64)
// then acc / ||acc|| cast to fp32, or — when every sign cancels or there is no
// token — a one-hot at blake2b(b"raw:" + text) with the same bucket/sign rule.
// The accumulators are small integers, so ||acc||² is an exact integer and the
// result is bit-identical to numpy regardless of summation order; division and
// sqrt are IEEE round-to-nearest on both sides.
//
// The GPU handles ASCII texts (where Python's \w is [A-Za-z0-9_]); a text with
// any byte >= 0x80, no bytes at all, or more than EMB_MAXTOK tokens is flagged
// for the host embedder.  One warp per text: lane 0 tokenises, lanes hash
// tokens in parallel, the warp writes the row coalesced.
#include "common.cuh"

namespace pr {

__host__ __device__ __forceinline__ uint64_t rotr64(uint64_t x, int r) { return (x >> r) | (x << (64 - r)); }

__constant__ uint8_t c_sigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};
static const uint8_t h_sigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

__host__ __device__ __forceinline__ uint64_t b2_iv(int i) {
    const uint64_t iv[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                            0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                            0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
    return iv[i];
}

#define B2_G(a, b, c, d, x, y)         \
    do {                               \
        a = a + b + (x);               \
        d = rotr64(d ^ a, 32);         \
        c = c + d;                     \
        b = rotr64(b ^ c, 24);         \
        a = a + b + (y);               \
        d = rotr64(d ^ a, 16);         \
        c = c + d;                     \
        b = rotr64(b ^ c, 63);         \
    } while (0)

__host__ __device__ inline void b2_compress(uint64_t h[8], const uint64_t m[16], uint64_t t, bool last) {
    uint64_t v[16];
    for (int i = 0; i < 8; ++i) {
        v[i] = h[i];
        v[i + 8] = b2_iv(i);
    }
    v[12] ^= t;  // message byte counter (high word stays 0 for our lengths)
    if (last) v[14] = ~v[14];
    for (int r = 0; r < 12; ++r) {
#ifdef __CUDA_ARCH__
        const uint8_t *s = c_sigma[r];
#else
        const uint8_t *s = h_sigma[r];
#endif
        B2_G(v[0], v[4], v[8], v[12], m[s[0]], m[s[1]]);
        B2_G(v[1], v[5], v[9], v[13], m[s[2]], m[s[3]]);
        B2_G(v[2], v[6], v[10], v[14], m[s[4]], m[s[5]]);
        B2_G(v[3], v[7], v[11], v[15], m[s[6]], m[s[7]]);
        B2_G(v[0], v[5], v[10], v[15], m[s[8]], m[s[9]]);
        B2_G(v[1], v[6], v[11], v[12], m[s[10]], m[s[11]]);
        B2_G(v[2], v[7], v[8], v[13], m[s[12]], m[s[13]]);
        B2_G(v[3], v[4], v[9], v[14], m[s[14]], m[s[15]]);
    }
    for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
}

// blake2b(prefix4 + data, digest_size=8, key=8-byte big-endian `key`) as a
// big-endian integer (what int.from_bytes(digest, "big") returns)
__host__ __device__ inline uint64_t b2_hash64(uint64_t key, const char prefix[4], const uint8_t *data, int64_t len) {
    uint64_t h[8];
    for (int i = 0; i < 8; ++i) h[i] = b2_iv(i);
    h[0] ^= 0x01010000ull ^ (8ull << 8) ^ 8ull;  // fanout/depth 1, key length 8, digest length 8
    uint64_t m[16];
    // key block: the 8 key bytes (big-endian serialisation) padded to 128 bytes
    for (int i = 0; i < 16; ++i) m[i] = 0;
    {
        uint64_t w = 0;
        for (int b = 0; b < 8; ++b) w |= ((key >> (8 * (7 - b))) & 0xFFull) << (8 * b);  // bytes k0..k7 little-endian
        m[0] = w;
    }
    const int64_t total = 4 + len;
    b2_compress(h, m, 128, false);  // message is never empty here, so the key block is not last
    uint64_t t = 128;
    int64_t pos = 0;  // position in the (prefix + data) stream
    while (true) {
        const int64_t rem = total - pos;
        const int64_t take = rem < 128 ? rem : 128;
        for (int i = 0; i < 16; ++i) m[i] = 0;
        for (int64_t b = 0; b < take; ++b) {
            const int64_t p = pos + b;
            const uint8_t byte = (p < 4) ? (uint8_t)prefix[p] : data[p - 4];
            m[b >> 3] |= (uint64_t)byte << (8 * (b & 7));
        }
        pos += take;
        t += (uint64_t)take;
        const bool last = pos >= total;
        b2_compress(h, m, t, last);
        if (last) break;
    }
    uint64_t be = 0;  // digest bytes = h[0] little-endian; read them big-endian
    for (int b = 0; b < 8; ++b) be = (be << 8) | ((h[0] >> (8 * b)) & 0xFFull);
    return be;
}

__host__ __device__ __forceinline__ bool is_word_ascii(uint8_t c) {
    return (c >= '0' && c <= '9') || (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_';
}

constexpr int EMB_MAXTOK = 256;
constexpr int EMB_WARPS = 4;

__global__ void __launch_bounds__(EMB_WARPS * 32) hash_embed_kernel(const uint8_t *__restrict__ bytes,
                                                                     const int64_t *__restrict__ off, int64_t n,
                                                                     int dim, uint64_t key, float *__restrict__ out,
                                                                     uint8_t *__restrict__ host_flag) {
    __shared__ int32_t tstart[EMB_WARPS][EMB_MAXTOK];
    __shared__ int32_t tlen[EMB_WARPS][EMB_MAXTOK];
    __shared__ uint64_t thash[EMB_WARPS][EMB_MAXTOK];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t i = (int64_t)blockIdx.x * EMB_WARPS + w; i < n; i += (int64_t)gridDim.x * EMB_WARPS) {
        const uint8_t *s = bytes + off[i];
        const int64_t L = off[i + 1] - off[i];
        int ntok = 0, flag = (L == 0);
        if (lane == 0 && !flag) {
            int64_t p = 0;
            while (p < L) {
                const uint8_t c = s[p];
                if (c >= 0x80) { flag = 1; break; }
                if (is_word_ascii(c)) {
                    int64_t q = p;
                    while (q < L && s[q] < 0x80 && is_word_ascii(s[q])) ++q;
                    if (q < L && s[q] >= 0x80) { flag = 1; break; }
                    if (ntok == EMB_MAXTOK) { flag = 1; break; }
                    tstart[w][ntok] = (int32_t)p;
                    tlen[w][ntok] = (int32_t)(q - p);
                    ++ntok;
                    p = q;
                } else {
                    ++p;
                }
            }
        }
        ntok = __shfl_sync(0xffffffffu, ntok, 0);
        flag = __shfl_sync(0xffffffffu, flag, 0);
        __syncwarp();
        float *row = out + i * (int64_t)dim;
        for (int j = lane; j < dim; j += 32) row[j] = 0.0f;
        if (lane == 0) host_flag[i] = (uint8_t)flag;
        if (flag) continue;
        for (int t = lane; t < ntok; t += 32) thash[w][t] = b2_hash64(key, "tok:", s + tstart[w][t], tlen[w][t]);
        __syncwarp();
        if (lane == 0) {
            // integer accumulators per distinct bucket, in first-appearance order
            int64_t ss = 0;
            for (int t = 0; t < ntok; ++t) {
                const uint64_t h = thash[w][t];
                const int b = (int)(h % (uint64_t)dim);
                bool seen = false;
                for (int u = 0; u < t; ++u)
                    if ((int)(thash[w][u] % (uint64_t)dim) == b) { seen = true; break; }
                if (seen) continue;
                int64_t acc = 0;
                for (int u = t; u < ntok; ++u) {
                    const uint64_t hu = thash[w][u];
                    if ((int)(hu % (uint64_t)dim) == b) acc += (hu >> 63) ? 1 : -1;
                }
                tlen[w][t] = (int32_t)acc;  // reuse: per-first-occurrence bucket total
                tstart[w][t] = b;
                ss += acc * acc;
            }
            if (ss == 0) {
                const uint64_t h = b2_hash64(key, "raw:", s, L);
                row[(int)(h % (uint64_t)dim)] = (h >> 63) ? 1.0f : -1.0f;
            } else {
                const double norm = sqrt((double)ss);
                for (int t = 0; t < ntok; ++t) {
                    const uint64_t h = thash[w][t];
                    const int b = (int)(h % (uint64_t)dim);
                    bool first = true;
                    for (int u = 0; u < t; ++u)
                        if ((int)(thash[w][u] % (uint64_t)dim) == b) { first = false; break; }
                    if (first) row[b] = (float)((double)tlen[w][t] / norm);
                }
            }
        }
        __syncwarp();
    }
}

}  // namespace pr

using namespace pr;

extern "C" {

int pr_hash_embed(const uint8_t *d_bytes, const int64_t *d_off, int64_t n, int dim, uint64_t seed, float *d_out,
                  uint8_t *d_host_flag, void *stream) {
    if (n < 0 || dim < 1) PR_FAIL(PR_ERR_BAD_ARG, "bad hash_embed");
    if (n == 0) return PR_OK;
    const int64_t blocks = ceil_div<int64_t>(n, EMB_WARPS);
    const int grid = (int)(blocks < (int64_t)sm_count() * 16 ? blocks : (int64_t)sm_count() * 16);
    ::pr::count_launch();
    hash_embed_kernel<<<grid, EMB_WARPS * 32, 0, as_stream(stream)>>>(d_bytes, d_off, n, dim, seed, d_out,
                                                                       d_host_flag);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

uint64_t pr_blake2b64_host(uint64_t key, const char *prefix4, const uint8_t *data, int64_t len) {
    return b2_hash64(key, prefix4, data, len);
}

}  // extern "C"
