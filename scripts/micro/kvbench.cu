// Standalone harness for the KV probe kernel (includes the library's kv.cu) and two
// diagnostics: the front half alone (offsets, key words, hash) and + the home-slot load.
// Round-2 results of the 128-byte bucket-line layout and its variants are in
// profiles/r02_kv_layout_experiments.txt.
// Builds a 100M-key table of "query-%09d" keys through pr_kv_put_text, then times
// lookups: B=65536 batches on S concurrent streams (graph-free, back to back) and one
// 4M-key batch, for each variant.  Parity is checked for every variant.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <string>

#include "../../paper_2506_21593_b200/csrc/kv.cu"

namespace pr {
void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vfprintf(stderr, fmt, ap);
    va_end(ap);
    fprintf(stderr, "\n");
}
const char *last_error() { return ""; }
void count_launch() {}
int sm_count() { return 148; }


// software-pipelined grid-stride loop: key j's slot load is in flight while key j+1's
// offsets / key words load and hash
struct FH {
    int64_t len, a;
    uint32_t tag, hb;
    uint64_t k0, k1;
};
__device__ __forceinline__ FH front(const KvTable &t, const KeyBatch &kb, int64_t i) {
    FH f;
    f.a = __ldg(kb.off + i);
    f.len = __ldg(kb.off + i + 1) - f.a;
    const KeyRef k(kb.bytes + f.a, f.len);
    uint32_t pw[4];
    hash_key(k, t.weak, f.tag, f.hb, pw);
    f.k0 = ((uint64_t)pw[1] << 32) | pw[0];
    f.k1 = ((uint64_t)pw[3] << 32) | pw[2];
    return f;
}
__global__ void __launch_bounds__(KV_THREADS) get_pipe(KvTable t, KeyBatch kb, int64_t *out_vals, uint8_t *out_hit) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= kb.n) return;
    FH f = front(t, kb, i);
    while (true) {
        int64_t s = (int64_t)(f.hb & (uint32_t)(t.ns - 1));
        uint64_t w0, w1, w2, w3;
        ld_slot(t.slot(s), w0, w1, w2, w3);
        const int64_t i2 = i + T;
        FH g;
        if (i2 < kb.n) g = front(t, kb, i2);
        int64_t val = -1;
        for (int64_t p = 0; p < t.ns; ++p) {
            const uint32_t st = (uint32_t)w3;
            if (st == TAG_EMPTY) break;
            if (st == f.tag && w0 == f.k0 && w1 == f.k1 && (int64_t)(w2 & 0xffffffull) == f.len &&
                (f.len <= KV_INLINE ||
                 tail_matches<false>(t.arena + ((int64_t)(uint32_t)(w3 >> 32) << 5), KeyRef(kb.bytes + f.a, f.len)))) {
                val = (int64_t)(w2 >> 24);
                break;
            }
            s = (s + 1) & (t.ns - 1);
            ld_slot(t.slot(s), w0, w1, w2, w3);
        }
        out_vals[i] = val;
        out_hit[i] = val >= 0;
        if (i2 >= kb.n) break;
        i = i2;
        f = g;
    }
}

// diagnostics (wrong results by design): the front half alone (offsets, key words, hash)
// and the front half + the tag-vector load (no slot body)
template <int TAGS>
__global__ void __launch_bounds__(KV_THREADS) get_diag(KvTable t, KeyBatch kb, int64_t *out_vals, uint8_t *out_hit) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= kb.n) return;
    const int64_t a = __ldg(kb.off + i);
    const KeyRef k(kb.bytes + a, __ldg(kb.off + i + 1) - a);
    uint32_t tag, hb, pw[4];
    hash_key(k, t.weak, tag, hb, pw);
    int64_t v = tag ^ pw[0];
    if (TAGS) {
        const uint4 tg = ld4<false>(t.slot((int64_t)(hb & (uint32_t)(t.ns - 1))));
        v ^= tg.x ^ tg.y ^ tg.z ^ tg.w;
    }
    out_vals[i] = v;
    out_hit[i] = v & 1;
}
}  // namespace pr

using namespace pr;

static void key_arena(const std::vector<int64_t> &ids, std::vector<uint8_t> &buf, std::vector<int64_t> &off) {
    buf.clear();
    off.assign(1, 0);
    char tmp[32];
    for (int64_t id : ids) {
        int n = snprintf(tmp, sizeof tmp, "query-%09lld", (long long)id);
        buf.insert(buf.end(), tmp, tmp + n);
        off.push_back((int64_t)buf.size());
    }
}

int main(int argc, char **argv) {
    const int64_t nkeys = argc > 1 ? atoll(argv[1]) : 100000000;
    pr_kv *h;
    if (pr_kv_create(nkeys, &h)) return 1;
    const int64_t chunk = 8000000;
    uint8_t *dbuf; int64_t *doff, *dval;
    cudaMalloc(&dbuf, chunk * 16 + 64); cudaMalloc(&doff, (chunk + 1) * 8); cudaMalloc(&dval, chunk * 8);
    std::vector<uint8_t> buf; std::vector<int64_t> off, ids;
    for (int64_t c0 = 0; c0 < nkeys; c0 += chunk) {
        const int64_t m = std::min(chunk, nkeys - c0);
        ids.resize(m);
        for (int64_t i = 0; i < m; ++i) ids[i] = c0 + i;
        key_arena(ids, buf, off);
        cudaMemcpy(dbuf, buf.data(), buf.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(doff, off.data(), off.size() * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dval, ids.data(), m * 8, cudaMemcpyHostToDevice);
        if (pr_kv_put_text(h, dbuf, doff, m, (int64_t)buf.size(), dval, nullptr)) return 2;
    }
    cudaDeviceSynchronize();
    printf("built %lld keys, size %lld\n", (long long)nkeys, (long long)pr_kv_size(h, nullptr));
    // lookup batches: 32 x 65536 + one 4M
    const int nb = 32, B = 65536, BIG = 4 << 20;
    srand(3);
    std::vector<uint8_t *> bb(nb + 1); std::vector<int64_t *> bo(nb + 1), bv(nb + 1), want(nb + 1);
    std::vector<uint8_t *> bh(nb + 1);
    std::vector<std::vector<int64_t>> wants(nb + 1);
    for (int j = 0; j <= nb; ++j) {
        const int64_t m = j < nb ? B : BIG;
        ids.resize(m);
        for (int64_t i = 0; i < m; ++i) {
            uint64_t r = ((uint64_t)rand() << 31) ^ (uint64_t)rand();
            ids[i] = (i & 1) ? (int64_t)(r % nkeys) : nkeys + (int64_t)(r % nkeys);
        }
        key_arena(ids, buf, off);
        cudaMalloc(&bb[j], buf.size() + 64); cudaMalloc(&bo[j], off.size() * 8);
        cudaMalloc(&bv[j], m * 8); cudaMalloc(&bh[j], m);
        cudaMemcpy(bb[j], buf.data(), buf.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(bo[j], off.data(), off.size() * 8, cudaMemcpyHostToDevice);
        wants[j].resize(m);
        for (int64_t i = 0; i < m; ++i) wants[j][i] = ids[i] < nkeys ? ids[i] : -1;
    }
    KvTable t = table_of(h);
    const int S = 8;
    cudaStream_t st[S];
    for (int s = 0; s < S; ++s) cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto launch = [&](int v, int j, cudaStream_t s) {
        const int64_t m = j < nb ? B : BIG;
        KeyBatch kb{bb[j], bo[j], m};
        const unsigned g = (unsigned)((m + KV_THREADS - 1) / KV_THREADS);
        if (v == 0) kv_get_kernel<<<g, KV_THREADS, 0, s>>>(t, kb, 0, 1, bv[j], bh[j]);
        if (v == 30) get_pipe<<<std::min<unsigned>(g, 148 * 16), KV_THREADS, 0, s>>>(t, kb, bv[j], bh[j]);
        if (v == 31) get_pipe<<<std::min<unsigned>(g, 148 * 8), KV_THREADS, 0, s>>>(t, kb, bv[j], bh[j]);
        if (v == 32) get_pipe<<<(g + 1) / 2, KV_THREADS, 0, s>>>(t, kb, bv[j], bh[j]);
        if (v == 11) get_diag<0><<<g, KV_THREADS, 0, s>>>(t, kb, bv[j], bh[j]);
        if (v == 12) get_diag<1><<<g, KV_THREADS, 0, s>>>(t, kb, bv[j], bh[j]);
    };
    for (int v : {0, 30, 31, 32}) {
        for (int ns : {1, 8}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaDeviceSynchronize();
                cudaEventRecord(e0, st[0]);
                for (int s = 1; s < ns; ++s) cudaStreamWaitEvent(st[s], e0, 0);
                for (int it = 0; it < 5; ++it)
                    for (int j = 0; j < nb; ++j) launch(v, j, st[j % ns]);
                cudaEvent_t ej[S];
                for (int s = 1; s < ns; ++s) { cudaEventCreate(&ej[s]); cudaEventRecord(ej[s], st[s]); cudaStreamWaitEvent(st[0], ej[s], 0); }
                cudaEventRecord(e1, st[0]);
                cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (rep) printf("variant %d streams %d: %.2f us/batch  %.2f G lookups/s\n", v, ns, ms * 1e3 / (5 * nb),
                                5.0 * nb * B / (ms * 1e-3) / 1e9);
            }
        }
        for (int rep = 0; rep < 2; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(e0, st[0]);
            launch(v, nb, st[0]);
            cudaEventRecord(e1, st[0]);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("variant %d big batch: %.1f us  %.2f G lookups/s\n", v, ms * 1e3, BIG / (ms * 1e-3) / 1e9);
        }
        // parity
        long long bad = 0;
        for (int j = 0; j <= nb; ++j) {
            const int64_t m = j < nb ? B : BIG;
            std::vector<int64_t> got(m);
            cudaMemcpy(got.data(), bv[j], m * 8, cudaMemcpyDeviceToHost);
            for (int64_t i = 0; i < m; ++i) bad += got[i] != wants[j][i];
        }
        printf("variant %d mismatches %lld\n", v, bad);
    }
    return 0;
}
