// Standalone harness for KV probe kernel variants (includes the library's kv.cu).
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


// K keys per thread, interleaved (more independent probes in flight per thread)
template <int K>
__global__ void __launch_bounds__(KV_THREADS) get_multi(KvTable t, KeyBatch kb, int64_t *out_vals, uint8_t *out_hit) {
    const int64_t base = blockIdx.x * (int64_t)blockDim.x * K + threadIdx.x;
    int64_t a[K], len[K];
    uint32_t tag[K], hb[K], pw[K][4];
    bool have[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const int64_t i = base + q * blockDim.x;
        have[q] = i < kb.n;
        a[q] = have[q] ? __ldg(kb.off + i) : 0;
        len[q] = have[q] ? __ldg(kb.off + i + 1) - a[q] : 0;
    }
#pragma unroll
    for (int q = 0; q < K; ++q) hash_key(KeyRef(kb.bytes + a[q], len[q]), t.weak, tag[q], hb[q], pw[q]);
    uint4 tg[K];
    int64_t b[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
        b[q] = (int64_t)(hb[q] & (uint32_t)(t.nb - 1));
        tg[q] = have[q] ? ld4<false>(t.tag(b[q], 0)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < K; ++q) {
        if (!have[q]) continue;
        const KeyRef k(kb.bytes + a[q], len[q]);
        int64_t val = -1;
        int64_t bb = b[q];
        uint4 cur = tg[q];
        for (int64_t p = 0; p < t.nb; ++p) {
            const uint32_t tv[4] = {cur.x, cur.y, cur.z, cur.w};
            bool done = false;
            for (int j = 0; j < KV_BUCKET && !done; ++j) {
                if (tv[j] == tag[q]) {
                    int64_t v;
                    if (slot_holds<false>(t, bb, j, k, pw[q], &v)) { val = v; done = true; }
                } else if (tv[j] == TAG_EMPTY) {
                    done = true;
                }
            }
            if (done) break;
            bb = (bb + 1) & (t.nb - 1);
            cur = ld4<false>(t.tag(bb, 0));
        }
        const int64_t i = base + q * blockDim.x;
        out_vals[i] = val;
        out_hit[i] = val >= 0;
    }
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
        if (v == 2) get_multi<2><<<(unsigned)((m + 2 * KV_THREADS - 1) / (2 * KV_THREADS)), KV_THREADS, 0, s>>>(t, kb, bv[j], bh[j]);
        if (v == 4) get_multi<4><<<(unsigned)((m + 4 * KV_THREADS - 1) / (4 * KV_THREADS)), KV_THREADS, 0, s>>>(t, kb, bv[j], bh[j]);
    };
    for (int v : {0, 2, 4}) {
        for (int ns : {1, 4, 8}) {
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
