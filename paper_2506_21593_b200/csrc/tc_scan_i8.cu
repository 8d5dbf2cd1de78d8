// Int8 tensor-core score + select for FlatIndex.search (index.py:155-189), sm_100a.
//
// The fp16 scan (tc_scan.cu) is tensor-bound at ~0.93 of the sustained fp16
// peak; kind::i8 runs the same contraction at ~1.6x the rate under the 1 kW
// power cap (cuBLAS at the scan's shape: 1802 vs 1136 TOP/s sustained,
// scripts/probe_lowp_peaks.py).  Exactness comes from a rigorous PER-ROW
// bound on the quantisation error and a complete candidate set:
//
//   row r:   x ~= s_r * xq_r      (xq int8, ||xq||_2 <= 2047)   dx_r >= ||x_r - s_r xq_r||_2
//   query q: q ~= t_q * qq       (qq int8)  A_q >= ||t_q qq||_2,  B_q >= ||q - t_q qq||_2
//   acc = qq . xq_r exactly (int32 TMEM accumulator, |acc| < 2^22), ap = t_q s_r acc
//   |q.x_r - ap| <= A_q dx_r + B_q ||x_r|| <= A_q dx_r + C_q,   C_q = B_q max||x|| + rounding slack
//   u_r = ap + A_q dx_r + C_q  >=  exact score of row r (numpy einsum, fp64)
//
//   l_r = ap - A_q dx_r - C_q  <=  exact score of row r
//
// L = the k-th largest l over all rows is a lower bound on the true k-th score
// e_k (k rows score >= L), and so is the exact k-th score of any k distinct
// rows.  Every row of the true top-k (ties included) has u >= exact >= e_k.
// 1) A pilot scan over every 128th 256-row tile keeps per-thread top-k lists of
//    l; the seed kernel scores the best k of them exactly: seeds + a first
//    bound per query.  2) The main scan APPENDS every row with u >= the current
//    bound (the max of the seed bound, the thread's running k-th l, and the
//    running values other CTAs scanning the same query publish in global
//    memory).  3) The post kernel streams the appended rows with u >= the
//    seeds' k-th exact score through an exact running top-k and ranks by
//    (score desc, row asc): the reference's top-k, bit for bit, with no
//    certificate that can fail (only a per-query buffer overflow sends a
//    query to the exact fp64 scan).
#include <cuda.h>

#include <algorithm>
#include <vector>
#include <cmath>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"
#include "select.cuh"
#include "tc_scan.cuh"

namespace pr {

constexpr int I8_BLOCK_K = 128;  // int8 columns per stage = one 128-B swizzle atom
// epilogue: I8_EPI_WARPS warps; with 8, two warps per SM sub-partition split each
// tile's columns (latency hiding), which leaves room for 3 operand stages
constexpr int I8_EPI_WARPS = 8;
constexpr int I8_HALVES = I8_EPI_WARPS / 4;
constexpr int I8_CPW = (TC_BLOCK_N / 32) / I8_HALVES;  // 32-column chunks per epilogue warp per tile
constexpr int I8_STAGES = I8_EPI_WARPS == 8 ? 3 : 4;  // cta_group::1: 48 KB per stage
constexpr int I8_STAGES2 = 5;                          // cta_group::2: 32 KB per stage and CTA
constexpr int I8_EPI = 32 * I8_EPI_WARPS;
constexpr int I8_THREADS = 128 + I8_EPI;
constexpr int I8_A_BYTES = TC_BLOCK_M * I8_BLOCK_K;  // 16 KB
constexpr int I8_B_BYTES = TC_BLOCK_N * I8_BLOCK_K;  // 32 KB
constexpr int I8_META_BYTES = TC_BLOCK_N * 4 * 2 + (int)sizeof(I8TileMeta);  // s_r[256], dx_r[256], tile bounds
constexpr int I8_TMEM_COLS = 512;
constexpr int I8_CAP = 32768;              // appended candidates per query before the exact fallback

// ||qq||_2, ||xq||_2 <= I8_KMAX, so |acc| <= I8_KMAX^2 < 2^22 and the int32 -> fp32
// conversion is exact with one integer add + one fp32 subtract (no XU-pipe I2F)
constexpr double I8_KMAX = 2047.0;
constexpr int32_t I8_MAGIC_I = 0x4B400000;  // bits of 1.5 * 2^23
constexpr float I8_MAGIC_F = 12582912.0f;

// kind::i8 instruction descriptor: D = S32, A,B = signed int8 K-major, N = 256, M = 128
constexpr uint32_t I8_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_BLOCK_N >> 3) << 17) |
                              ((uint32_t)(TC_BLOCK_M >> 4) << 24);

// CG = CTAs per MMA (tcgen05 cta_group): with 2, an SM pair computes a 256-query x
// 256-row tile; each CTA stages its own 128 queries and HALF of the 256 store rows
// ARES (CG == 2, dp128 <= 1024): each CTA's 128-query A tile stays resident in smem for
// the whole item, so per store tile only its half of B streams in (32 instead of 64
// B/clk of TMA ingress per SM at the int8 MMA rate)
constexpr int I8_ARES_BYTES = TC_BLOCK_M * 1024;  // 128 queries x up to 1024 int8 columns
template <int CG, bool ARES = false>
struct I8Cfg {
    static constexpr int STAGES = ARES ? 4 : (CG == 2 ? I8_STAGES2 : I8_STAGES);
    static constexpr int B_ROWS = TC_BLOCK_N / CG;
    static constexpr int B_BYTES = B_ROWS * I8_BLOCK_K;
    static constexpr int A_STAGE_BYTES = ARES ? 0 : I8_A_BYTES;
    static constexpr int A_RES_BYTES = ARES ? I8_ARES_BYTES : 0;
};
// in-kernel exact refiner (warps 2-3): job table + per-query exact lists
constexpr int I8_RQ = 256;
constexpr size_t I8_REFINER_BYTES = (size_t)I8_RQ * 8 + (size_t)TC_BLOCK_M * TC_KP * 4 + (size_t)TC_BLOCK_M * 8 + 64;
// per epilogue warp: queued (query, 8-row group) records awaiting evaluation (16 spill rows x
// 32 ints = 64 records of 8 accumulators) and their {owner lane, chunk, group} tags
constexpr int I8_QCAP = 64;
constexpr size_t I8_QUEUE_BYTES = (size_t)I8_EPI_WARPS * I8_QCAP * 2;
template <int CG, bool ARES = false>
constexpr size_t i8_smem_bytes() {
    using Cf = I8Cfg<CG, ARES>;
    return 1024 + (size_t)Cf::A_RES_BYTES + (size_t)Cf::STAGES * (Cf::A_STAGE_BYTES + Cf::B_BYTES) +
           2 * (size_t)I8_META_BYTES + (size_t)16 * I8_EPI * 4 + 256 + I8_REFINER_BYTES +
           I8_QUEUE_BYTES;
}
static_assert(i8_smem_bytes<2, true>() <= 232448, "A-resident 2-CTA scan exceeds the 227 KB smem limit");
static_assert(i8_smem_bytes<2, false>() <= 232448, "2-CTA scan exceeds the 227 KB smem limit");

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(I8_IDESC), "r"(accum)
        : "memory");
}

// M = 256 (both CTAs of the pair), N = 256
constexpr uint32_t I8_IDESC2 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_BLOCK_N >> 3) << 17) |
                               ((uint32_t)(256 >> 4) << 24);
__device__ __forceinline__ void mma_i8_cg2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(I8_IDESC2), "r"(accum)
        : "memory");
}
// arrive on the same barrier in every CTA of `mask` (cluster ranks; default: the pair
// 0/1) when the issued MMAs complete
__device__ __forceinline__ void mma_commit_cg2(uint64_t *bar, uint16_t mask = 3) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on a (possibly remote) barrier of the cluster; default .release.cta semantics as
// CUTLASS's ClusterBarrier::arrive — the TMEM reads it orders are covered by
// tcgen05.fence::before_thread_sync, so no cluster-scope fence (ERRBAR) is needed
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-CTA TMA tile load: data lands in this CTA's smem, bytes are counted on the
// leader CTA's barrier (cluster address)
__device__ __forceinline__ void tma_load_2d_cg2(void *dst, const CUtensorMap *map, uint32_t bar_cluster, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}

// 2-CTA TMA tile load multicast to every CTA of `mask` (same smem offset); each
// destination's bytes are counted on the barrier at `bar_cluster`'s offset in the
// destination's pair leader (the peer bit of the address is clear)
__device__ __forceinline__ void tma_load_2d_cg2_mc(void *dst, const CUtensorMap *map, uint32_t bar_cluster,
                                                   uint16_t mask, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}

// exact for |v| < 2^22
__device__ __forceinline__ float i2f_exact(uint32_t v) {
    return __fsub_rn(__int_as_float((int32_t)v + I8_MAGIC_I), I8_MAGIC_F);
}

// order-preserving float <-> uint32 (0 = below every float = "no bound yet")
__device__ __forceinline__ uint32_t f2ord(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
    if (u == 0) return -INFINITY;
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

struct I8ScanParams {
    int64_t n;
    int nkb;  // K blocks (dp128 / 128)
    int nsplit, tiles_per_split, ntiles, qtiles;
    int k;
    const float *xs;      // [rows] s_r
    const float *xe;      // [rows] dx_r
    const I8TileMeta *xt; // [tiles] per-tile bounds
    const float4 *qmeta;  // [nq_pad] {t_q, A_q, C_q, -}
    const int64_t *row_limit;
    int64_t nq;
    uint32_t *lg;     // [nq] published lower bounds on e_k (f2ord, rounded down)
    int32_t *acount;  // [nq] appended rows
    uint2 *abuf;      // [nq][cap] {row, u bits}
    int cap;
    float thr_floor;  // measurement only: a floor under every bound (-inf normally)
    int noepi;        // measurement only: the epilogue releases each tile untouched
    // pilot mode: scan store tiles idx * tile_stride only, keep the per-thread top-k of
    // l (no appends) and write it to pcand[((q * nsplit + split) * I8_HALVES + half) * TC_KP + i]
    int tile_stride;
    uint64_t *pcand;
    // exact rows / queries for the in-kernel refiner
    const float *x32;
    const float *qp;
    int dp8, d;
    int refine;  // hand rows at the bound to the exact refiner warps
    // L2 lockstep: the SM pairs scanning one split read the same store tiles; a pair
    // more than `window` tiles ahead of the slowest started pair of its split waits,
    // so each tile is still in L2 when the others read it (0 = off)
    int32_t *prog;  // [nsplit][qgroups]: tiles loaded + 1 (0 = not started, INT_MAX = done)
    int window;
    const int32_t *nq_dev;  // device query count (nullable): queries >= *nq_dev are skipped
    // per query, the k largest rounded-down EXACT scores found by ANY CTA's refiner (f2ord
    // keys, 0 = empty; nullable): their minimum bounds e_k from below like one CTA's refiner
    // list, but over the union of every split (see gunion_insert)
    uint32_t *gun;
    int fast2;  // two-level fast path (PR_I8_FAST=1 single level, A/B knob)
    int gskip;  // level (2) skips groups no lane passed (1) for (PR_I8_GSKIP=0: every group; A/B knob)
    int refine_fast;   // refiner publishes fp32 lower bounds (PR_I8_REFINEF=0: exact fp64 einsum scores)
    float refine_err;  // the factor g of dot_f32_lower's error bound (m 2^-24 / (1 - m 2^-24), m = d + 3)
    // measurement only (PR_I8_VERBOSE): [0] warp-chunks that took the cooperative path,
    // [1] warp-chunks, [2] flagged (query, 8-row group) pairs
    uint32_t *dbg;
};

// the live query count of a search: the device count of a compacted list, else nq
__device__ __forceinline__ int64_t live_nq(const int32_t *nq_dev, int64_t nq) {
    return nq_dev ? min(nq, (int64_t)max(0, __ldg(nq_dev))) : nq;
}

// loose per-tile test in the scaled domain: a row can pass u = t s acc + A dx + C >= thr
// only if s * acc >= (thr - C - A dxmax) / t.  1e-6 (score units) absorbs every fp32
// rounding of either side.
// inv = {rd(1/t), ru(1/t)}: lhs / t is bounded below by rd(lhs * rd(1/t)) for lhs >= 0
// and by rd(lhs * ru(1/t)) for lhs < 0 (t > 0) — one FMUL, no division subroutine
__device__ __forceinline__ float2 inv_bounds(float t) {
    return t > 0.f ? make_float2(__frcp_rd(t), __frcp_ru(t)) : make_float2(0.f, 0.f);
}
__device__ __forceinline__ float div_down(float lhs, float2 inv) {
    return __fmul_rd(lhs, lhs >= 0.f ? inv.x : inv.y);
}
__device__ __forceinline__ float loose_threshold(float thr, float2 inv, float A, float C, float dxmax) {
    if (thr == -INFINITY || inv.x <= 0.f) return -INFINITY;
    const float lhs = __fsub_rn(__fsub_rn(thr, __fmaf_ru(A, dxmax, C)), 1e-6f);
    return div_down(lhs, inv);
}

// pilot: l = ap - A dx - C > thr needs ap > thr + C
__device__ __forceinline__ float loose_pilot(float thr, float2 inv, float C) {
    if (thr == -INFINITY || inv.x <= 0.f) return -INFINITY;
    return div_down(__fsub_rn(__fadd_rn(thr, C), 1e-6f), inv);
}

// relaxed gpu-scope load: the value is only consumed a tile later, so its
// latency overlaps a whole tile of epilogue work
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// fp32 dot of two [d] rows with four independent chains, lowered by a rigorous bound on the
// fp32 error: for m = d + 3 fp32 roundings in any order, |dot_fp32 - exact| <= g * S with
// g = m 2^-24 / (1 - m 2^-24) and S = sum |x_i q_i|, which is accumulated alongside (in fp32,
// so it is itself within a factor (1 + g) of the true S).  A lower bound on the exact dot for
// any vectors (unnormalised rows included), ~6x fewer cycles than the fp64 einsum chain.
__device__ __forceinline__ float dot_f32_lower(const float *__restrict__ x, const float *__restrict__ q, int d,
                                               float g) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, s0 = 0.f, s1 = 0.f;
    int j = 0;
#pragma unroll 4
    for (; j + 4 <= d; j += 4) {
        const float4 xa = __ldg(reinterpret_cast<const float4 *>(x + j));
        const float4 qa = __ldg(reinterpret_cast<const float4 *>(q + j));
        a0 = __fmaf_rn(xa.x, qa.x, a0);
        a1 = __fmaf_rn(xa.y, qa.y, a1);
        a2 = __fmaf_rn(xa.z, qa.z, a2);
        a3 = __fmaf_rn(xa.w, qa.w, a3);
        s0 = __fmaf_rn(fabsf(xa.x), fabsf(qa.x), s0);
        s1 = __fmaf_rn(fabsf(xa.y), fabsf(qa.y), s1);
        s0 = __fmaf_rn(fabsf(xa.z), fabsf(qa.z), s0);
        s1 = __fmaf_rn(fabsf(xa.w), fabsf(qa.w), s1);
    }
    for (; j < d; ++j) {
        a0 = __fmaf_rn(x[j], q[j], a0);
        s0 = __fmaf_rn(fabsf(x[j]), fabsf(q[j]), s0);
    }
    const float dot = __fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3));
    const float S = __fmul_ru(__fadd_ru(s0, s1), 1.0f + 2.0f * g);  // >= the true S
    return __fsub_rd(dot, __fadd_ru(__fmul_ru(g, S), 1e-30f));
}

// Insert a lower bound (f2ord key) into a query's k-slot union list and publish the list's
// minimum once all k slots are filled.  Every (query, row) pair reaches exactly one refiner
// once, so the slots always hold k DISTINCT rows' lower bounds: their minimum is a valid
// lower bound on the true k-th score, and it is the union's k-th largest, not one thread's.
// Slots only grow (a CAS replaces the current minimum by a larger key), so a minimum read
// slot by slot is still a minimum over k distinct rows at the end of the read.
__device__ __forceinline__ void gunion_insert(uint32_t *slots, int k, uint32_t key, uint32_t *lg) {
    for (;;) {
        uint32_t mn = 0xFFFFFFFFu;
        int mi = 0;
        for (int i = 0; i < k; ++i) {
            const uint32_t v = ld_relaxed(slots + i);
            if (v < mn) {
                mn = v;
                mi = i;
            }
        }
        if (key <= mn) return;
        if (atomicCAS(slots + mi, mn, key) == mn) {
            uint32_t m2 = 0xFFFFFFFFu;
            for (int i = 0; i < k; ++i) m2 = min(m2, ld_relaxed(slots + i));
            if (m2 != 0u) atomicMax(lg, m2);
            return;
        }
    }
}

// index of the n-th (0-based) set bit of m
__device__ __forceinline__ int nth_set_bit(uint32_t m, int n) {
    for (int i = 0; i < n; ++i) m &= m - 1;
    return __ffs(m) - 1;
}

// MC = CTA pairs per cluster (ARES only).  The MC pairs of a cluster scan MC different
// 256-query groups over the SAME store tiles in lockstep: each store half-tile is
// fetched once per cluster — every CTA loads 1/MC of its half and multicasts it to the
// MC CTAs holding the same half — so L2->SM operand bytes drop by MC.  A stage slot is
// refilled only after every pair's MMAs released it (MC arrivals on each empty barrier).
template <bool PILOT, int CG, bool ARES, int MC = 1>
__global__ void __launch_bounds__(I8_THREADS, 1)
    tc8_scan_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tx, I8ScanParams p) {
    static_assert(!ARES || CG == 2, "A-resident operands are a 2-CTA variant");
    static_assert(MC == 1 || (ARES && !PILOT), "multicast store tiles: A-resident main scan only");
    constexpr int STAGES = I8Cfg<CG, ARES>::STAGES;
    constexpr int B_BYTES = I8Cfg<CG, ARES>::B_BYTES;
    constexpr int A_STAGE = I8Cfg<CG, ARES>::A_STAGE_BYTES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for SWIZZLE_128B, as an offset from the __shared__ array so
    // every derived pointer stays in the shared window (LDS/STS, not generic LD/ST)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *sAres = smem;                                      // [nkb][16 KB] (ARES) resident A
    uint8_t *sA = sAres + I8Cfg<CG, ARES>::A_RES_BYTES;         // [STAGES][16 KB] streamed A (!ARES)
    uint8_t *sB = sA + STAGES * A_STAGE;
    uint8_t *smeta = sB + STAGES * B_BYTES;  // [2][I8_META_BYTES]
    int32_t *spill = reinterpret_cast<int32_t *>(smeta + 2 * I8_META_BYTES);  // [16][I8_EPI]
    uint64_t *full = reinterpret_cast<uint64_t *>(spill + 16 * I8_EPI);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint64_t *mfull = tempty + 2;
    uint64_t *mempty = mfull + 2;
    uint64_t *afull = mempty + 2;   // ARES: the item's A tile landed (leader's copy counts both CTAs)
    uint64_t *aempty = afull + 1;   // ARES: the item's MMAs are done with A
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(aempty + 1);
    uint64_t *rq = reinterpret_cast<uint64_t *>(smem + (size_t)I8Cfg<CG, ARES>::A_RES_BYTES +
                                                (size_t)STAGES * (A_STAGE + B_BYTES) + 2 * I8_META_BYTES +
                                                16 * I8_EPI * 4 + 256);  // [I8_RQ] refiner jobs {q+1, row}
    float *rel = reinterpret_cast<float *>(rq + I8_RQ);  // [128][TC_KP] exact lists, rounded down
    int32_t *rown = reinterpret_cast<int32_t *>(rel + TC_BLOCK_M * TC_KP);  // [128] list owner (global q)
    int32_t *rcnt = rown + TC_BLOCK_M;                                    // [128] entries
    uint32_t *rq_tail = reinterpret_cast<uint32_t *>(rcnt + TC_BLOCK_M);
    uint32_t *epi_done = rq_tail + 1;
    uint16_t *wqmeta = reinterpret_cast<uint16_t *>(reinterpret_cast<uint8_t *>(rq) + I8_REFINER_BYTES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (!PILOT) {
        for (int i = threadIdx.x; i < I8_RQ; i += blockDim.x) rq[i] = 0ull;
        for (int i = threadIdx.x; i < TC_BLOCK_M; i += blockDim.x) {
            rown[i] = -1;
            rcnt[i] = 0;
        }
        if (threadIdx.x == 0) {
            *rq_tail = 0;
            *epi_done = 0;
        }
    }
    // CG == 2: the CTA pair shares items; rank r (role in the pair) scans query tile 2*qp + r.
    // MC > 1: pair `pair` of the cluster takes query group MC*g + pair of the cluster's item
    const uint32_t crank = CG == 2 ? cluster_rank() : 0u;
    const uint32_t rank = crank & 1u, pair = crank >> 1, leader = crank & ~1u;
    // with a device query count only the query groups that hold live queries get items
    // (the grid is shaped for the host's estimate; CTAs past the live items exit)
    const int64_t nq_live = live_nq(p.nq_dev, p.nq);
    const int qgroups = p.nq_dev ? (int)ceil_div<int64_t>(nq_live, (int64_t)CG * TC_BLOCK_M) : p.qtiles / CG;
    const int qgc = (qgroups + MC - 1) / MC;  // cluster items per split
    const int nitems = qgc * p.nsplit;
    const int item0 = blockIdx.x / (CG * MC), istride = gridDim.x / (CG * MC);
    auto item_of = [&](int item, int &qtile, int &split, int &t0, int &nloc) {
        qtile = ((item % qgc) * MC + (int)pair) * CG + (int)rank;  // past the last group: all queries invalid
        split = item / qgc;
        t0 = split * p.tiles_per_split;
        nloc = max(0, min(p.ntiles, t0 + p.tiles_per_split) - t0);
    };

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tq);
        tma_prefetch_desc(&tx);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], MC);  // one commit per pair of the cluster
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], CG * I8_EPI / 32);  // every epilogue warp of the pair (leader's copy)
            mbar_init(&mfull[a], 1);
            mbar_init(&mempty[a], I8_EPI / 32);
        }
        mbar_init(afull, 1);
        mbar_init(aempty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        if (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(I8_TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(I8_TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();  // peer barriers initialised before any remote arrive / TMA
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer: row meta per tile + operand K-slices ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int tix = 0;
            uint32_t apar = 0;
            for (int item = item0; item < nitems; item += istride) {
                int qtile, split, t0, nloc;
                item_of(item, qtile, split, t0, nloc);
                if (ARES) {
                    // the item's query tile, once: wait until the previous item's MMAs released it
                    mbar_wait(aempty, apar ^ 1);
                    if (rank == 0) mbar_expect_tx(afull, CG * p.nkb * I8_A_BYTES);
                    const uint32_t fa = mapa_u32(smem_u32(afull), leader);
                    for (int kb = 0; kb < p.nkb; ++kb)
                        tma_load_2d_cg2(sAres + kb * I8_A_BYTES, &tq, fa, kb * I8_BLOCK_K, qtile * TC_BLOCK_M);
                    apar ^= 1;
                }
                int32_t *myprog = nullptr, *splitprog = nullptr;
                if (!PILOT && MC == 1 && p.window > 0 && rank == 0) {
                    splitprog = p.prog + (int64_t)split * qgroups;
                    myprog = splitprog + item % qgroups;
                }
                for (int i = 0; i < nloc; ++i, ++tix) {
                    if (myprog && (i & 7) == 0) {
                        asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(myprog), "r"(i + 1) : "memory");
                        for (;;) {  // wait while more than `window` tiles ahead of the slowest started pair
                            int lo = INT_MAX;
                            for (int g = 0; g < qgroups; ++g) {
                                int v;
                                asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(splitprog + g) : "memory");
                                if (v > 0) lo = min(lo, v);
                            }
                            if (lo == INT_MAX || i + 1 - lo <= p.window) break;
                            __nanosleep(1000);
                        }
                    }
                    const int t = (t0 + i) * p.tile_stride;
                    const int acc = tix & 1;
                    const uint32_t aphase = (tix >> 1) & 1;
                    uint8_t *m = smeta + acc * I8_META_BYTES;
                    mbar_wait(&mempty[acc], aphase ^ 1);
                    mbar_expect_tx(&mfull[acc], I8_META_BYTES);
                    bulk_load_1d(m, p.xs + (int64_t)t * TC_BLOCK_N, TC_BLOCK_N * 4, &mfull[acc]);
                    bulk_load_1d(m + TC_BLOCK_N * 4, p.xe + (int64_t)t * TC_BLOCK_N, TC_BLOCK_N * 4, &mfull[acc]);
                    bulk_load_1d(m + TC_BLOCK_N * 8, p.xt + t, sizeof(I8TileMeta), &mfull[acc]);
                    for (int kb = 0; kb < p.nkb; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        if (p.noepi == 2) {  // measurement only: no operand traffic (MMAs read stale smem)
                            if (rank == 0) mbar_arrive(&full[stage]);
                            if (++stage == STAGES) { stage = 0; phase ^= 1; }
                            continue;
                        }
                        if (CG == 2) {
                            // the leader's barrier counts both CTAs' bytes; its producer posts the total
                            if (rank == 0) mbar_expect_tx(&full[stage], CG * (A_STAGE + B_BYTES));
                            const uint32_t fb = mapa_u32(smem_u32(&full[stage]), leader);
                            if (!ARES)
                                tma_load_2d_cg2(sA + stage * A_STAGE, &tq, fb, kb * I8_BLOCK_K, qtile * TC_BLOCK_M);
                            if (MC == 1) {
                                tma_load_2d_cg2(sB + stage * B_BYTES, &tx, fb, kb * I8_BLOCK_K,
                                                t * TC_BLOCK_N + (int)rank * I8Cfg<CG, ARES>::B_ROWS);
                            } else {
                                // slice `pair` of this CTA's half, to the same half in every pair
                                constexpr int SR = I8Cfg<CG, ARES>::B_ROWS / MC;
                                const uint16_t mask = (uint16_t)((0x5555u & ((1u << (2 * MC)) - 1u)) << rank);
                                tma_load_2d_cg2_mc(sB + stage * B_BYTES + pair * SR * I8_BLOCK_K, &tx, fb, mask,
                                                   kb * I8_BLOCK_K,
                                                   t * TC_BLOCK_N + (int)rank * I8Cfg<CG, ARES>::B_ROWS + (int)pair * SR);
                            }
                        } else {
                            mbar_expect_tx(&full[stage], I8_A_BYTES + B_BYTES);
                            tma_load_2d(sA + stage * A_STAGE, &tq, &full[stage], kb * I8_BLOCK_K, qtile * TC_BLOCK_M);
                            tma_load_2d(sB + stage * B_BYTES, &tx, &full[stage], kb * I8_BLOCK_K, t * TC_BLOCK_N);
                        }
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
                if (myprog) asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(myprog), "r"(INT_MAX) : "memory");
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (single thread; the pair's leader for CG == 2) ----------------
        if (lane == 0 && rank == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int tix = 0;
            uint32_t apar = 0;
            for (int item = item0; item < nitems; item += istride) {
                int qtile, split, t0, nloc;
                item_of(item, qtile, split, t0, nloc);
                if (ARES) {
                    mbar_wait(afull, apar);
                    tc_fence_after();
                }
                for (int i = 0; i < nloc; ++i, ++tix) {
                    const int acc = tix & 1;
                    const uint32_t aphase = (tix >> 1) & 1;
                    mbar_wait(&tempty[acc], aphase ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem + acc * TC_BLOCK_N;
                    for (int kb = 0; kb < p.nkb; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint64_t ad =
                            sw128_desc(smem_u32(ARES ? sAres + kb * I8_A_BYTES : sA + stage * A_STAGE));
                        const uint64_t bd = sw128_desc(smem_u32(sB + stage * B_BYTES));
#pragma unroll
                        for (int k = 0; k < I8_BLOCK_K / 32; ++k) {  // K = 32 int8 = 32 B per MMA inside the atom
                            if (CG == 2)
                                mma_i8_cg2(d_tmem, ad + 2 * k, bd + 2 * k, (kb | k) != 0);
                            else
                                mma_i8(d_tmem, ad + 2 * k, bd + 2 * k, (kb | k) != 0);
                        }
                        if (CG == 2)  // the slot is free once every pair of the cluster released it
                            mma_commit_cg2(&empty[stage], (uint16_t)((1u << (2 * MC)) - 1u));
                        else
                            mma_commit(&empty[stage]);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    if (CG == 2)
                        mma_commit_cg2(&tfull[acc], (uint16_t)(3u << leader));
                    else
                        mma_commit(&tfull[acc]);
                }
                if (ARES) {  // both producers may overwrite A once these MMAs complete
                    mma_commit_cg2(aempty, (uint16_t)(3u << leader));
                    apar ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> bounds -> append + running top-k of l ----------------
        const int ew = (warp - 4) & 3;                // TMEM lane group
        const int half = (warp - 4) >> 2;             // column slice of the tile
        const int et = ew * 32 + lane;                // TMEM lane == query within the tile
        int32_t *wspill = spill + (warp - 4) * 32;  // this warp's columns of the [16][I8_EPI] spill: the queue
        uint16_t *wq = wqmeta + (warp - 4) * I8_QCAP;  // queued records {owner lane, chunk, group}
        int tix = 0;
        // the MMA issuer waits on the leader's tempty: every epilogue warp of the pair arrives there
        const uint32_t tempty_leader0 = mapa_u32(smem_u32(&tempty[0]), leader);
        for (int item = item0; item < nitems; item += istride) {
            int qtile, split, t0, nloc;
            item_of(item, qtile, split, t0, nloc);
            const int64_t q = (int64_t)qtile * TC_BLOCK_M + et;
            const bool valid = q < nq_live;
            float tq_ = 0.f, A = 0.f, C = 0.f;
            int64_t lim = 0;
            if (valid) {
                const float4 qm = p.qmeta[q];
                tq_ = qm.x;
                A = qm.y;
                C = qm.z;
                lim = p.row_limit ? min(p.n, p.row_limit[q]) : p.n;
            }
            uint32_t *lgq = p.lg + (valid ? q : 0);
            uint32_t lg_next = valid ? ld_relaxed(lgq) : 0u;
            const float2 inv = inv_bounds(tq_);
            // running top-k of l: the first TC_KP - k slots hold +inf sentinels that no
            // insert displaces, so ts[TC_KP - 1] is always the k-th largest l seen
            float ts[TC_KP];
            uint32_t tr[TC_KP];
#pragma unroll
            for (int i = 0; i < TC_KP; ++i) {
                ts[i] = (i < TC_KP - p.k) ? INFINITY : -INFINITY;
                tr[i] = 0xFFFFFFFFu;
            }
            float Lpub = -INFINITY;
            uint32_t n_coop = 0, n_chunks = 0, n_flag = 0, n_fine = 0;
            for (int i = 0; i < nloc; ++i, ++tix) {
                const int acc = tix & 1;
                const uint32_t aphase = (tix >> 1) & 1;
                mbar_wait(&mfull[acc], aphase);
                mbar_wait(&tfull[acc], aphase);
                tc_fence_after();
                if (p.noepi) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (CG == 2)
                            mbar_arrive_cluster(tempty_leader0 + acc * 8);
                        else
                            mbar_arrive(&tempty[acc]);
                        mbar_arrive(&mempty[acc]);
                    }
                    continue;
                }
                const float *ss = reinterpret_cast<const float *>(smeta + acc * I8_META_BYTES);
                const float *se = ss + TC_BLOCK_N;
                const I8TileMeta *tm = reinterpret_cast<const I8TileMeta *>(se + TC_BLOCK_N);
                const float dxmax = tm->dxmax;
                // main: append rows with u >= thr; pilot: insert rows with l > thr
                float thr = fmaxf(fmaxf(ts[TC_KP - 1], p.thr_floor), ord2f(lg_next));
                if (valid) lg_next = ld_relaxed(lgq);  // for the next tile
                float thr2 = PILOT ? loose_pilot(thr, inv, C) : loose_threshold(thr, inv, A, C, dxmax);
                const int64_t rbase = (int64_t)(t0 + i) * p.tile_stride * TC_BLOCK_N;
                const uint32_t taddr = tmem + ((uint32_t)(ew * 32) << 16) + acc * TC_BLOCK_N;
                // Flagged (query, 8-row group) pairs are QUEUED (their 8 accumulators in this
                // warp's spill rows, {owner lane, chunk, group} in wq) and evaluated after the
                // accumulator is released, so the rare expensive groups do not hold TMEM while
                // the next tile's MMAs wait for it.  The tile's row meta (ss, se) stays valid
                // until mempty is released after the queue drains.
                int qn = 0;
                // evaluate the queue cooperatively: 4 records (32 rows) per pass, one row per lane,
                // the owner lane's (query's) constants by shuffle
                auto drain = [&]() {
                    __syncwarp();
#pragma unroll 1
                    for (int base = 0; base < qn; base += 4) {
                        const int r = base + (lane >> 3);
                        bool act = r < qn;
                        const int mt = act ? (int)wq[r] : 0;
                        const int owner = mt & 31;
                        const int j = ((mt >> 5) & 7) * 32 + ((mt >> 8) & 3) * 8 + (lane & 7);  // row in the tile
                        const float o_t = __shfl_sync(0xffffffffu, tq_, owner);
                        const float o_A = __shfl_sync(0xffffffffu, A, owner);
                        const float o_C = __shfl_sync(0xffffffffu, C, owner);
                        const float o_thr = __shfl_sync(0xffffffffu, thr, owner);
                        const float o_kth = __shfl_sync(0xffffffffu, ts[TC_KP - 1], owner);
                        const int64_t o_lim = __shfl_sync(0xffffffffu, lim, owner);
                        const uint32_t row = (uint32_t)(rbase + j);
                        act = act && (int64_t)row < o_lim;
                        float l = -INFINITY;
                        if (act) {
                            const int e = r * 8 + (lane & 7);
                            const float dx = se[j];
                            const float ap =
                                __fmul_rn(__fmul_rn(i2f_exact((uint32_t)wspill[(e >> 5) * I8_EPI + (e & 31)]), ss[j]), o_t);
                            l = __fsub_rn(ap, __fmaf_rn(o_A, dx, o_C));
                            if (!PILOT) {
                                const float u = __fadd_rn(__fmaf_rn(o_A, dx, ap), o_C);
                                if (u >= o_thr) {
                                    const int64_t oq = (int64_t)qtile * TC_BLOCK_M + ew * 32 + owner;
                                    const int o = atomicAdd(&p.acount[oq], 1);
                                    if (o < p.cap) p.abuf[oq * (int64_t)p.cap + o] = make_uint2(row, __float_as_uint(u));
                                    // approximate score at the bound: hand the row to the refiner
                                    // (a full table just drops the job: the bound is a heuristic)
                                    if (p.refine && ap >= o_thr) {
                                        const uint32_t slot = atomicAdd(rq_tail, 1u) & (I8_RQ - 1);
                                        atomicCAS(reinterpret_cast<unsigned long long *>(&rq[slot]), 0ull,
                                                  ((unsigned long long)(oq + 1) << 32) | row);
                                    }
                                }
                            }
                        }
                        // list inserts happen in the owner lane
                        uint32_t wb = __ballot_sync(0xffffffffu, act && l > o_kth);
                        while (wb) {
                            const int src = __ffs(wb) - 1;
                            wb &= wb - 1;
                            const float lv = __shfl_sync(0xffffffffu, l, src);
                            const uint32_t rv = __shfl_sync(0xffffffffu, row, src);
                            const int ow = __shfl_sync(0xffffffffu, owner, src);
                            if (lane == ow && lv > ts[TC_KP - 1]) {
                                topk_insert(ts, tr, lv, rv);
                                if (ts[TC_KP - 1] > thr) {
                                    thr = ts[TC_KP - 1];
                                    thr2 = PILOT ? loose_pilot(thr, inv, C) : loose_threshold(thr, inv, A, C, dxmax);
                                }
                            }
                        }
                    }
                    qn = 0;
                    __syncwarp();
                };
                uint32_t va[32], vb[32];
                TMEM_LD32(taddr + half * I8_CPW * 32, va);
                tmem_wait_ld();
#pragma unroll 1
                for (int cp = 0; cp < I8_CPW / 2; ++cp) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c = half * I8_CPW + 2 * cp + h;
                        uint32_t(&v)[32] = h ? vb : va;
                        // the next chunk streams in while this one is scored
                        if (h == 0) {
                            TMEM_LD32(taddr + (c + 1) * 32, vb);
                        } else if (cp + 1 < I8_CPW / 2) {
                            TMEM_LD32(taddr + (c + 1) * 32, va);
                        }
                        // fast path, two levels.  (1) per 8-row group, the integer max of the
                        // accumulators times the group's max scale s_g (tile meta): for acc >= 0,
                        // fl(s_r acc_r) <= fl(s_g acc_r) <= fl(s_g max acc) (monotone rounding), and a
                        // negative acc cannot reach a positive thr2, so a group no row of which passes
                        // (2) is never dropped — ~1.4 ops per score instead of ~4.  (2) only where some
                        // lane's group passed (1): per row s_r * acc (exact int -> fp32), the test that
                        // flags groups for the cooperative path (the same flags as before).
                        const int64_t rb = rbase + c * 32;
                        uint32_t gmask = 0;
                        uint32_t cmask = 0xFu;
                        if (p.fast2) {
                            const float4 gs = reinterpret_cast<const float4 *>(tm->gmax)[c];
                            const float sg[4] = {gs.x, gs.y, gs.z, gs.w};
                            cmask = 0;
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                int m0 = max((int32_t)v[8 * g + 0], (int32_t)v[8 * g + 1]);
                                int m1 = max((int32_t)v[8 * g + 2], (int32_t)v[8 * g + 3]);
                                m0 = max(m0, (int32_t)v[8 * g + 4]);
                                m1 = max(m1, (int32_t)v[8 * g + 5]);
                                m0 = max(m0, (int32_t)v[8 * g + 6]);
                                m1 = max(m1, (int32_t)v[8 * g + 7]);
                                const float cm = __fmul_rn(i2f_exact((uint32_t)max(m0, m1)), sg[g]);
                                cmask |= (thr2 <= 0.f || cm >= thr2 ? 1u : 0u) << g;
                            }
                        }
                        if (__any_sync(0xffffffffu, cmask != 0)) {
                            if (p.dbg) ++n_fine;
                            const float4 *s4 = reinterpret_cast<const float4 *>(ss + c * 32);
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                // a group no lane passed (1) for: skip it warp-uniformly
                                if (p.gskip && !__any_sync(0xffffffffu, (cmask >> g) & 1u)) continue;
                                const float4 sa = s4[2 * g], sb = s4[2 * g + 1];
                                float m0 = fmaxf(__fmul_rn(i2f_exact(v[8 * g + 0]), sa.x),
                                                 __fmul_rn(i2f_exact(v[8 * g + 1]), sa.y));
                                float m1 = fmaxf(__fmul_rn(i2f_exact(v[8 * g + 2]), sa.z),
                                                 __fmul_rn(i2f_exact(v[8 * g + 3]), sa.w));
                                m0 = fmaxf(m0, __fmul_rn(i2f_exact(v[8 * g + 4]), sb.x));
                                m1 = fmaxf(m1, __fmul_rn(i2f_exact(v[8 * g + 5]), sb.y));
                                m0 = fmaxf(m0, __fmul_rn(i2f_exact(v[8 * g + 6]), sb.z));
                                m1 = fmaxf(m1, __fmul_rn(i2f_exact(v[8 * g + 7]), sb.w));
                                gmask |= (((cmask >> g) & 1u) && fmaxf(m0, m1) >= thr2 ? 1u : 0u) << g;
                            }
                        }
                        if (rb >= lim) gmask = 0;
                        if (p.dbg) {
                            ++n_chunks;
                            n_flag += __popc(gmask);
                        }
                        if (__any_sync(0xffffffffu, gmask != 0)) {
                            if (p.dbg) ++n_coop;
                            uint32_t bg[4];
#pragma unroll
                            for (int g = 0; g < 4; ++g) bg[g] = __ballot_sync(0xffffffffu, (gmask >> g) & 1u);
                            const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                // groups {0,1} then {2,3}: at most 64 records each; a full queue is
                                // evaluated first, while TMEM is still held (rare: cold bounds)
                                if ((g & 1) == 0 && qn + __popc(bg[g]) + __popc(bg[g + 1]) > I8_QCAP) drain();
                                if (!bg[g]) continue;
                                if ((gmask >> g) & 1u) {
                                    const int r = qn + __popc(bg[g] & lt);
#pragma unroll
                                    for (int x = 0; x < 8; ++x) {
                                        const int e = r * 8 + x;
                                        wspill[(e >> 5) * I8_EPI + (e & 31)] = (int32_t)v[8 * g + x];
                                    }
                                    wq[r] = (uint16_t)(lane | (c << 5) | (g << 8));
                                }
                                qn += __popc(bg[g]);
                            }
                        }
                        if (h == 0 || cp + 1 < I8_CPW / 2) tmem_wait_ld();
                    }
                }
                // release the accumulator, then evaluate the queued groups
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 2)
                        mbar_arrive_cluster(tempty_leader0 + acc * 8);
                    else
                        mbar_arrive(&tempty[acc]);
                }
                if (qn) drain();
                if (lane == 0) mbar_arrive(&mempty[acc]);
                if (valid && ts[TC_KP - 1] > Lpub) {
                    Lpub = ts[TC_KP - 1];
                    atomicMax(lgq, f2ord(Lpub));
                }
            }
            if (p.dbg) {
                n_flag = __reduce_add_sync(0xffffffffu, n_flag);
                if (lane == 0) {
                    atomicAdd(&p.dbg[0], n_coop);
                    atomicAdd(&p.dbg[1], n_chunks);
                    atomicAdd(&p.dbg[2], n_flag);
                    atomicAdd(&p.dbg[3], n_fine);
                }
            }
            if (PILOT && valid) {
                uint64_t *out = p.pcand + ((q * p.nsplit + split) * I8_HALVES + half) * TC_KP;
#pragma unroll
                for (int s = 0; s < TC_KP; ++s)
                    out[s] = (tr[s] == 0xFFFFFFFFu) ? 0ull : cand_key(ts[s], tr[s]);
            }
        }
        if (!PILOT) {
            __threadfence_block();
            __syncwarp();
            if (lane == 0) atomicAdd(epi_done, 1u);
        }
    } else if (!PILOT && (warp == 2 || warp == 3)) {
        // ---------------- exact refiner: score handed-over rows in fp64 einsum order ----------------
        // warp 2 owns even local queries, warp 3 odd ones (each list has a single writer)
        const uint32_t par = (uint32_t)(warp - 2);
        uint32_t seen = 0;  // pushes observed so far: an idle poll is one shared load
        for (;;) {
            const uint32_t tail = *reinterpret_cast<volatile uint32_t *>(rq_tail);
            const bool done = *reinterpret_cast<volatile uint32_t *>(epi_done) == I8_EPI / 32;
            if (tail == seen && !done) {
                __nanosleep(2000);
                continue;
            }
            uint64_t job = 0;
            for (int i = lane; i < I8_RQ && !job; i += 32) {
                const uint64_t v = *reinterpret_cast<volatile uint64_t *>(&rq[i]);
                if (v && ((uint32_t)((v >> 32) - 1) & 1u) == par)
                    job = atomicExch(reinterpret_cast<unsigned long long *>(&rq[i]), 0ull);
            }
            const uint32_t has = __ballot_sync(0xffffffffu, job != 0);
            if (!has) {
                seen = tail;  // every job pushed before `tail` was read has been taken (by either warp)
                if (done) {
                    // the epilogue finished (its pushes precede the count): drain once more, then stop
                    bool any = false;
                    for (int i = lane; i < I8_RQ; i += 32) any |= *reinterpret_cast<volatile uint64_t *>(&rq[i]) != 0;
                    if (!__any_sync(0xffffffffu, any)) break;
                }
                continue;
            }
            const int64_t qg = job ? (int64_t)(job >> 32) - 1 : 0;
            const uint32_t row = (uint32_t)job;
            double ex = 0.0;
            if (job) {
                if (p.refine_fast) {
                    // a rigorous LOWER bound is all the refiner publishes, so the fp64 einsum
                    // chain (24-cycle dependent DFMAs) is not needed: four independent fp32 FMA
                    // chains, then minus the accumulation error bound — for any order of n fp32
                    // FMAs, |sum - exact| <= n 2^-24 sum|x_i q_i| / (1 - n 2^-24), and
                    // sum|x_i q_i| <= ||x|| ||q|| (unit vectors within 1e-4; row norms <= maxnorm)
                    ex = (double)dot_f32_lower(p.x32 + (int64_t)row * p.dp8, p.qp + qg * p.dp8, p.d, p.refine_err);
                } else {
                    ex = einsum_dot_f32(p.x32 + (int64_t)row * p.dp8, p.qp + qg * p.dp8, p.d);
                }
            }
            for (uint32_t m = has; m; m &= m - 1) {
                const int src = __ffs(m) - 1;
                if (lane == src) {
                    const int ql = (int)(qg % TC_BLOCK_M);
                    if (rown[ql] != (int32_t)qg) {  // a new item brought new queries
                        rown[ql] = (int32_t)qg;
                        rcnt[ql] = 0;
                    }
                    // rounded-down exact scores: the k-th entry is still a lower bound on e_k
                    float *L = rel + ql * TC_KP;
                    const float exf = __double2float_rd(ex);
                    int n = rcnt[ql];
                    if (n < p.k || exf > L[p.k - 1]) {
                        int pos = n < p.k ? n++ : p.k - 1;
                        while (pos > 0 && exf > L[pos - 1]) {
                            L[pos] = L[pos - 1];
                            --pos;
                        }
                        L[pos] = exf;
                        rcnt[ql] = n;
                        // k distinct rows score >= L[k-1]: a valid lower bound on e_k
                        if (n == p.k) atomicMax(p.lg + qg, f2ord(L[p.k - 1]));
                    }
                    // ... and the union over every CTA's refiner: each (query, row) is handed to
                    // one refiner once, so the union list holds distinct rows' exact scores
                    if (p.gun) {
                        const uint32_t key = f2ord(exf);
                        if (key > ld_relaxed(p.lg + qg)) gunion_insert(p.gun + qg * TC_KP, p.k, key, p.lg + qg);
                    }
                }
                __syncwarp();
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();  // no CTA leaves while its peer may still signal its barriers
    if (warp == 2) {
        tc_fence_after();
        if (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(I8_TMEM_COLS)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(I8_TMEM_COLS)
                         : "memory");
    }
}

// ---------------------------------------------------------------------------
// per-row / per-query quantisation, one warp per vector.
//   out8[dp128] = rint(v / s) (zero padded), s = max(max|v| / 127, ||v|| / (KMAX - sqrt(d)/2))
//   so |out8| <= 127 and ||out8||_2 <= ||v|| / s + sqrt(d)/2 <= KMAX.
//   err = ||v - s*out8||_2, nrm = ||v||_2, rec = ||s*out8||_2 — fp64 sums of squares
__device__ __forceinline__ void quantize_vec_warp(const float *__restrict__ v, int d, int dp128, int8_t *__restrict__ out8,
                                                  float *s_out, double *err2, double *nrm2, double *rec2) {
    const int lane = threadIdx.x & 31;
    float mx = 0.f;
    double n2 = 0.0;
    for (int j = lane; j < d; j += 32) {
        mx = fmaxf(mx, fabsf(v[j]));
        n2 = fma((double)v[j], (double)v[j], n2);
    }
    for (int o = 16; o; o >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        n2 += __shfl_xor_sync(0xffffffffu, n2, o);
    }
    float s = 0.f;
    if (mx > 0.f) {
        const double nrm = sqrt(n2) * (1.0 + 1e-12);
        s = __double2float_ru(fmax((double)mx / 127.0, nrm / (I8_KMAX - 0.5 * sqrt((double)d))));
    }
    double e2 = 0.0, r2 = 0.0;
    for (int j = lane; j < dp128; j += 32) {
        int qv = 0;
        if (j < d && s > 0.f) {
            const float x = v[j];
            qv = (int)rintf(x / s);
            qv = max(-127, min(127, qv));
            const double rec = (double)s * (double)qv;  // exact: 24-bit x 8-bit product
            const double dx = (double)x - rec;          // exact in fp64 (significands of 24 and 32 bits)
            e2 = fma(dx, dx, e2);
            r2 = fma(rec, rec, r2);
        }
        out8[j] = (int8_t)qv;
    }
    for (int o = 16; o; o >>= 1) {
        e2 += __shfl_xor_sync(0xffffffffu, e2, o);
        r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    }
    *s_out = s;
    *err2 = e2;
    *nrm2 = n2;
    *rec2 = r2;
}

// sqrt of an fp64 sum of d squares, bounded above
__device__ __forceinline__ double norm_up(double sumsq) { return sqrt(sumsq) * (1.0 + 1e-12) + 1e-30; }

__global__ void quantize_rows_kernel(const float *__restrict__ src, int64_t n, int d, const int64_t *__restrict__ rows,
                                     int64_t row0, int dp128, int8_t *__restrict__ x8, float *__restrict__ xs,
                                     float *__restrict__ xe, I8TileMeta *__restrict__ xt, uint32_t *__restrict__ maxnorm) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    if (w >= n) return;
    const int64_t r = rows ? rows[w] : row0 + w;
    float s;
    double e2, n2, r2;
    quantize_vec_warp(src + w * (int64_t)d, d, dp128, x8 + r * (int64_t)dp128, &s, &e2, &n2, &r2);
    if ((threadIdx.x & 31) == 0) {
        const float dx = __double2float_ru(norm_up(e2));
        xs[r] = s;
        xe[r] = dx;
        // positive floats order as uints; both maxima only grow (stay valid bounds)
        atomicMax(reinterpret_cast<uint32_t *>(&xt[r / TC_BLOCK_N].dxmax), __float_as_uint(dx));
        atomicMax(reinterpret_cast<uint32_t *>(&xt[r / TC_BLOCK_N].gmax[(r % TC_BLOCK_N) / 8]), __float_as_uint(s));
        atomicMax(maxnorm, __float_as_uint(__double2float_ru(norm_up(n2))));
    }
}

__global__ void gather_i8_kernel(const int8_t *__restrict__ sx8, const float *__restrict__ sxs,
                                 const float *__restrict__ sxe, const uint32_t *__restrict__ smaxnorm,
                                 const int64_t *__restrict__ src_rows, int64_t n, int dp128, int64_t row0,
                                 int8_t *__restrict__ x8, float *__restrict__ xs, float *__restrict__ xe,
                                 I8TileMeta *__restrict__ xt, uint32_t *__restrict__ maxnorm) {
    // the gathered rows' norms are bounded by the source's maximum
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicMax(maxnorm, *smaxnorm);
    const int64_t total = n * (int64_t)(dp128 / 16);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / (dp128 / 16);
        const int j = (int)(t - i * (dp128 / 16));
        const int64_t s = src_rows[i];
        reinterpret_cast<int4 *>(x8 + (row0 + i) * dp128)[j] = reinterpret_cast<const int4 *>(sx8 + s * dp128)[j];
        if (j == 0) {
            const int64_t r = row0 + i;
            xs[r] = sxs[s];
            xe[r] = sxe[s];
            atomicMax(reinterpret_cast<uint32_t *>(&xt[r / TC_BLOCK_N].dxmax), __float_as_uint(sxe[s]));
            atomicMax(reinterpret_cast<uint32_t *>(&xt[r / TC_BLOCK_N].gmax[(r % TC_BLOCK_N) / 8]),
                      __float_as_uint(sxs[s]));
        }
    }
}

// queries: padded fp32 [nq, dp8] -> int8 [nq_pad, dp128] + {t, A, C}
__global__ void quantize_queries_kernel(const float *__restrict__ qp, int64_t nq, int64_t nq_pad, int dp8, int d,
                                        int dp128, const uint32_t *__restrict__ maxnorm, int8_t *__restrict__ q8,
                                        float4 *__restrict__ qmeta, const int32_t *__restrict__ nq_dev) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (w >= nq_pad) return;
    nq = live_nq(nq_dev, nq);
    if (w >= nq) {
        for (int j = lane; j < dp128; j += 32) q8[w * dp128 + j] = 0;
        if (lane == 0) qmeta[w] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    float t;
    double e2, n2, r2;
    quantize_vec_warp(qp + w * (int64_t)dp8, d, dp128, q8 + w * dp128, &t, &e2, &n2, &r2);
    if (lane == 0) {
        const double nmax = (double)__uint_as_float(*maxnorm);
        const double A = norm_up(r2), B = norm_up(e2);
        // rounding slack: |fl(ap) - t s acc| <= 2 * 2^-24 * A * (nmax + dxmax) and a few
        // fp32 roundings in u / l; 1e-6 * (1 + 2 A nmax) dominates both for any d <= 8192
        const double C = B * nmax + 1e-6 * (1.0 + 2.0 * A * nmax);
        qmeta[w] = make_float4(t, __double2float_ru(A), __double2float_ru(C), 0.f);
    }
}

// ---------------------------------------------------------------------------
// exact rescoring, one WARP per query: seeds = the exact top-k over the scan's
// per-split lists (k distinct rows, so their k-th score L <= e_k); stream the
// appended rows with u >= L (L rising as better rows are scored) through an
// exact running top-k.  A row with u < L has exact <= u < L <= e_k.
constexpr int W8_WARPS = 8;
constexpr int W8_BATCH = 16;  // rows scored per warp batch (2 lanes per row)

// exact einsum-order partial of lane chain `ch` (0: elements 6,4,2,0 of each
// block of 8, 1: 7,5,3,1 — einsum_dot_f32's two fp64 lanes); q in smem
__device__ __forceinline__ double einsum_chain(const float *__restrict__ x, const float *__restrict__ q, int d, int ch) {
    double a = 0.0;
    int j = 0;
#pragma unroll 8
    for (; j + 8 <= d; j += 8) {
        const float4 xa = __ldg(reinterpret_cast<const float4 *>(x + j));
        const float4 xb = __ldg(reinterpret_cast<const float4 *>(x + j + 4));
        const float4 qa = *reinterpret_cast<const float4 *>(q + j);
        const float4 qb = *reinterpret_cast<const float4 *>(q + j + 4);
        a = fma((double)(ch ? xb.w : xb.z), (double)(ch ? qb.w : qb.z), a);
        a = fma((double)(ch ? xb.y : xb.x), (double)(ch ? qb.y : qb.x), a);
        a = fma((double)(ch ? xa.w : xa.z), (double)(ch ? qa.w : qa.z), a);
        a = fma((double)(ch ? xa.y : xa.x), (double)(ch ? qa.y : qa.x), a);
    }
    for (; j < d; j += 2) a = fma((double)x[j + ch], (double)q[j + ch], a);
    return a;
}

// exact scores of rows[0..nb) (nb <= 16) by one warp: lane pair (2i, 2i+1) scores row i
__device__ __forceinline__ void warp_score(const float *__restrict__ x32, int dp8, int d, const int32_t *rows, int nb,
                                           const float *qs, double *out) {
    const int lane = threadIdx.x & 31, r = lane >> 1, ch = lane & 1;
    double a = 0.0;
    if (r < nb) a = einsum_chain(x32 + (int64_t)rows[r] * dp8, qs, d, ch);
    const double other = __shfl_xor_sync(0xffffffffu, a, 1);
    if (ch == 0 && r < nb) out[r] = 0.0 + (a + other);
    __syncwarp();
}

// lane 0: insert (sc, r) into the top list sorted by (score desc, row asc)
__device__ __forceinline__ void top_insert(double *ts, int32_t *tr, int &n, int take, double sc, int32_t r) {
    if (n == take && !ranks_before(sc, r, ts[take - 1], tr[take - 1])) return;
    int pos = (n < take) ? n++ : take - 1;
    while (pos > 0 && ranks_before(sc, r, ts[pos - 1], tr[pos - 1])) {
        ts[pos] = ts[pos - 1];
        tr[pos] = tr[pos - 1];
        --pos;
    }
    ts[pos] = sc;
    tr[pos] = r;
}

struct I8SeedArgs {
    const uint64_t *pcand;  // [nq][nsplit][TC_KP] pilot keys (l, row), 0 = empty
    int nsplit;
    int64_t nq;
    int k;
    const float *x32;
    int dp8, d;
    const float *qp;
    int32_t *seed_rows;  // [nq][TC_KP]
    double *seed_s;      // [nq][TC_KP]
    int32_t *seed_n;     // [nq]
    uint32_t *lg;        // [nq] <- max(lg, rounded-down exact k-th seed score)
    const int32_t *nq_dev;
};

// per query (one warp): the k pilot rows with the largest l, scored exactly
__global__ void __launch_bounds__(W8_WARPS * 32) tc8_seed_kernel(I8SeedArgs a) {
    extern __shared__ __align__(16) float qdyn[];  // [W8_WARPS][dp8 + 8]
    __shared__ int32_t rows_sh[W8_WARPS][TC_KP];
    __shared__ double ex_sh[W8_WARPS][TC_KP];
    __shared__ double ts_sh[W8_WARPS][TC_KP];
    __shared__ int32_t tr_sh[W8_WARPS][TC_KP];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * W8_WARPS + w;
    const int64_t nw = (int64_t)gridDim.x * W8_WARPS;
    const int M = a.nsplit * I8_HALVES * TC_KP;
    float *qs = qdyn + w * (a.dp8 + 8);
    const int64_t nq_live = live_nq(a.nq_dev, a.nq);
    for (int64_t q = wid; q < nq_live; q += nw) {
        const uint64_t *cq = a.pcand + q * (int64_t)M;
        uint64_t last = ~0ull;
        int n = 0;
        for (int j = 0; j < a.k; ++j) {
            uint64_t best = 0;
            for (int e = lane; e < M; e += 32) {
                const uint64_t key = cq[e];
                if (key < last && key > best) best = key;
            }
            for (int o = 16; o; o >>= 1) {
                const uint64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
                best = ob > best ? ob : best;
            }
            if (best == 0) break;
            if (lane == 0) rows_sh[w][n] = (int32_t)key_row(best);
            ++n;
            last = best;
        }
        const float *qv = a.qp + q * (int64_t)a.dp8;
        for (int j = lane; j < a.dp8; j += 32) qs[j] = qv[j];
        __syncwarp();
        warp_score(a.x32, a.dp8, a.d, rows_sh[w], n, qs, ex_sh[w]);
        if (lane == 0) {
            int m = 0;
            for (int j = 0; j < n; ++j) top_insert(ts_sh[w], tr_sh[w], m, a.k, ex_sh[w][j], rows_sh[w][j]);
            for (int j = 0; j < m; ++j) {
                a.seed_rows[q * TC_KP + j] = tr_sh[w][j];
                a.seed_s[q * TC_KP + j] = ts_sh[w][j];
            }
            a.seed_n[q] = m;
            // k distinct rows score >= ts[k-1] exactly: a lower bound on the true k-th score
            if (m == a.k) atomicMax(&a.lg[q], f2ord(__double2float_rd(ts_sh[w][a.k - 1])));
        }
        __syncwarp();
    }
}

struct I8PostArgs {
    unsigned long long *clk;  // measurement only (PR_I8_VERBOSE): per-phase cycles, rounds, passes
    int pf;                   // ring-prefetched chains (PR_I8_POSTPF=0: the plain loop; A/B knob)
    const int32_t *acount;
    const uint2 *abuf;
    int cap;
    int64_t nq;
    int k;
    int64_t take;
    const int64_t *row_limit;
    const float *x32;
    int dp8, d;
    const float *qp;
    const int32_t *seed_rows;  // [nq][TC_KP] exact seeds from the pilot (nullable)
    const double *seed_s;
    const int32_t *seed_n;
    int64_t *rows;
    double *raw, *rep;
    int32_t *count;
    int32_t *counters;  // [0] fallback, [1] rescored rows, [3] appended rows
    int32_t *fallback;
    const int32_t *nq_dev;
    // the scan's published lower bounds on e_k (f2ord; nullable): a valid filter for the
    // appended rows from the start, so the post kernel needs ONE scoring round, not two
    // (PR_I8_POSTLG=0 restores the first round over the largest-u rows; A/B knob)
    const uint32_t *lg;
    // prefetch each refilled row into L2 (PR_I8_POSTL2=1; A/B knob).  Off: at 10M x 1024, B = 4096
    // the prefetches cost more than they hide (score+refill 132k -> 96k cycles per query; the
    // ring chain's own loads keep enough in flight).  A lane pair splitting each block's loads
    // (twice the blocks in flight in the same registers, two shuffles per block) was slower still.
    int l2pf = 0;
};

__global__ void __launch_bounds__(W8_WARPS * 32) tc8_post_kernel(I8PostArgs a) {
    extern __shared__ __align__(16) float qdyn[];  // [W8_WARPS][dp8 + 8]
    __shared__ double top_s[W8_WARPS][TC_KP];
    __shared__ int32_t top_r[W8_WARPS][TC_KP];
    __shared__ int32_t cand[W8_WARPS][64];
    __shared__ double bex[W8_WARPS][W8_BATCH];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * W8_WARPS + w;
    const int64_t nw = (int64_t)gridDim.x * W8_WARPS;
    double *ts = top_s[w];
    int32_t *tr = top_r[w];
    float *qs = qdyn + w * (a.dp8 + 8);
    const int64_t nq_live = live_nq(a.nq_dev, a.nq);
    for (int64_t q = wid; q < nq_live; q += nw) {
        const int take = (int)(a.row_limit ? min(a.take, max((int64_t)0, a.row_limit[q])) : a.take);
        const int cnt = a.acount[q];
        if (lane == 0) atomicAdd(&a.counters[3], cnt);
        if (take > 0 && cnt > a.cap) {
            if (lane == 0) a.fallback[atomicAdd(&a.counters[0], 1)] = (int32_t)q;
            continue;
        }
        const float *qv = a.qp + q * (int64_t)a.dp8;
        int n = 0;  // entries in the top list (lane-uniform)
        int scored = 0;
        if (take > 0) {
            for (int j = lane; j < a.dp8; j += 32) qs[j] = qv[j];
            // seeds: the pilot's exact top-k ...
            if (a.seed_n) {
                n = min(a.seed_n[q], take);
                if (lane < n) {
                    ts[lane] = a.seed_s[q * TC_KP + lane];
                    tr[lane] = a.seed_rows[q * TC_KP + lane];
                }
            }
            __syncwarp();
            const uint2 *e = a.abuf + q * (int64_t)a.cap;
            {
                // ... and the take appended rows with the largest (u, row) keys, scored exactly
                uint64_t lastk = ~0ull;
                int nb = 0;
                for (int j = 0; j < take; ++j) {
                    uint64_t best = 0;
                    for (int i = lane; i < cnt; i += 32) {
                        const uint2 v = e[i];
                        const uint64_t key = cand_key(__uint_as_float(v.y), v.x);
                        if (key < lastk && key > best) best = key;
                    }
                    for (int o = 16; o; o >>= 1) {
                        const uint64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
                        best = ob > best ? ob : best;
                    }
                    if (best == 0) break;
                    lastk = best;
                    const int32_t row = (int32_t)key_row(best);
                    bool dup = false;
                    for (int t = 0; t < n; ++t) dup |= (tr[t] == row);
                    if (!dup) {
                        if (lane == 0) cand[w][nb] = row;
                        ++nb;
                    }
                }
                __syncwarp();
                if (nb > 0) {
                    warp_score(a.x32, a.dp8, a.d, cand[w], nb, qs, bex[w]);
                    if (lane == 0)
                        for (int j = 0; j < nb; ++j) top_insert(ts, tr, n, take, bex[w][j], cand[w][j]);
                    scored += nb;
                    n = __shfl_sync(0xffffffffu, n, 0);
                    __syncwarp();
                }
            }
            float L = (n == take) ? __double2float_rd(ts[take - 1]) : -INFINITY;
            int pend = 0;  // rows waiting in cand[w][0..pend)
            for (int base = 0; base < cnt || pend > 0; base += 32) {
                if (base < cnt) {
                    const int i = base + lane;
                    bool pass = false;
                    int32_t row = -1;
                    if (i < cnt) {
                        const uint2 v = e[i];
                        row = (int32_t)v.x;
                        pass = __uint_as_float(v.y) >= L;
                        for (int j = 0; j < n && pass; ++j) pass = (tr[j] != row);
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, pass);
                    if (pass) cand[w][pend + __popc(m & ((1u << lane) - 1))] = row;
                    pend += __popc(m);
                    __syncwarp();
                }
                const bool last = base + 32 >= cnt;
                while (pend >= W8_BATCH || (last && pend > 0)) {
                    const int nb = min(pend, W8_BATCH);
                    warp_score(a.x32, a.dp8, a.d, cand[w], nb, qs, bex[w]);
                    if (lane == 0) {
                        for (int j = 0; j < nb; ++j) top_insert(ts, tr, n, take, bex[w][j], cand[w][j]);
                    }
                    scored += nb;
                    n = __shfl_sync(0xffffffffu, n, 0);
                    // shift the remaining pending rows down
                    const int32_t mv = (lane + nb < pend) ? cand[w][lane + nb] : 0;
                    const int32_t mv2 = (lane + 32 + nb < pend) ? cand[w][lane + 32 + nb] : 0;
                    __syncwarp();
                    if (lane + nb < pend) cand[w][lane] = mv;
                    if (lane + 32 + nb < pend) cand[w][lane + 32] = mv2;
                    pend -= nb;
                    __syncwarp();
                    if (n == take) L = __double2float_rd(ts[take - 1]);
                }
                if (base >= cnt) break;
            }
            if (lane == 0) atomicAdd(&a.counters[1], scored);
        }
        // outputs: self-snap (element-wise equal stored row, index.py:180-181) + clamp (:185)
        for (int j = 0; j < a.k; ++j) {
            const int64_t o = q * a.k + j;
            if (j >= n) {
                if (lane == 0) {
                    a.rows[o] = -1;
                    if (a.raw) a.raw[o] = 0.0;
                    if (a.rep) a.rep[o] = 0.0;
                }
                continue;
            }
            const double bs = ts[j];
            const int64_t br = tr[j];
            double rep = bs;
            if (bs > 1.0 - 1e-6) {
                const float *x = a.x32 + br * (int64_t)a.dp8;
                int bad = 0;
                for (int t = lane; t < a.d; t += 32) bad |= !(x[t] == qv[t]);
                if (!__any_sync(0xffffffffu, bad)) rep = 1.0;
            }
            if (lane == 0) {
                a.rows[o] = br;
                if (a.raw) a.raw[o] = bs;
                if (a.rep) a.rep[o] = fmax(-1.0, fmin(1.0, rep));
            }
        }
        if (lane == 0) a.count[q] = n;
        __syncwarp();
    }
}

// The same post-processing with ONE CTA PER QUERY (the default): the warp-per-query kernel
// above streams each candidate row through one lane pair with ~16 rows in flight per
// query, so a query with many appended rows serialised ~16 DRAM round trips per batch of
// 16 rows and set the kernel's tail (1.1 ms of a 34.5-ms C4 step).  Here 256 threads
// select the `take` best appended rows by (u, row) with block-wide reductions, score them,
// then filter EVERY appended row against the resulting exact bound L at once and score the
// survivors P8_ROWS at a time (two threads per row: numpy's two einsum lanes).  Same rows in,
// same exact top-k out: any row with u < L has exact <= u < L <= e_k (strictly below the final k-th,
// so not even a tie), whatever order the survivors are scored in.
constexpr int P8_THREADS = 256;
constexpr int P8_ROWS = P8_THREADS / 2;  // rows scored per round (a thread pair per row)

// einsum_chain with the query already in fp64 (converted once per query): the fp64 pipe runs
// the dependent DFMA chain (24-cycle latency on B200, scripts/micro/dfma.cu) and every
// F2F.F64.F32 conversion, so converting the query once halves the conversions.  Bit-identical:
// (double)q is exact, so fma((double)x, qd, a) == fma((double)x, (double)q, a).
__device__ __forceinline__ double einsum_chain_qd(const float *__restrict__ x, const double *__restrict__ qd, int d,
                                                  int ch) {
    double a = 0.0;
    int j = 0;
#pragma unroll 8
    for (; j + 8 <= d; j += 8) {
        const float4 xa = __ldg(reinterpret_cast<const float4 *>(x + j));
        const float4 xb = __ldg(reinterpret_cast<const float4 *>(x + j + 4));
        a = fma((double)(ch ? xb.w : xb.z), qd[j + 6 + ch], a);
        a = fma((double)(ch ? xb.y : xb.x), qd[j + 4 + ch], a);
        a = fma((double)(ch ? xa.w : xa.z), qd[j + 2 + ch], a);
        a = fma((double)(ch ? xa.y : xa.x), qd[j + ch], a);
    }
    for (; j < d; j += 2) a = fma((double)x[j + ch], qd[j + ch], a);
    return a;
}
constexpr int P8_LIST = 2048;            // survivors buffered per pass over the appended rows

__device__ __forceinline__ void prefetch_row_l2(const float *x, int dp8, int t, int nthreads) {
    // 128-byte lines of one row, spread over the calling threads
    const char *p = reinterpret_cast<const char *>(x);
    for (int o = t * 128; o < dp8 * 4; o += nthreads * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + o));
}

// The chain with the row streamed through a ring of P8_G blocks of 8 elements: each block's
// slot is refilled with the block P8_G ahead right after it is consumed (static register
// indices: the inner loop is unrolled over the ring), so P8_G blocks stay in flight instead of
// one memory round trip per block.  d must be a multiple of 8 P8_G (else the plain loop).
constexpr int P8_G = 4;
__device__ __forceinline__ double einsum_chain_qd_pf(const float *__restrict__ x, const double *__restrict__ qd, int d,
                                                     int ch) {
    const float4 *xp = reinterpret_cast<const float4 *>(x);
    const int nblk = d >> 3;
    float4 ring[2 * P8_G];
#pragma unroll
    for (int u = 0; u < 2 * P8_G; ++u) ring[u] = __ldg(xp + u);
    double a = 0.0;
#pragma unroll 1
    for (int b0 = 0; b0 < nblk; b0 += P8_G) {
#pragma unroll
        for (int u = 0; u < P8_G; ++u) {
            const float4 xa = ring[2 * u], xb = ring[2 * u + 1];
            const int nb = b0 + u + P8_G;
            if (nb < nblk) {
                ring[2 * u] = __ldg(xp + 2 * nb);
                ring[2 * u + 1] = __ldg(xp + 2 * nb + 1);
            }
            const double *q = qd + (b0 + u) * 8;
            a = fma((double)(ch ? xb.w : xb.z), q[6 + ch], a);
            a = fma((double)(ch ? xb.y : xb.x), q[4 + ch], a);
            a = fma((double)(ch ? xa.w : xa.z), q[2 + ch], a);
            a = fma((double)(ch ? xa.y : xa.x), q[ch], a);
        }
    }
    return a;
}

__global__ void __launch_bounds__(P8_THREADS, 4) tc8_post_cta_kernel(I8PostArgs a) {
    extern __shared__ __align__(16) double qd[];  // [dp8] the query in fp64
    __shared__ double ts[TC_KP];
    __shared__ int32_t tr[TC_KP];
    __shared__ int32_t list[P8_LIST];
    __shared__ double ex[P8_ROWS];
    __shared__ int32_t ins[P8_ROWS];
    __shared__ uint64_t keys[P8_THREADS];
    __shared__ uint64_t red[P8_THREADS / 32];
    __shared__ int s_n, s_nl, s_scored, s_nins;
    __shared__ float s_L;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nq_live = live_nq(a.nq_dev, a.nq);
    for (int64_t q = blockIdx.x; q < nq_live; q += gridDim.x) {
        const int take = (int)(a.row_limit ? min(a.take, max((int64_t)0, a.row_limit[q])) : a.take);
        const int cnt = a.acount[q];
        long long c0 = a.clk ? clock64() : 0, c1 = c0, c2 = c0;
        int rounds = 0, passes = 0;
        if (tid == 0) atomicAdd(&a.counters[3], cnt);
        if (take > 0 && cnt > a.cap) {
            if (tid == 0) a.fallback[atomicAdd(&a.counters[0], 1)] = (int32_t)q;
            continue;  // uniform: every thread read the same cnt
        }
        const float *qv = a.qp + q * (int64_t)a.dp8;
        if (take > 0) {
            for (int j = tid; j < a.dp8; j += P8_THREADS) qd[j] = (double)qv[j];
            if (tid == 0) {
                const int n0 = a.seed_n ? min(a.seed_n[q], take) : 0;
                for (int j = 0; j < n0; ++j) {
                    ts[j] = a.seed_s[q * TC_KP + j];
                    tr[j] = a.seed_rows[q * TC_KP + j];
                }
                s_n = n0;
                s_nl = 0;
                s_scored = 0;
            }
            __syncthreads();
            const uint2 *e = a.abuf + q * (int64_t)a.cap;
            // the scan published a lower bound on e_k for this query (k distinct rows' exact
            // scores, rounded down): every row that can reach the top-k has u >= it, so the
            // refill below can filter with it at once — no first round of scoring
            const float Lscan = a.lg ? ord2f(__ldg(a.lg + q)) : -INFINITY;
            // (1) promising rows to score first, in ONE pass over the appended list: every
            // thread's largest (u, row) key, then the `take` largest of those 256 (warp 0).
            // Any rows would do for correctness (the refill below filters against the exact
            // bound they yield); the largest u give a tight bound early.
            if (Lscan == -INFINITY) {
                uint64_t best = 0;
#pragma unroll 4
                for (int i = tid; i < cnt; i += P8_THREADS) {
                    const uint2 v = e[i];
                    const uint64_t key = cand_key(__uint_as_float(v.y), v.x);
                    best = key > best ? key : best;
                }
                keys[tid] = best;
                __syncthreads();
                if (warp == 0) {
                    uint64_t kl[P8_THREADS / 32];
#pragma unroll
                    for (int x = 0; x < P8_THREADS / 32; ++x) kl[x] = keys[lane * (P8_THREADS / 32) + x];
                    for (int j = 0; j < take; ++j) {
                        uint64_t m = 0;
                        int mx = 0;
#pragma unroll
                        for (int x = 0; x < P8_THREADS / 32; ++x)
                            if (kl[x] > m) {
                                m = kl[x];
                                mx = x;
                            }
                        uint64_t wm = m;
                        for (int o = 16; o; o >>= 1) {
                            const uint64_t ob = __shfl_xor_sync(0xffffffffu, wm, o);
                            wm = ob > wm ? ob : wm;
                        }
                        if (wm == 0) break;
                        if (m == wm) {  // keys are unique (rows are): exactly one lane owns it
#pragma unroll
                            for (int x = 0; x < P8_THREADS / 32; ++x)
                                if (x == mx) kl[x] = 0;
                            const int32_t row = (int32_t)key_row(wm);
                            bool dup = false;
                            for (int t = 0; t < s_n; ++t) dup |= (tr[t] == row);
                            if (!dup) list[s_nl++] = row;
                        }
                        __syncwarp();
                    }
                }
                __syncthreads();
            }
            // the bound before any appended row is scored: the seeds' k-th (phase (1) may have
            // selected only seeds, and then no scoring round below sets it)
            if (tid == 0) s_L = fmaxf(Lscan, (s_n == take) ? __double2float_rd(ts[take - 1]) : -INFINITY);
            __syncthreads();
            int nl = s_nl;
            if (a.clk) c1 = clock64();
            // (2) score the buffered rows P8_ROWS at a time, insert, tighten L; (3) refill the
            // buffer with every appended row still able to reach the top-k, repeat
            int next = 0;  // next appended entry to filter
            bool filtered_all = false;
            for (;;) {
                for (int b0 = 0; b0 < nl; b0 += P8_ROWS) {
                    ++rounds;
                    const int nb = min(P8_ROWS, nl - b0);
                    const int r = tid >> 1, ch = tid & 1;
                    double acc = 0.0;
                    if (r < nb) {
                        const float *xr = a.x32 + (int64_t)list[b0 + r] * a.dp8;
                        if (a.pf && a.d % (8 * P8_G) == 0)
                            acc = einsum_chain_qd_pf(xr, qd, a.d, ch);
                        else
                            acc = einsum_chain_qd(xr, qd, a.d, ch);
                    }
                    const double other = __shfl_xor_sync(0xffffffffu, acc, 1);
                    // only rows that rank before the current k-th can enter the list (the k-th only
                    // rises while they are inserted, so this pre-filter never drops one that would
                    // stay): thread 0 inserts those few instead of walking all nb scored rows
                    if (tid == 0) s_nins = 0;
                    __syncthreads();
                    if (ch == 0 && r < nb) {
                        const double sc = 0.0 + (acc + other);
                        const int n0 = s_n;
                        if (n0 < take || ranks_before(sc, list[b0 + r], ts[take - 1], tr[take - 1])) {
                            const int slot = atomicAdd(&s_nins, 1);
                            ex[slot] = sc;
                            ins[slot] = list[b0 + r];
                        }
                    }
                    __syncthreads();
                    if (tid == 0) {
                        int n = s_n;
                        for (int j = 0; j < s_nins; ++j) top_insert(ts, tr, n, take, ex[j], ins[j]);
                        s_n = n;
                        s_scored += nb;
                        s_L = fmaxf(Lscan, (n == take) ? __double2float_rd(ts[take - 1]) : -INFINITY);
                    }
                    __syncthreads();
                }
                if (filtered_all) break;
                // refill: appended rows with u >= L that are not in the list yet
                if (tid == 0) s_nl = 0;
                __syncthreads();
                const float L = s_L;
                const int n = s_n;
                constexpr int P8_U = 4;  // entries per thread per pass: loads in flight together
                for (; next < cnt; next += P8_U * P8_THREADS) {
                    ++passes;
                    uint2 v[P8_U];
#pragma unroll
                    for (int u = 0; u < P8_U; ++u) {
                        const int i = next + u * P8_THREADS + tid;
                        v[u] = i < cnt ? e[i] : make_uint2(0u, 0u);
                    }
#pragma unroll
                    for (int u = 0; u < P8_U; ++u) {
                        const int32_t row = (int32_t)v[u].x;
                        bool pass = next + u * P8_THREADS + tid < cnt && __uint_as_float(v[u].y) >= L;
                        for (int j = 0; j < n && pass; ++j) pass = (tr[j] != row);
                        const unsigned m = __ballot_sync(0xffffffffu, pass);
                        int base = 0;
                        if (lane == 0 && m) base = atomicAdd(&s_nl, __popc(m));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (pass) {
                            const int pos = base + __popc(m & ((1u << lane) - 1));
                            list[pos] = row;
                            if (a.l2pf) prefetch_row_l2(a.x32 + (int64_t)row * a.dp8, a.dp8, 0, 1);
                        }
                    }
                    __syncthreads();
                    if (s_nl > P8_LIST - P8_U * P8_THREADS) {  // buffer nearly full: score, then continue
                        next += P8_U * P8_THREADS;
                        break;
                    }
                    __syncthreads();
                }
                nl = s_nl;
                if (next >= cnt) filtered_all = true;
                __syncthreads();
                if (nl == 0 && filtered_all) break;
            }
            if (tid == 0) atomicAdd(&a.counters[1], s_scored);
            if (a.clk) c2 = clock64();
        } else if (tid == 0) {
            s_n = 0;
        }
        __syncthreads();
        // outputs (warp 0): self-snap (element-wise equal stored row, index.py:180-181) + clamp (:185)
        if (warp == 0) {
            const int n = s_n;
            for (int j = 0; j < a.k; ++j) {
                const int64_t o = q * a.k + j;
                if (j >= n) {
                    if (lane == 0) {
                        a.rows[o] = -1;
                        if (a.raw) a.raw[o] = 0.0;
                        if (a.rep) a.rep[o] = 0.0;
                    }
                    continue;
                }
                const double bs = ts[j];
                const int64_t br = tr[j];
                double rep = bs;
                if (bs > 1.0 - 1e-6) {
                    const float *x = a.x32 + br * (int64_t)a.dp8;
                    int bad = 0;
                    for (int t = lane; t < a.d; t += 32) bad |= !(x[t] == qv[t]);
                    if (!__any_sync(0xffffffffu, bad)) rep = 1.0;
                }
                if (lane == 0) {
                    a.rows[o] = br;
                    if (a.raw) a.raw[o] = bs;
                    if (a.rep) a.rep[o] = fmax(-1.0, fmin(1.0, rep));
                }
            }
            if (lane == 0) a.count[q] = n;
        }
        if (a.clk && tid == 0) {
            const long long c3 = clock64();
            atomicAdd(&a.clk[0], (unsigned long long)(c1 - c0));
            atomicAdd(&a.clk[1], (unsigned long long)(c2 - c1));
            atomicAdd(&a.clk[2], (unsigned long long)(c3 - c2));
            atomicAdd(&a.clk[3], (unsigned long long)rounds);
            atomicAdd(&a.clk[4], (unsigned long long)passes);
            atomicAdd(&a.clk[5], 1ull);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// host side

int i8_quantize_rows(const float *src, int64_t n, int d, const int64_t *rows, int64_t row0, int dp128, I8Rows &m,
                     cudaStream_t st) {
    if (n == 0) return PR_OK;
    const int64_t threads = n * 32;
    ::pr::count_launch();
    quantize_rows_kernel<<<(unsigned)ceil_div<int64_t>(threads, 256), 256, 0, st>>>(src, n, d, rows, row0, dp128, m.x8,
                                                                                   m.xs, m.xe, m.xt, m.maxnorm);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

int i8_gather_rows(const I8Rows &src, const int64_t *src_rows, int64_t n, int dp128, int64_t row0, I8Rows &m,
                   cudaStream_t st) {
    if (n == 0) return PR_OK;
    const int64_t total = n * (dp128 / 16);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div<int64_t>(total, 256), (int64_t)sm_count() * 16));
    ::pr::count_launch();
    gather_i8_kernel<<<grid, 256, 0, st>>>(src.x8, src.xs, src.xe, src.maxnorm, src_rows, n, dp128, row0, m.x8, m.xs,
                                           m.xe, m.xt, m.maxnorm);
    PR_LAUNCH_CHECK();
    return PR_OK;
}

int i8_make_store_map(TcStoreMap *m, const int8_t *x8, int64_t rows, int dp128, int box_rows) {
    return make_map_2d(&m->map, x8, rows, dp128, 1, I8_BLOCK_K, box_rows);
}

// appended rows kept per query (a query that overflows is rescanned exactly):
// min(32768, n), shrunk only when the batch's buffer would pass 1 GB
static int i8_cap(int64_t n, int64_t nq) {
    int64_t cap = std::min<int64_t>(I8_CAP, round_up<int64_t>(std::max<int64_t>(n, 1), 256));
    const int64_t budget = (int64_t)1 << 30;
    if (cap * 8 * std::max<int64_t>(nq, 1) > budget) cap = std::max<int64_t>(4096, budget / (8 * std::max<int64_t>(nq, 1)));
    return (int)cap;
}

// pilot: every stride-th 256-row tile, the stride chosen so the pilot samples ~160 tiles
// (clamped to [16, 128]), when the store has at least 8 strides of tiles.  With the refiners'
// union bound (gunion_insert) the main scan tightens its own bound, so a sparse pilot is
// enough on a large store — continuous blocks, top-5, B = 4096: 10M rows: stride 128 vs 32,
// 35.92 vs 36.45 ms (no pilot 38.67); 2.5M rows: 128 / 64 / 32 all 9.92-9.99 ms — while a short
// store wants a denser one — 1.25M rows (one of 8 row shards): 128 / 64 / 32 / 24 / 16 / 8 ->
// 6.08 / 5.94 / 5.79 / 5.76 / 5.77 / 5.96 ms
static int pilot_stride(int64_t ntiles) {
    const char *e = getenv("PR_I8_PILOT_STRIDE");  // measurement knob (read per search)
    if (e) return std::max(2, atoi(e));
    return (int)std::min<int64_t>(128, std::max<int64_t>(16, ntiles / 160));
}

static int pilot_splits(int64_t qtiles, int64_t ntiles) {
    const int stride = pilot_stride(ntiles);
    if (ntiles < 8 * (int64_t)stride) return 0;
    const int64_t ptiles = ceil_div<int64_t>(ntiles, stride);
    const char *e = getenv("PR_I8_PSPLIT");  // measurement knob: pilot row splits
    if (e && atoi(e) > 0) return (int)std::min<int64_t>(ptiles, atoi(e));
    // ONE wave: each pilot item pays a cold start (its first tile floods the cooperative path
    // before its lists fill), so fewer, longer items win — measured at 10M x 1024 (pilot ms,
    // ncu): B = 4096: 4 splits 0.66 vs 9 (two waves) 0.74; B = 2048: 2/3/4/6 splits 0.93 /
    // 0.74 / 0.65 / 0.54 vs 18 (two waves) 0.94
    return (int)std::max<int64_t>(1, std::min<int64_t>(ptiles, (int64_t)sm_count() / std::max<int64_t>(1, qtiles)));
}

bool tc8_eligible(int d) { return d <= 2048; }

// PR_I8_CG=1 selects the single-CTA MMA (default: 2-CTA pairs)
static int i8_cg() {
    const char *e = getenv("PR_I8_CG");
    return (e && e[0] == '1') ? 1 : 2;
}

template <bool PILOT, int CG, bool ARES = false, int MC = 1>
static int scan8_config(cudaLaunchConfig_t &cfg, cudaLaunchAttribute *at, int64_t ctas, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        PR_CUDA(cudaFuncSetAttribute(tc8_scan_kernel<PILOT, CG, ARES, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)i8_smem_bytes<CG, ARES>()));
        attr = true;
    }
    cfg = {};
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3(I8_THREADS);
    cfg.dynamicSmemBytes = i8_smem_bytes<CG, ARES>();
    cfg.stream = st;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG * MC;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return PR_OK;
}

template <bool PILOT, int CG, bool ARES = false, int MC = 1>
static int launch_scan8(int64_t ctas, const CUtensorMap &tq, const CUtensorMap &tx, const I8ScanParams &p,
                        cudaStream_t st) {
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[1];
    int rc = scan8_config<PILOT, CG, ARES, MC>(cfg, at, ctas, st);
    if (rc) return rc;
    ::pr::count_launch();
    PR_CUDA(cudaLaunchKernelEx(&cfg, tc8_scan_kernel<PILOT, CG, ARES, MC>, tq, tx, p));
    return PR_OK;
}

// clusters of 2 * MC CTAs the device holds at once (a GPC need not split into them evenly)
template <int MC>
static int scan8_max_clusters() {
    static int cached = -1;
    if (cached < 0) {
        cudaLaunchConfig_t cfg;
        cudaLaunchAttribute at[1];
        int n = 0;
        if (scan8_config<false, 2, true, MC>(cfg, at, 2 * MC, nullptr) != PR_OK ||
            cudaOccupancyMaxActiveClusters(&n, tc8_scan_kernel<false, 2, true, MC>, &cfg) != cudaSuccess || n <= 0) {
            (void)cudaGetLastError();
            n = sm_count() / (2 * MC);
        }
        cached = n;
    }
    return cached;
}

template <bool PILOT>
static int launch_scan8_cg(int cg, bool ares, int64_t ctas, const CUtensorMap &tq, const CUtensorMap &tx,
                           const I8ScanParams &p, cudaStream_t st) {
    if (cg == 2)
        return ares ? launch_scan8<PILOT, 2, true>(ctas, tq, tx, p, st) : launch_scan8<PILOT, 2, false>(ctas, tq, tx, p, st);
    return launch_scan8<PILOT, 1>(ctas, tq, tx, p, st);
}

// Query tile resident in smem (PR_I8_ARES=0 streams it with every store tile instead).  Measured in
// continuous runs (scripts/clock_probe.sh): 35.1 vs 38.4 ms at 10M x 1024 — half the L2->SM bytes,
// so the power-capped clock rises 1510 -> 1640 MHz.  (Interleaved in-process A/B cannot see this:
// alternating calls share one power-averaging window.)
static bool i8_ares(int cg, int dp128) {
    const char *e = getenv("PR_I8_ARES");
    return cg == 2 && dp128 <= 1024 && !(e && e[0] == '0');
}

// CTA pairs per cluster sharing multicast store tiles in the A-resident main scan
// (PR_I8_MC = 1 (default), 2 or 4; see tc8_scan_kernel and DESIGN §4.0: fewer L2->SM bytes,
// but 4-CTA clusters fit on only 132 of the 148 SMs and the energy per search rose)
static int i8_mc(bool ares) {
    if (!ares) return 1;
    const char *e = getenv("PR_I8_MC");
    const int v = e ? atoi(e) : 1;
    return (v == 2 || v == 4) ? v : 1;
}

size_t tc8_scratch_bytes(int64_t nq, int dp128, int64_t n) {
    const int64_t nq_pad = round_up<int64_t>(nq, 2 * TC_BLOCK_M);
    const int64_t qtiles = nq_pad / TC_BLOCK_M, ntiles = ceil_div<int64_t>(n, TC_BLOCK_N);
    const int ps = pilot_splits(qtiles, ntiles);
    return (size_t)nq_pad * dp128 + (size_t)nq_pad * 16 + (size_t)nq * (4 + 4 + 4 + 4) +
           (size_t)nq * i8_cap(n, nq) * 8 + (size_t)nq * ps * I8_HALVES * TC_KP * 8 + (size_t)nq * TC_KP * 12 +
           (size_t)qtiles * 4 * 1024 + (size_t)nq * TC_KP * 4 + 65536;
}

int tc8_search(Tc8Search &s, Carve &cv, cudaStream_t st, pr_search_stats *stats) {
    const int cg = i8_cg();
    const int64_t nq_pad = round_up<int64_t>(s.nq, cg * TC_BLOCK_M);
    const int64_t qtiles = nq_pad / TC_BLOCK_M;
    const int64_t ntiles = ceil_div<int64_t>(s.n, TC_BLOCK_N);
    // a device-sized query list: shape the grid for the host's estimate of the live count
    const int64_t qtiles_hint =
        s.nq_dev ? round_up<int64_t>(ceil_div<int64_t>(std::max<int64_t>(1, std::min(s.nq_hint, s.nq)), TC_BLOCK_M), cg)
                 : qtiles;
    const bool ares = i8_ares(cg, s.dp128);
    const int mc = i8_mc(ares);
    // MC > 1: one work unit = a cluster of MC pairs; the split count is chosen for the
    // clusters the device holds at once
    const int64_t units_hint = ceil_div<int64_t>(qtiles_hint, 2 * mc);
    int nsplit = mc > 1 ? choose_nsplit_slots(units_hint, ntiles, mc == 4 ? scan8_max_clusters<4>() : scan8_max_clusters<2>())
                        : choose_nsplit_waves(qtiles_hint, ntiles);
    const char *ns_env = getenv("PR_I8_NSPLIT");  // measurement knob
    if (ns_env && atoi(ns_env) > 0) nsplit = (int)std::min<int64_t>(ntiles, atoi(ns_env));
    const int tps = (int)ceil_div<int64_t>(ntiles, nsplit);
    nsplit = (int)ceil_div<int64_t>(ntiles, tps);
    if (getenv("PR_I8_VERBOSE"))  // measurement knob
        fprintf(stderr, "tc8_search: nq=%lld qtiles=%lld ntiles=%lld mc=%d max_clusters=%d nsplit=%d tps=%d\n",
                (long long)s.nq, (long long)qtiles_hint, (long long)ntiles, mc,
                mc == 4 ? scan8_max_clusters<4>() : (mc == 2 ? scan8_max_clusters<2>() : 0), nsplit, tps);
    const int cap = i8_cap(s.n, s.nq);
    int8_t *q8 = cv.take<int8_t>((size_t)nq_pad * s.dp128);
    float4 *qmeta = cv.take<float4>((size_t)nq_pad);
    uint32_t *lg = cv.take<uint32_t>((size_t)s.nq);
    int32_t *acount = cv.take<int32_t>((size_t)s.nq);
    uint2 *abuf = cv.take<uint2>((size_t)s.nq * cap);
    s.fallback_list = cv.take<int32_t>((size_t)s.nq);
    PR_CUDA(cudaMemsetAsync(lg, 0, (size_t)s.nq * 4, st));
    PR_CUDA(cudaMemsetAsync(acount, 0, (size_t)s.nq * 4, st));
    PR_CUDA(cudaMemsetAsync(s.counters, 0, 4 * sizeof(int32_t), st));
    {
        const int64_t threads = nq_pad * 32;
        ::pr::count_launch();
        quantize_queries_kernel<<<(unsigned)ceil_div<int64_t>(threads, 256), 256, 0, st>>>(
            s.qp, s.nq, nq_pad, s.dp8, s.d, s.dp128, s.rows8.maxnorm, q8, qmeta, s.nq_dev);
        PR_LAUNCH_CHECK();
    }
    TcStoreMap qmap;
    int rc = make_map_2d(&qmap.map, q8, nq_pad, s.dp128, 1, I8_BLOCK_K, TC_BLOCK_M);
    if (rc) return rc;
    const size_t wsmem = (size_t)W8_WARPS * (s.dp8 + 8) * sizeof(float);
    const CUtensorMap &xmap = (cg == 2 ? s.store_map_half : s.store_map)->map;
    TcStoreMap xmap_mc;  // MC > 1: each CTA fetches 128 / MC rows of its half-tile
    if (mc > 1) {
        rc = i8_make_store_map(&xmap_mc, s.rows8.x8, s.x8_rows, s.dp128, 128 / mc);
        if (rc) return rc;
    }
    static bool attr = false;
    if (!attr) {
        PR_CUDA(cudaFuncSetAttribute(tc8_seed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024));
        PR_CUDA(cudaFuncSetAttribute(tc8_post_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024));
        attr = true;
    }
    const char *ceil_env = getenv("PR_I8_CEILING");  // 1: no row can pass (results invalid): fast-path timing
    // a caller's floor (pr_index_search_floor) as the scan's first bound: rows with u < floor
    // have exact < floor.  Snapped self-matches (raw > 1 - 1e-6, reported 1.0) must survive a
    // floor up to 1, and the bound is an fp32 value rounded DOWN.
    float floor_thr = -INFINITY;
    if (s.floor > -INFINITY) {
        const double fe = std::min(s.floor, 1.0 - 1e-6) - 1e-6;
        floor_thr = (float)fe;
        if ((double)floor_thr > fe) floor_thr = std::nextafter(floor_thr, -INFINITY);
    }
    if (ceil_env && ceil_env[0] == '1') floor_thr = INFINITY;
    const unsigned wgrid = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(ceil_div<int64_t>(s.nq, W8_WARPS), (int64_t)sm_count() * 8));

    // 1) pilot over a tile subsample -> exact seeds and a first bound per query
    const int psplit = s.floor > -INFINITY ? 0 : pilot_splits(qtiles_hint, ntiles);
    int32_t *seed_rows = nullptr, *seed_n = nullptr;
    double *seed_s = nullptr;
    if (psplit > 0) {
        const int pstride = pilot_stride(ntiles);
        const int64_t ptiles = ceil_div<int64_t>(ntiles, pstride);
        uint64_t *pcand = cv.take<uint64_t>((size_t)s.nq * psplit * I8_HALVES * TC_KP);
        seed_rows = cv.take<int32_t>((size_t)s.nq * TC_KP);
        seed_s = cv.take<double>((size_t)s.nq * TC_KP);
        seed_n = cv.take<int32_t>((size_t)s.nq);
        I8ScanParams pp{s.n, s.dp128 / I8_BLOCK_K, psplit, (int)ceil_div<int64_t>(ptiles, psplit), (int)ptiles,
                        (int)qtiles, s.k, s.rows8.xs, s.rows8.xe, s.rows8.xt, qmeta, s.row_limit, s.nq, lg, acount,
                        abuf, cap, floor_thr, 0, pstride, pcand, s.x32, s.qp, s.dp8, s.d, 0, nullptr, 0, s.nq_dev};
        rc = launch_scan8_cg<true>(cg, ares, (s.nq_dev ? qtiles_hint : qtiles) * psplit, qmap.map, xmap,
                                   pp, st);
        if (rc) return rc;
        I8SeedArgs sa{pcand, psplit, s.nq, s.k, s.x32, s.dp8, s.d, s.qp, seed_rows, seed_s, seed_n, lg, s.nq_dev};
        ::pr::count_launch();
        tc8_seed_kernel<<<wgrid, W8_WARPS * 32, wsmem, st>>>(sa);
        PR_LAUNCH_CHECK();
    }
    // 2) main scan: append every row whose upper bound reaches the running bound
    I8ScanParams p{s.n, s.dp128 / I8_BLOCK_K, nsplit, tps, (int)ntiles, (int)qtiles, s.k, s.rows8.xs, s.rows8.xe,
                   s.rows8.xt, qmeta, s.row_limit, s.nq, lg, acount, abuf, cap, floor_thr, 0, 1, nullptr, s.x32, s.qp,
                   s.dp8, s.d, 1, nullptr, 0, s.nq_dev};
    {
        const char *rf_env = getenv("PR_I8_REFINEF");  // 0: exact fp64 refiner scores (A/B knob)
        p.refine_fast = !(rf_env && rf_env[0] == '0');
        {
            // the factor g of dot_f32_lower's error bound, rounded up
            const double u = std::ldexp(1.0, -24), m = (double)s.d + 3.0;
            p.refine_err = (float)(m * u / (1.0 - m * u) * 1.0001);
        }
        const char *f_env = getenv("PR_I8_FAST");  // 1: the single-level fast path (A/B knob)
        p.fast2 = !(f_env && f_env[0] == '1');
        const char *gs_env = getenv("PR_I8_GSKIP");
        p.gskip = !(gs_env && gs_env[0] == '0');
        const char *g_env = getenv("PR_I8_GUNION");  // 0: no union list (A/B knob)
        if (!(g_env && g_env[0] == '0')) {
            p.gun = cv.take<uint32_t>((size_t)s.nq * TC_KP);
            PR_CUDA(cudaMemsetAsync(p.gun, 0, (size_t)s.nq * TC_KP * sizeof(uint32_t), st));
        }
    }
    {
        const char *w_env = getenv("PR_I8_WINDOW");  // tiles a pair may run ahead of its split (0 = off)
        p.window = w_env ? atoi(w_env) : 0;  // measured: 48 tiles halves DRAM reads but costs 50 % time
        if (cg == 2 && mc == 1 && p.window > 0 && !s.nq_dev) {
            p.prog = cv.take<int32_t>((size_t)nsplit * (qtiles / 2));
            PR_CUDA(cudaMemsetAsync(p.prog, 0, (size_t)nsplit * (qtiles / 2) * sizeof(int32_t), st));
        } else {
            p.window = 0;
        }
    }
    const char *ref_env = getenv("PR_I8_REFINE");  // 0: no in-kernel refinement (A/B knob)
    p.refine = !(ref_env && ref_env[0] == '0');
    const char *noepi_env = getenv("PR_I8_NOEPI");  // 1: epilogue does nothing (results invalid): MMA/TMA timing
    if (noepi_env && noepi_env[0] >= '1') p.noepi = noepi_env[0] - '0';  // 2: also skip operand loads
    const bool verbose = getenv("PR_I8_VERBOSE") != nullptr;
    if (verbose) {
        p.dbg = cv.take<uint32_t>(4);
        PR_CUDA(cudaMemsetAsync(p.dbg, 0, 16, st));
    }
    if (s.ev_begin) PR_CUDA(cudaEventRecord(s.ev_begin, st));
    if (mc > 1) {
        const int64_t units = ceil_div<int64_t>(s.nq_dev ? qtiles_hint : qtiles, 2 * mc);
        rc = mc == 4 ? launch_scan8<false, 2, true, 4>(units * 8 * nsplit, qmap.map, xmap_mc.map, p, st)
                     : launch_scan8<false, 2, true, 2>(units * 4 * nsplit, qmap.map, xmap_mc.map, p, st);
    } else {
        rc = launch_scan8_cg<false>(cg, ares, (s.nq_dev ? qtiles_hint : qtiles) * nsplit, qmap.map, xmap, p, st);
    }
    if (rc) return rc;
    if (s.ev_end) PR_CUDA(cudaEventRecord(s.ev_end, st));
    if (verbose) {  // measurement only: synchronises the stream
        uint32_t h[4];
        PR_CUDA(cudaMemcpyAsync(h, p.dbg, 16, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr,
                "tc8_search: cooperative warp-chunks %u of %u (%.4f), flagged groups %u (%.2f per query), per-row "
                "fast-path warp-chunks %u (%.4f)\n",
                h[0], h[1], h[1] ? (double)h[0] / h[1] : 0.0, h[2], (double)h[2] / std::max<int64_t>(1, s.nq), h[3],
                h[1] ? (double)h[3] / h[1] : 0.0);
        std::vector<int32_t> ac((size_t)s.nq);
        PR_CUDA(cudaMemcpyAsync(ac.data(), acount, (size_t)s.nq * 4, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
        std::vector<int32_t> srt(ac);
        std::sort(srt.begin(), srt.end());
        const size_t m = srt.size();
        if (m)
            fprintf(stderr, "tc8_search: appended per query: median %d p90 %d p99 %d max %d (query %lld)\n", srt[m / 2],
                    srt[m * 9 / 10], srt[m * 99 / 100], srt[m - 1],
                    (long long)(std::max_element(ac.begin(), ac.end()) - ac.begin()));
    }
    // 3) exact rescoring of the complete candidate set
    unsigned long long *pclk = nullptr;
    if (verbose) {
        pclk = cv.take<unsigned long long>(8);
        PR_CUDA(cudaMemsetAsync(pclk, 0, 64, st));
    }
    const char *pf_env = getenv("PR_I8_POSTPF");
    I8PostArgs pa{pclk, !(pf_env && pf_env[0] == '0'), acount, abuf, cap, s.nq, s.k, std::min<int64_t>(s.k, s.n), s.row_limit, s.x32, s.dp8, s.d, s.qp,
                  seed_rows, seed_s, seed_n, s.rows, s.raw, s.rep, s.count, s.counters, s.fallback_list, s.nq_dev,
                  nullptr};
    const char *pl2_env = getenv("PR_I8_POSTL2");
    if (pl2_env && pl2_env[0] == '1') pa.l2pf = 1;
    const char *plg_env = getenv("PR_I8_POSTLG");
    if (!(plg_env && plg_env[0] == '0')) pa.lg = lg;
    const char *post_env = getenv("PR_I8_POST");  // "warp": the warp-per-query kernel (A/B knob)
    ::pr::count_launch();
    if (post_env && post_env[0] == 'w') {
        tc8_post_kernel<<<wgrid, W8_WARPS * 32, wsmem, st>>>(pa);
    } else {
        const char *pg_env = getenv("PR_I8_POSTGRID");  // measurement knob: post CTAs per SM
        const int per_sm = pg_env && atoi(pg_env) > 0 ? atoi(pg_env) : 8;
        const unsigned pgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(s.nq, (int64_t)sm_count() * per_sm));
        const size_t psmem = (size_t)s.dp8 * sizeof(double);
        static bool p8_attr = false;
        if (!p8_attr) {
            PR_CUDA(cudaFuncSetAttribute(tc8_post_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
            p8_attr = true;
        }
        tc8_post_cta_kernel<<<pgrid, P8_THREADS, psmem, st>>>(pa);
    }
    PR_LAUNCH_CHECK();
    if (pclk) {  // measurement only: synchronises
        unsigned long long h[8];
        PR_CUDA(cudaMemcpyAsync(h, pclk, 64, cudaMemcpyDeviceToHost, st));
        PR_CUDA(cudaStreamSynchronize(st));
        const double nq = (double)std::max<unsigned long long>(1, h[5]);
        fprintf(stderr, "tc8_post: per query: select %.0f cycles, score+refill %.0f cycles (%.2f rounds, %.2f passes), "
                        "outputs %.0f cycles\n", h[0] / nq, h[1] / nq, h[3] / nq, h[4] / nq, h[2] / nq);
    }
    stats->nsplit = nsplit;
    return PR_OK;
}

}  // namespace pr
