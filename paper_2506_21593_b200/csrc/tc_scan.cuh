// Internal interface between index.cu (orchestration) and the tensor-core
// score+select path (tc_scan.cu) / the large-k path (bigk.cu).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace pr {

struct alignas(64) TcStoreMap {
    CUtensorMap map;
};

// Candidates kept per (query, row split) by the tcgen05 epilogue.
constexpr int TC_KP = 16;
constexpr int TC_BLOCK_M = 128;  // queries per CTA (TMEM lanes)
constexpr int TC_BLOCK_N = 256;  // store rows per MMA tile (TMEM columns)
constexpr int TC_BLOCK_K = 64;   // fp16 columns per stage = one 128B swizzle atom

struct Carve;

struct TcSearch {
    const float *x32;
    const __half *x16;
    const TcStoreMap *store_map;
    int64_t n;
    int d, dp8, dp64;
    const float *q32;  // caller queries [nq, d]
    const float *qp;   // padded fp32 queries [nq, dp8]
    int64_t nq;
    int k;
    int64_t *rows;
    double *raw, *rep;
    int32_t *count;
    int32_t *counters;      // [0] fallback count, [1] rescored candidates
    int32_t *fallback_list; // out: query ids failing the certificate
    cudaEvent_t ev_begin = nullptr, ev_end = nullptr;  // optional scan-kernel timing
    const int64_t *row_limit = nullptr;                  // per query: rows >= limit invisible
};

// int8 tcgen05 scan (tc_scan_i8.cu): per-row quantised store + complete candidate set
// per 256-row tile: max quantisation error bound and per-8-row-group max scale
// (loose tests of the scan's fast path); both only grow, so they stay bounds
struct alignas(16) I8TileMeta {
    float dxmax;
    float pad[3];
    float gmax[32];
};
struct I8Rows {
    int8_t *x8 = nullptr;         // [cap256, dp128] quantised rows
    float *xs = nullptr;          // [cap256] per-row scale s_r
    float *xe = nullptr;          // [cap256] rounded-up ||x_r - s_r xq_r||_2
    I8TileMeta *xt = nullptr;     // [cap256 / 256] per-tile bounds
    uint32_t *maxnorm = nullptr;  // device scalar: max ||x_r|| (fp32 bits, rounded up)
};
struct Tc8Search {
    const float *x32;
    const TcStoreMap *store_map;       // TMA map of rows8.x8, 256-row boxes (cta_group::1)
    const TcStoreMap *store_map_half;  // ... 128-row boxes (cta_group::2: each CTA loads half a tile)
    I8Rows rows8;
    int64_t x8_rows = 0;  // rows of rows8.x8 (the TMA maps' extent)
    int64_t n;
    int d, dp8, dp128;
    const float *qp;  // padded fp32 queries [nq, dp8]
    int64_t nq;
    int k;
    int64_t *rows;
    double *raw, *rep;
    int32_t *count;
    int32_t *counters;       // [0] fallback, [1] rescored rows, [3] appended rows
    int32_t *fallback_list;  // out: queries whose candidate buffer overflowed
    cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
    const int64_t *row_limit = nullptr;
    // device-resident query count (a compacted miss list): queries [*nq_dev, nq) are
    // skipped by every kernel; the grid is shaped for nq_hint queries (host estimate)
    const int32_t *nq_dev = nullptr;
    int64_t nq_hint = 0;
    // pr_index_search_floor: rows whose exact score is below the floor need not be found
    // (-inf = a plain search); the scan's bound starts at the floor and the pilot is skipped
    double floor = -INFINITY;
};
int i8_quantize_rows(const float *src, int64_t n, int d, const int64_t *rows, int64_t row0, int dp128, I8Rows &m,
                     cudaStream_t st);
int i8_gather_rows(const I8Rows &src, const int64_t *src_rows, int64_t n, int dp128, int64_t row0, I8Rows &m,
                   cudaStream_t st);
int i8_make_store_map(TcStoreMap *m, const int8_t *x8, int64_t rows, int dp128, int box_rows);
bool tc8_eligible(int d);
size_t tc8_scratch_bytes(int64_t nq, int dp128, int64_t n);
int tc8_search(Tc8Search &s, Carve &cv, cudaStream_t st, pr_search_stats *stats);

bool tc_eligible(int d, int64_t n, int k);
bool tc_worthwhile(int64_t n, int64_t nq);
size_t tc_scratch_bytes(int64_t nq, int dp64, int64_t n, int k);
int tc_make_store_map(TcStoreMap *m, const __half *x16, int64_t rows, int dp64);
int tc_search(TcSearch &s, Carve &cv, cudaStream_t st, pr_search_stats *stats);
int make_map_2d(CUtensorMap *m, const void *base, int64_t rows, int cols, int elem_bytes, int box_cols, int box_rows);
int choose_nsplit_waves(int64_t qtiles, int64_t ntiles);
int choose_nsplit_slots(int64_t units, int64_t ntiles, int slots);
// fp16 rounding + tensor-core accumulation error bound for unit vectors of dim d
double tc_error_bound(int d, int dp64);

int big_k_search(const float *x32, int64_t n, int dp8, int d, const float *q, int64_t nq, int k,
                 const int64_t *row_limit, int64_t *rows, double *raw, double *rep, int32_t *count, cudaStream_t st);

}  // namespace pr
