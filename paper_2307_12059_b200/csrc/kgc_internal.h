// kgc_internal.h -- internal (non-ABI) declarations shared by the libkgc
// translation units: tile geometry, kernel launchers, parameter blocks.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

namespace kgc {

// Experiment knobs (environment variables such as KGC_KD, KGC_GT_TB, KGC_SCHED_TC) are read
// only by a debug build (nvcc -DKGC_EXPERIMENTS): in the product build every choice is fixed by
// kgc_options and the size rules, so the environment cannot change what or how a join computes.
inline const char* kgc_knob(const char* name) {
#ifdef KGC_EXPERIMENTS
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

constexpr int BM = 128;          // query rows per tile (= TMEM lanes = UMMA M)
constexpr int BN_TC = 256;       // tail rows per tile, tensor-core engine (UMMA N)
constexpr int BN_PAIR = 128;     // tail rows per tile, CTA-pair engine on contiguous tiles (UMMA N = 128)
constexpr int BN_HALF = 128;     // tile rows (query and tail), FP16x2 L1 engine
constexpr int EST_SAMPLES = 256;  // sampled queries per relation, rank-local split estimate
constexpr int SIMT_T = 64;       // tile rows (query and tail), FP32 SIMT engines
constexpr int SORT_IPB = 2048;   // radix-sort items per block (256 threads x 8)
constexpr int TC_MAX_KPAD = 256; // tensor-core engine supports d <= 256
constexpr int MP_MAX = 128;      // multi-pivot pruning: at most 128 pivots (2..8, 12, 16, 24, 32; 48 ... 128 with L2)
constexpr int MP_G = 8;          // pivots of the per-tail test of the gathered engines (the first 8)
inline bool mp_pivots_ok(int k) {
    return k <= 8 || k == 12 || k == 16 || k == 24 || k == 32 || k == 48 || k == 64 || k == 96 || k == 128;
}
constexpr int MP_MAX_L1 = 32;    // the L1 keys (FP32, materialised) support at most 32 pivots

constexpr int MP_MAX_DIM = 256;  // multi-pivot pruning supports d <= 256
constexpr int MP_SORT_PIVOTS = 4; // Morton order over the first 4 pivots (8 bits each: 32-bit code)

// Counters block in device memory (zeroed per join).
struct DevCounters {
    unsigned long long cand;      // candidates appended by the tile kernels
    unsigned long long res;       // results appended by the verify kernel
    unsigned int nonfinite;       // != 0 if E or Rel holds a non-finite value
    unsigned int twid;            // L2 K pivots: tail-key bound delta_t 2^23 (float bits, rounded up)
    long long total_cost;         // surviving tile pairs, all shards
    long long my_cost;            // surviving tile pairs, this shard
    int tq_begin, tq_end;         // query-tile range of this shard [begin, end)
    long long n_items;            // work items of this shard
    unsigned int absmax_bits;     // max |value| over E and Rel (float bits), for the FP16 engine
    unsigned int pad1;
    long long gblocks;            // gathered-tail engine: GT_ROWS-tail blocks of this shard
    unsigned long long gpairs;    // gathered-tail engine: surviving tails summed over query tiles
};

struct TileParams {
    const float* Qp;        // staged query tiles of this shard
    const float4* qs;       // per staged query row: {Q2, Qn, Qd, thr}
    const float* Tp;        // staged tail tiles
    const float* T2;        // per staged tail row ||t||^2 (3e38 for padding rows)
    const float2* tstile;   // per tail tile {max ||t||, max ||t - tf32(t)||}
    const int4* items;      // {tq, j0, j1, list_off}: tiles j0..j1 (list_off < 0) or list[list_off + j0..j1]
    const int* tile_list;   // multi-pivot surviving tail tiles of this shard
    long long n_items;
    const long long* item_cum;  // exclusive prefix of item tile counts (cost-balanced CTA ranges)
    long long total_tiles;
    int t2pf;                   // tensor-core epilogues: prefetch ||t||^2 lines into L1 (experiment knob)
    int l2hint;                 // pair engine: L2 evict-last on the staged tails, evict-first on entity rows
    int sched;                  // 0 = round-robin items, 1 = contiguous cost-balanced blocks
    int Kpad;
    int bq, bn;             // query / tail tile rows of the plan
    int tq0;                // first staged query tile
    int N;                  // entities (query rows per relation)
    int Nt;                 // tails (valid sorted tail positions are < Nt; a partition of E, or N)
    float theta;
    float eta;              // tensor-core accumulation error coefficient
    float gam;              // FP16 engine: relative error factor (1 + gamma)
    const float* Rt;        // FP16 engine: per staged tail row residual
    int2* cand;
    unsigned long long* cand_count;
    long long cand_cap;
    // tensor-core engine: query tiles are formed on the fly from these
    const float* E;
    const float* Rel;
    const int* qperm;
    int d;
    int QT;
    // gathered-tail SIMT engine (GT_ROWS tails per block, see tiles_simt.cu)
    const float* Ts;              // sorted tails, row-major [N + 1][Kpad] (row N: sentinel)
    const int* glist;             // per query tile (at bn x its tile-list offset): surviving sorted
                                  // tail positions, padded with N to whole blocks of bn
    const float* gT2;             // tensor-core gathered blocks: ||t||^2 / 2 per list entry (3e38 padding)
    const float2* gtst;           // tensor-core gathered blocks: per block {max ||t||, max ||t - tf32(t)||}
    const void* tmap;             // tensor-core gathered blocks: CUtensorMap over Ts (device memory)
    int gb;                       // SIMT gathered blocks: tails per block (32 or 64)
    // relation-factored tensor-core engine (tiles_tc.cu, MODE 2)
    const float* fz;              // [R][N] (||h + r||^2 - theta^2) / 2 rounded down
    const float* frt;             // [R][ntpad] r.t (sorted tail positions; 0 past N)
    const float* frn;             // [R] ||r|| rounded up
    int R;
    long long ntpad;
    const long long* dn_items;    // device: work items of this shard
    const long long* dtotal;      // device: blocks of this shard (balanced CTA ranges)
    unsigned long long* prof;     // experiment: wait-cycle counters (KGC_GT_PROF), else nullptr
};

// ---- launchers (prep.cu) ----
void launch_tail_keys(const float* E, long long N, int d, int norm, const double* pivot, float* kt,
                      unsigned int* minmax_seg, unsigned int* nonfinite, cudaStream_t s);
void launch_query_keys(const float* E, const float* Rel, long long N, long long R, int d, int norm,
                       const double* pivot, float* kq, unsigned int* minmax, unsigned int* nonfinite,
                       cudaStream_t s);
void launch_pivot_mean(const float* E, long long N, int d, double* pivot, cudaStream_t s);
int  radix_sort_segments(const float* keys, const unsigned int* minmax, long long S, long long L,
                         unsigned int* k0, unsigned int* v0, unsigned int* k1, unsigned int* v1, int* counts,
                         int* perm_out, float* skeys_out, void* scan_tmp, size_t scan_tmp_bytes,
                         cudaStream_t s, int* launches);
size_t radix_counts_len(long long S, long long L);
size_t scan_tmp_bytes(size_t n);
void scan_exclusive_i32(const int* in, int* out, size_t n, void* tmp, cudaStream_t s, int* launches);
void scan_exclusive_i64(const long long* in, long long* out, size_t n, long long* total, void* tmp,
                        cudaStream_t s, int* launches);
void launch_tail_tile_bounds(const float* tskey, long long N, int BN, int TT, float* tmin, float* tmax,
                             float* cmax, float* cmin, cudaStream_t s, int* launches);
void launch_query_ranges(const float* qskey, long long N, long long R, int QT, int TT, int bq, const float* cmax,
                         const float* cmin, float theta, int prune, int2* ranges, long long* cost,
                         cudaStream_t s);
void launch_shard_items(const int2* ranges, const long long* cost, const long long* cum, long long nq,
                        int rank, int world, int chunk, DevCounters* ctr, int* nitem, int* item_off,
                        int4* items, long long* item_tiles, void* tmp, cudaStream_t s, int* launches, int phase,
                        int list_mode, long long force_lo, long long force_hi);
void launch_stage_tails(const float* E, const int* tperm, long long N, int d, int Kpad, int BN, int TT,
                        int tc_layout, float* Tp, float* T2, float2* tstile, cudaStream_t s);
void launch_stage_queries(const float* E, const float* Rel, const int* qperm, long long N, int d, int Kpad,
                          int QT, int bq, int tq0, int tq1, int tc_layout, int norm, float theta, float* Qp,
                          float4* qs, cudaStream_t s, int cyc_world = 0, int cyc_rank = 0);
// FP16x2 L1 engine staging: tiles of half2 words, element (i, k-pair p) at p * ROWS + i;
// per row the exact residual R = sum_k |v_k - fp16(v_k)| (rounded up)
void launch_stage_half(const float* E, const float* Rel, const int* perm, long long N, int d, int Kpad, int ROWS,
                       int QT, int tile0, int ntiles, float theta, float gam, void* out, float4* qs, float* rt,
                       cudaStream_t s);
void launch_split_estimate(const float* E, const float* Rel, long long N, long long R, int d, int norm, float theta,
                           float* kt, unsigned int* mm, unsigned int* hist, unsigned long long* cnt, cudaStream_t s);
void launch_absmax(const float* E, long long nE, const float* Rel, long long nR, unsigned int* out, cudaStream_t s);

// ---- multi-pivot pruning (pivots.cu) ----
void radix_sort_u64_segments(long long S, long long L, int bits, unsigned long long* k0, unsigned int* v0,
                             unsigned long long* k1, unsigned int* v1, int* counts, void* scan_tmp, cudaStream_t s,
                             int* launches);
void radix_sort_u32_segments(long long S, long long L, int bits, unsigned int* k0, unsigned int* v0, unsigned int* k1,
                             unsigned int* v1, int* counts, void* scan_tmp, cudaStream_t s, int* launches);
void launch_pick_pivots(const float* E, long long N, int d, int norm, int K, const double* p0, float* P,
                        cudaStream_t s);
void launch_mp_keys(const float* E, const float* Rel, long long N, long long nseg, int d, int norm, int K,
                    const float* P, float* keys, unsigned int* minmax, unsigned int* qnmax, unsigned int* nonfinite,
                    cudaStream_t s);
// L2 with K pivots: tail and query keys from the FP64 factorisation
// ||h + r - p||^2 = ||h - p||^2 + 2 h.r - 2 r.p + ||r||^2 (pivots.cu); scratch: A N x K, Bhr R x N,
// Cg R x (K + 1) doubles
void launch_mp_keys_l2f(const float* E, const float* Rel, long long N, long long R, const float* Et, long long NT,
                        int d, int K, const float* P, float* tkeys, unsigned int* tminmax, float* qkeys4,
                        unsigned int* qmm4, unsigned int* qnmax, double* A, double* Bhr, double* Cg, double* HP,
                        unsigned int* hmax, unsigned int* nonfinite, unsigned int* twid, cudaStream_t s,
                        cudaEvent_t bready);
void launch_mp_qkeys_all(const double* Bhr, const double* A, const double* Cg, long long N, long long R, int K,
                         float* keys, cudaStream_t s);
void launch_mp_qboxes_fact(const unsigned int* perm, const double* Bhr, const double* A, const double* Cg, long long N,
                           long long R, int K, int ROWS, int QT, const unsigned int* qnmax, float* bmin, float* bmax,
                           cudaStream_t s);
// B[r][h] = E_h . Rel_r in FP64 (the pivot-independent part of the factorised keys)
void launch_mp_hr(const float* E, const float* Rel, long long N, long long R, int d, double* B, cudaStream_t s);
bool launch_mp_sort_small(const float* keys, const unsigned int* minmax, long long nseg, long long L, int K, int bits,
                          int* perm, cudaStream_t s);
void launch_mp_morton(const float* keys, const unsigned int* minmax, long long nseg, long long L, int K, int bits,
                      unsigned int* code, unsigned int* idx, cudaStream_t s);
void launch_kd_refine(const float* keys, int* perm, long long nseg, long long L, int K, cudaStream_t s);
void launch_mp_boxes(const float* keys, const unsigned int* perm, long long nseg, long long L, int ROWS, int ntile,
                     int K, float* bmin, float* bmax, const unsigned int* qnmax, cudaStream_t s, int transpose = 0);
// bits (optional, nq x ceil(TT / 32) words): mp_count stores each query tile's survival masks
// there and mp_emit expands them instead of repeating the box tests
void launch_mp_count(const float* qbmin, const float* qbmax, const float* tbmin, const float* tbmax, long long nq,
                     int TT, int K, float theta, float relm, int prune, int2* ranges, long long* cost, unsigned int* bits,
                     cudaStream_t s);
void launch_mp_emit(const float* qbmin, const float* qbmax, const float* tbmin, const float* tbmax,
                    const long long* cum, const DevCounters* ctr, long long nq, int TT, int K, float theta, float relm,
                    int prune, int* list, const unsigned int* bits, cudaStream_t s);

// ---- gathered-tail SIMT engine (pivots.cu): element-level tail pruning against query-tile boxes
constexpr int GT_ROWS = 64;  // tails per gathered block (= SIMT_T)
void launch_stage_rows(const float* E, const int* tperm, const float* keys, long long N, int d, int Kpad, int K,
                       float* Ts, float* tks, float4* tsc, cudaStream_t s);
// BN = 64 (SIMT engine) or 256 (tensor-core engine: also gT2 / gtst)
void launch_gather_tails(const float* qbmin, const float* qbmax, const float* tks, const int* list,
                         const long long* cum, const int2* ranges, DevCounters* ctr, long long N, int BN, int K,
                         float theta, float relm, int chunk, long long nq, long long* gblocks, int2* granges,
                         int* nitem, int* glist, const float4* tsc, float* gT2, float2* gtst, int cyc_world,
                         int cyc_rank, cudaStream_t s, int gb = 64);

// Tail tile of position j of item w (contiguous range or multi-pivot list).
__device__ __forceinline__ int item_tile(const int4& w, int j, const int* __restrict__ list) {
    return w.w < 0 ? j : __ldg(list + w.w + j);
}

// ---- tile engines ----
int  tc_smem_bytes(int Kpad, int* a_stages, int* b_stages, int* kc);
void launch_tiles_tc(const TileParams& p, int num_sms, cudaStream_t s);
void launch_tiles_tc_gather(const TileParams& p, int num_sms, cudaStream_t s);
void launch_tiles_tc_factored(const TileParams& p, int num_sms, cudaStream_t s);
void launch_factored_tables(const float* E, const float* Rel, const int* tperm, long long N, long long R, int d,
                            float theta, long long ntpad, float* fz, float* frt, float* frn, unsigned int* nonfinite,
                            cudaStream_t s);
void launch_iota(int* out, long long n, cudaStream_t s);
int  tc_gather_ok(int Kpad);  // the gathered tensor-core engine needs 32-wide K-chunks
int  tc2_smem_bytes(int Kpad, int* a_stages, int* b_stages, int* kc, int bnt = BN_TC);
void launch_tiles_tc2(const TileParams& p, int num_sms, cudaStream_t s);
int  tc2_gather_ok(int Kpad);  // the gathered CTA-pair engine needs 32-wide K-chunks
void launch_tiles_tc2_gather(const TileParams& p, int num_sms, cudaStream_t s);  // p.n_items: a bound
void launch_tiles_simt(const TileParams& p, int norm, int num_sms, cudaStream_t s);
void launch_tiles_gather(const TileParams& p, int norm, int num_sms, long long max_items, cudaStream_t s);
void launch_tiles_half_l1(const TileParams& p, int num_sms, cudaStream_t s);
constexpr int HALF_FLUSH_PAIRS = 8;  // FP16x2 engine: flush to FP32 every 16 dims

// ---- verification (verify.cu) ----
struct KgcTripletDev { int h, r, t; float dist; };
// SE (se.cu)
void launch_se_connectors(const float* E, const float* Wl, const float* Wr, long long N, int d, double* A64,
                          double* B64, float* Af, float* Bf, unsigned int* maxa, unsigned int* maxb, cudaStream_t s);
void launch_verify_se(const int2* cand, const unsigned long long* cand_count, long long cand_cap, const int* qperm,
                      const int* tperm, const double* A64, const double* B64, long long N, long long rows, int d,
                      float theta, KgcTripletDev* out, unsigned long long* res_count, long long res_cap, int num_sms,
                      cudaStream_t s, int r);
// top-k (topk.cu)
void launch_sample_dist(const float* E, const float* Rel, long long N, long long R, int d, int norm, int S,
                        int exclude_self, float* out, cudaStream_t s);
void launch_count_le(const float* a, long long n, float theta, unsigned long long* cnt, cudaStream_t s);
void launch_count_res_le(const KgcTripletDev* res, long long n, float theta, int exclude_self,
                         unsigned long long* cnt, cudaStream_t s);
void launch_compact_res_le(const KgcTripletDev* res, long long n, float theta, int exclude_self, KgcTripletDev* out,
                           unsigned long long* cnt, long long cap, cudaStream_t s);
void launch_l2_prefetch(const void* p, size_t bytes, int num_sms, cudaStream_t s);
// E: heads (row h of the query side), Et: tails (row t of the tail side, e.g. E + t_off d for a
// tail partition); records carry h + h_off, r + r_off, t + t_off.
void launch_verify(const int2* cand, const unsigned long long* cand_count, long long cand_cap,
                   const int* qperm, const int* tperm, const float* E, const float* Rel, const float* Et, long long N,
                   int QT, int bq, int d, int norm, float theta, KgcTripletDev* out, unsigned long long* res_count,
                   long long res_cap, int num_sms, cudaStream_t s, int r_off, long long Nt = -1, long long t_off = 0,
                   long long h_off = 0, const int* hmap = nullptr);
// spatial block-cyclic head split (split.cu, kgc_options.split = 3): Morton codes of the
// distances to 4 pivots P (4 x d) in code, entity ids in idx (sort them with
// radix_sort_u32_segments); then the owned chunks' head ids and rows (chunk c = k + W i of
// nch equal chunks)
void launch_sp_order(const float* E, long long N, int d, const float* P, float* keys, unsigned int* mm,
                     unsigned int* code, unsigned int* idx, cudaStream_t s);
void launch_sp_gather(const float* E, int d, const unsigned int* order, long long N, long long nch, long long W,
                      long long k, long long owned, long long max_len, int* hidx, float* Eh, cudaStream_t s);

}  // namespace kgc
