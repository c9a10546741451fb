// tiles_simt.cu -- K5: surviving-tile distance reduction on the FP32 SIMT
// pipes (SURVEY §8(a) row a6, and the L2 "SIMT" control engine).
//
// L1 (TransE ||h + r - t||_1) has no dense-contraction form, so
// it runs as register-tiled |q - t| accumulation: a 64-query x 64-tail tile
// per CTA (small tiles prune better), 64 threads, an 8 x 8 micro-tile per
// thread (FADD + FADD|.| per element and k).  Query and tail K-chunks stream
// through a double buffer fed by 1-D bulk TMA copies (full barriers with
// transaction counts; the last warp to release a stage refills it, so there is
// no CTA-wide barrier and no blocking producer in the main loop; shared memory
// independent of d, 7 CTAs per SM).  A pair whose FP32 distance is within the row's
// rigorous bound (stage kernel) becomes a
// candidate; the FP64 re-check (verify.cu) decides.
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"

namespace kgc {

constexpr int SIMT_KC = 32;

constexpr int SIMT_NS = 3;  // pipeline stages (query chunk + tail chunk each)

// Walks (work item, tail tile, K-chunk) in the order every thread of the CTA
// consumes them; the producer thread runs a second copy SIMT_NS - 1 chunks ahead.
struct ChunkIter {
    long long it, end, step;
    int4 w;
    int j, c;
    __device__ __forceinline__ bool valid(const TileParams&) const { return it < end; }
    __device__ __forceinline__ void start(const TileParams& p) {
        // this CTA's contiguous, cost-balanced block of work items
        if (p.sched) {
            it = balanced_begin(p.item_cum, p.n_items, p.total_tiles, blockIdx.x, gridDim.x);
            end = balanced_begin(p.item_cum, p.n_items, p.total_tiles, blockIdx.x + 1, gridDim.x);
            step = 1;
        } else {
            it = blockIdx.x;
            end = p.n_items;
            step = gridDim.x;
        }
        if (it < end) {
            w = p.items[it];
            j = w.y;
        }
        c = 0;
    }
    __device__ __forceinline__ void next(const TileParams& p, int nkc) {
        if (++c < nkc) return;
        c = 0;
        if (++j <= w.z) return;
        if ((it += step) < end) {
            w = p.items[it];
            j = w.y;
        }
    }
};

// TBM x TBN tile, 256 threads in a (TBM/TM) x (TBN/TN) grid, TM x TN register
// micro-tile per thread.
template <int NORM, int TBM, int TBN, int TM, int TN, int KC = SIMT_KC, int NSTAGE = SIMT_NS>
__global__ void __launch_bounds__((TBM / TM) * (TBN / TN)) tiles_simt_kernel(TileParams p) {
    constexpr int NT = (TBM / TM) * (TBN / TN);
    static_assert(NT % 32 == 0 && NT <= 256 && TM * TN <= 64, "tile shape");
    constexpr int SIMT_KC = KC;
    constexpr int SIMT_NS = NSTAGE;
    constexpr int GX = TBN / TN;  // threads along the tail dimension
    extern __shared__ __align__(128) uint8_t smem[];
    const int Kpad = p.Kpad;
    const int nkc = (Kpad + SIMT_KC - 1) / SIMT_KC;
    // stage s: query chunk [SIMT_KC][TBM] followed by tail chunk [SIMT_KC][TBN]
    float* St = reinterpret_cast<float*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(St + SIMT_NS * SIMT_KC * (TBM + TBN));
    int* released = reinterpret_cast<int*>(full + SIMT_NS);  // warps done with each stage

    const int tid = threadIdx.x, lane = tid & 31;
    const int ty = tid / GX, tx = tid % GX;
    if (tid == 0) {
        for (int s = 0; s < SIMT_NS; ++s) {
            mbar_init(&full[s], 1);
            released[s] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();

    // Called by one thread once stage (g % SIMT_NS) is free.
    auto issue = [&](const ChunkIter& ci, long long g) {
        const int s = (int)(g % SIMT_NS);
        const int klen = Kpad - ci.c * SIMT_KC < SIMT_KC ? Kpad - ci.c * SIMT_KC : SIMT_KC;
        const uint32_t qbytes = (uint32_t)klen * TBM * 4, tbytes = (uint32_t)klen * TBN * 4;
        float* dst = St + (size_t)s * SIMT_KC * (TBM + TBN);
        mbar_arrive_expect_tx(&full[s], qbytes + tbytes);
        bulk_g2s(dst, p.Qp + (size_t)(ci.w.x - p.tq0) * TBM * Kpad + (size_t)ci.c * SIMT_KC * TBM, qbytes, &full[s]);
        bulk_g2s(dst + SIMT_KC * TBM,
                 p.Tp + (size_t)item_tile(ci.w, ci.j, p.tile_list) * TBN * Kpad + (size_t)ci.c * SIMT_KC * TBN, tbytes,
                 &full[s]);
    };

    ChunkIter cs;  // the chunk sequence every thread consumes
    cs.start(p);
    if (tid == 0) {  // prologue: fill every stage
        ChunkIter pr = cs;
        for (long long gp = 0; gp < SIMT_NS && pr.valid(p); ++gp) {
            issue(pr, gp);
            pr.next(p, nkc);
        }
    }

    float thr[TM];
    float acc[TM][TN];
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) acc[a][b] = 0.f;
    long long cur_item = -1;

    for (long long g = 0; cs.valid(p); ++g) {
        if (cs.it != cur_item) {
            cur_item = cs.it;
#pragma unroll
            for (int a = 0; a < TM; ++a) thr[a] = p.qs[(size_t)(cs.w.x - p.tq0) * TBM + ty * TM + a].w;
        }
        const int s = (int)(g % SIMT_NS);
        mbar_wait(&full[s], (uint32_t)(g / SIMT_NS) & 1u);
        const int klen = Kpad - cs.c * SIMT_KC < SIMT_KC ? Kpad - cs.c * SIMT_KC : SIMT_KC;
        const float* qk = St + (size_t)s * SIMT_KC * (TBM + TBN) + ty * TM;
        const float* tk = St + (size_t)s * SIMT_KC * (TBM + TBN) + SIMT_KC * TBM + tx * TN;
#pragma unroll 4
        for (int k = 0; k < klen; ++k) {
            float qv[TM], tv[TN];
#pragma unroll
            for (int a = 0; a < TM; a += 4) {
                const float4 v = *reinterpret_cast<const float4*>(qk + k * TBM + a);
                qv[a] = v.x; qv[a + 1] = v.y; qv[a + 2] = v.z; qv[a + 3] = v.w;
            }
#pragma unroll
            for (int b = 0; b < TN; b += 4) {
                const float4 v = *reinterpret_cast<const float4*>(tk + k * TBN + b);
                tv[b] = v.x; tv[b + 1] = v.y; tv[b + 2] = v.z; tv[b + 3] = v.w;
            }
#pragma unroll
            for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TN; ++b) {
                    const float df = qv[a] - tv[b];
                    if (NORM == 1) acc[a][b] += fabsf(df);
                    else acc[a][b] = fmaf(df, df, acc[a][b]);
                }
        }
        // The last warp to finish reading stage s refills it with chunk g + SIMT_NS:
        // no thread ever blocks waiting for the slowest warp.
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&released[s], 1) == NT / 32 - 1) {
                released[s] = 0;
                ChunkIter nx = cs;
#pragma unroll 1
                for (int x = 0; x < SIMT_NS && nx.valid(p); ++x) nx.next(p, nkc);
                if (nx.valid(p)) {
                    fence_proxy_async_smem();
                    issue(nx, g + SIMT_NS);
                }
            }
        }
        if (cs.c == nkc - 1) {
            const int j = item_tile(cs.w, cs.j, p.tile_list);
            unsigned long long hit = 0;
#pragma unroll
            for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TN; ++b) hit |= (unsigned long long)(acc[a][b] <= thr[a]) << (a * TN + b);
            if (__any_sync(0xffffffffu, hit != 0)) {
                // columns past the last tail are padding
                const int colb = j * TBN + tx * TN;
#pragma unroll
                for (int b = 0; b < TN; ++b)
                    if (colb + b >= p.Nt)
#pragma unroll
                        for (int a = 0; a < TM; ++a) hit &= ~(1ull << (a * TN + b));
                unsigned long long slot = warp_reserve(__popcll(hit), p.cand_count);
                while (hit) {
                    const int ab = __ffsll(hit) - 1;
                    if (slot < (unsigned long long)p.cand_cap)
                        p.cand[slot] = make_int2(cs.w.x * TBM + ty * TM + ab / TN, colb + ab % TN);
                    ++slot;
                    hit &= hit - 1;
                }
            }
#pragma unroll
            for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TN; ++b) acc[a][b] = 0.f;
        }
        cs.next(p, nkc);
    }
}

// ------------------------------------------------------------------------
// FP16x2 L1 engine.  Same tiling, ring and scheduling as above, operands are
// half2 words (two consecutive dims) and the inner step is
//     acc2 = acc2 + |q2 - t2|      (HADD2 with the |.| operand modifier:
// one instruction per element instead of FADD + FADD|.|), flushed into FP32
// every HALF_FLUSH_PAIRS pairs (16 dims).  A pair is a candidate iff the FP32
// sum <= thr_row + rt_col, the rigorous bound of DESIGN.md "FP16x2 L1 engine";
// the FP64 re-check decides.
constexpr int HKC = 16;  // pairs (= 32 dims) per stage

__global__ void __launch_bounds__(256, 1) tiles_half_l1_kernel(TileParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int KP = p.Kpad / 2;                         // pairs per row
    const int nkc = (KP + HKC - 1) / HKC;
    uint32_t* St = reinterpret_cast<uint32_t*>(smem);  // [stage][HKC][BM + BN] half2 words
    uint64_t* full = reinterpret_cast<uint64_t*>(St + SIMT_NS * HKC * (BN_HALF + BN_HALF));
    int* released = reinterpret_cast<int*>(full + SIMT_NS);

    const int tid = threadIdx.x, lane = tid & 31;
    const int ty = tid >> 4, tx = tid & 15;
    if (tid == 0) {
        for (int s = 0; s < SIMT_NS; ++s) {
            mbar_init(&full[s], 1);
            released[s] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t* Qw = reinterpret_cast<const uint32_t*>(p.Qp);
    const uint32_t* Tw = reinterpret_cast<const uint32_t*>(p.Tp);
    auto issue = [&](const ChunkIter& ci, long long g) {
        const int s = (int)(g % SIMT_NS);
        const int klen = KP - ci.c * HKC < HKC ? KP - ci.c * HKC : HKC;
        const uint32_t qbytes = (uint32_t)klen * BN_HALF * 4, tbytes = (uint32_t)klen * BN_HALF * 4;
        uint32_t* dst = St + (size_t)s * HKC * (BN_HALF + BN_HALF);
        mbar_arrive_expect_tx(&full[s], qbytes + tbytes);
        bulk_g2s(dst, Qw + (size_t)(ci.w.x - p.tq0) * BN_HALF * KP + (size_t)ci.c * HKC * BN_HALF, qbytes, &full[s]);
        bulk_g2s(dst + HKC * BN_HALF, Tw + (size_t)item_tile(ci.w, ci.j, p.tile_list) * BN_HALF * KP + (size_t)ci.c * HKC * BN_HALF,
                 tbytes, &full[s]);
    };

    ChunkIter cs;
    cs.start(p);
    if (tid == 0) {
        ChunkIter pr = cs;
        for (long long gp = 0; gp < SIMT_NS && pr.valid(p); ++gp) {
            issue(pr, gp);
            pr.next(p, nkc);
        }
    }

    float thr[8];
    float accf[8][8];
    __half2 acc2[8][8];
    const __half2 hz = __float2half2_rn(0.f);
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) { accf[a][b] = 0.f; acc2[a][b] = hz; }
    long long cur_item = -1;

    auto flush = [&]() {
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const float2 f = __half22float2(acc2[a][b]);
                accf[a][b] += f.x + f.y;
                acc2[a][b] = hz;
            }
    };

    for (long long g = 0; cs.valid(p); ++g) {
        if (cs.it != cur_item) {
            cur_item = cs.it;
#pragma unroll
            for (int a = 0; a < 8; ++a) thr[a] = p.qs[(size_t)(cs.w.x - p.tq0) * BN_HALF + ty * 8 + a].w;
        }
        const int s = (int)(g % SIMT_NS);
        mbar_wait(&full[s], (uint32_t)(g / SIMT_NS) & 1u);
        const int klen = KP - cs.c * HKC < HKC ? KP - cs.c * HKC : HKC;
        const uint32_t* qk = St + (size_t)s * HKC * (BN_HALF + BN_HALF) + ty * 8;
        const uint32_t* tk = St + (size_t)s * HKC * (BN_HALF + BN_HALF) + HKC * BN_HALF + tx * 8;
        for (int k0 = 0; k0 < klen; k0 += HALF_FLUSH_PAIRS) {
            const int kend = k0 + HALF_FLUSH_PAIRS < klen ? k0 + HALF_FLUSH_PAIRS : klen;
#pragma unroll 2
            for (int k = k0; k < kend; ++k) {
                const uint4 qa = *reinterpret_cast<const uint4*>(qk + k * BN_HALF);
                const uint4 qb = *reinterpret_cast<const uint4*>(qk + k * BN_HALF + 4);
                const uint4 ta = *reinterpret_cast<const uint4*>(tk + k * BN_HALF);
                const uint4 tb = *reinterpret_cast<const uint4*>(tk + k * BN_HALF + 4);
                const uint32_t qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
                const uint32_t tv[8] = {ta.x, ta.y, ta.z, ta.w, tb.x, tb.y, tb.z, tb.w};
#pragma unroll
                for (int a = 0; a < 8; ++a) {
                    const __half2 q2 = *reinterpret_cast<const __half2*>(&qv[a]);
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const __half2 t2 = *reinterpret_cast<const __half2*>(&tv[b]);
                        acc2[a][b] = __hadd2(acc2[a][b], __habs2(__hsub2(q2, t2)));
                    }
                }
            }
            flush();
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&released[s], 1) == 7) {
                released[s] = 0;
                ChunkIter nx = cs;
#pragma unroll 1
                for (int x = 0; x < SIMT_NS && nx.valid(p); ++x) nx.next(p, nkc);
                if (nx.valid(p)) {
                    fence_proxy_async_smem();
                    issue(nx, g + SIMT_NS);
                }
            }
        }
        if (cs.c == nkc - 1) {
            const int j = item_tile(cs.w, cs.j, p.tile_list);
            const int colb = j * BN_HALF + tx * 8;
            const float4 r0 = __ldg(reinterpret_cast<const float4*>(p.Rt + colb));
            const float4 r1 = __ldg(reinterpret_cast<const float4*>(p.Rt + colb + 4));
            const float rtc[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
            unsigned long long hit = 0;
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int b = 0; b < 8; ++b)
                    hit |= (unsigned long long)(accf[a][b] <= __fadd_ru(thr[a], rtc[b])) << (a * 8 + b);
            if (__any_sync(0xffffffffu, hit != 0)) {
#pragma unroll
                for (int b = 0; b < 8; ++b)
                    if (colb + b >= p.Nt) hit &= ~(0x0101010101010101ull << b);
                unsigned long long slot = warp_reserve(__popcll(hit), p.cand_count);
                while (hit) {
                    const int ab = __ffsll(hit) - 1;
                    if (slot < (unsigned long long)p.cand_cap)
                        p.cand[slot] = make_int2(cs.w.x * BN_HALF + ty * 8 + (ab >> 3), colb + (ab & 7));
                    ++slot;
                    hit &= hit - 1;
                }
            }
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int b = 0; b < 8; ++b) accf[a][b] = 0.f;
        }
        cs.next(p, nkc);
    }
}

void launch_tiles_half_l1(const TileParams& p, int num_sms, cudaStream_t s) {
    if (p.n_items <= 0) return;
    const size_t smem = (size_t)SIMT_NS * HKC * (BN_HALF + BN_HALF) * 4 + 64;
    cudaFuncSetAttribute(tiles_half_l1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tiles_half_l1_kernel, 256, smem);
    if (per_sm < 1) per_sm = 1;
    long long g = (long long)num_sms * per_sm;
    if (g > p.n_items) g = p.n_items;
    tiles_half_l1_kernel<<<(unsigned)g, 256, smem, s>>>(p);
}

template <int NORM, int TM, int TN, int KC, int NS = SIMT_NS, int T = SIMT_T>
static void launch_simt_variant(const TileParams& p, int num_sms, cudaStream_t s) {
    constexpr int NT = (T / TM) * (T / TN);
    const size_t smem = (size_t)NS * KC * (T + T) * 4 + 128;
    auto kern = tiles_simt_kernel<NORM, T, T, TM, TN, KC, NS>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
    if (per_sm < 1) per_sm = 1;
    long long g = (long long)num_sms * per_sm;
    if (g > p.n_items) g = p.n_items;
    kern<<<(unsigned)g, NT, smem, s>>>(p);
}

void launch_tiles_simt(const TileParams& p, int norm, int num_sms, cudaStream_t s) {
    if (p.n_items <= 0) return;
    // 64 x 64 tiles, 64 threads with 8 x 8 micro-tiles, 32-wide K-chunks, double buffer:
    // 32 KB of shared memory -> 7 CTAs per SM (register-limited).  Measured best of the
    // micro-tile / chunk / depth sweep on c2 L1.
    if (p.bq == 32) {  // 32 x 32 tiles (experiment: finer pruning), 64 threads with 4 x 4 micro-tiles
        if (norm == 1) launch_simt_variant<1, 4, 4, 32, 2, 32>(p, num_sms, s);
        else launch_simt_variant<2, 4, 4, 32, 2, 32>(p, num_sms, s);
        return;
    }
    if (norm == 1) launch_simt_variant<1, 8, 8, 32, 2>(p, num_sms, s);
    else launch_simt_variant<2, 8, 8, 32, 2>(p, num_sms, s);
}


// ------------------------------------------------------------------------
// Gathered-tail variant (l1_engine 3): the 64 tails of a block are not a
// contiguous tile but the next 64 entries of the query tile's list of
// surviving tails (pivots.cu, gather_tails_kernel), so the arithmetic skips
// every tail that fails the K-pivot test against the query tile's box.
// Per stage: the query K-chunk by one bulk copy (as above), the 64 tail rows'
// K-chunk gathered row-major by 16-byte cp.async pieces that arrive on the
// stage's mbarrier (cp.async.mbarrier.arrive.noinc), issued by the 32 lanes of
// the refilling warp.  K-chunks are balanced (a short last chunk left the next
// block's first refill exposed).  Refill duty alternates between the two warps
// by chunk parity, gated by an "empty" mbarrier the other warp arrives on.
// Thread tx owns tail rows tx, tx + 8, ..., tx + 56; its float4 row reads are
// conflict-free with a padded row stride KC + 4 (SWZ = 0) or with 16-byte
// piece p of row i stored at piece p ^ (i & 7) of a 32-float row (SWZ = 1).
// PROF = 1: clock64 wait instrumentation (KGC_GT_PROF=1, experiment only).
// TB = tails per block: 64 (two warps sharing the stages) or 32 (one warp per CTA:
// no lock-step between warps, half the padding; the query chunk is shared by 32 tails).
template <int NORM, int KC, int NSTAGE, int SWZ, int PROF = 0, int DUTY = 1, int MINB = 8, int KUN = 1, int TB = 64>
__global__ void __launch_bounds__(TB, MINB) tiles_gather_kernel(TileParams p) {
    constexpr int T = SIMT_T, TM = 8, TN = 8, NT = TB, GX = TB / TN, NWARP = TB / 32;
    static_assert(!SWZ || KC == 32, "swizzle over the 8 pieces of a 32-float row");
    static_assert(TB == 32 || TB == 64, "one or two warps");
    constexpr int LD = SWZ ? KC : KC + 4;  // tail row stride in shared memory (floats)
    constexpr int BPT = SIMT_T / TB;       // blocks per tile-list slot (list offsets are in 64-tail tiles)
    extern __shared__ __align__(128) uint8_t smem[];
    const int Kpad = p.Kpad;
    const int nkc = (Kpad + KC - 1) / KC;
    // balanced K-chunks (multiples of 4 floats, sizes differ by at most 4): a short last
    // chunk would leave too little compute to hide the next block's first refill
    const int cu = (Kpad / 4) / nkc, cr = (Kpad / 4) % nkc;
    auto chunk_k0 = [&](int c) { return 4 * (c * cu + (c < cr ? c : cr)); };
    auto chunk_len = [&](int c) { return 4 * (cu + (c < cr ? 1 : 0)); };
    // stage s: query chunk [KC][T] followed by tail rows [TB][LD]
    constexpr int STAGE = KC * T + TB * LD;
    float* St = reinterpret_cast<float*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(St + NSTAGE * STAGE);
    uint64_t* empty = full + NSTAGE;  // the non-duty warp has finished reading the stage
    int* released = reinterpret_cast<int*>(empty + NSTAGE);
    int* ridx = released + NSTAGE;  // [TB] row indices of the block being issued
    __shared__ long long issued_at[PROF ? NSTAGE : 1];

    const int tid = threadIdx.x, lane = tid & 31;
    const int ty = tid / GX, tx = tid % GX;
    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(&full[s], 1 + 32);  // the bulk copy's expect_tx arrival + 32 lanes' cp.async arrivals
            mbar_init(&empty[s], 1);
            released[s] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();
    const long long n_items = *p.dn_items, total = *p.dtotal;

    struct It {
        long long it, end;
        int4 w;
        int j, c;
    };
    auto valid = [&](const It& ci) { return ci.it < ci.end; };
    auto next = [&](It& ci) {
        if (++ci.c < nkc) return;
        ci.c = 0;
        if (++ci.j <= ci.w.z) return;
        if (++ci.it < ci.end) {
            ci.w = p.items[ci.it];
            ci.j = ci.w.y;
        }
    };
    // Called by all 32 lanes of one warp once stage (g % NSTAGE) is free: the query
    // chunk by one bulk copy (transaction bytes), the 64 gathered tail rows by 16-byte
    // cp.async pieces (8 consecutive lanes per 128-byte row chunk), each lane's pieces
    // arriving on the stage barrier through cp.async.mbarrier.arrive.noinc (barrier
    // count 1 + 32).  Row indices: lane l loads those of rows l and l + 32 once, the
    // pieces take them by shuffle.
    auto issue = [&](const It& ci, long long g) {
        const int s = (int)(g % NSTAGE);
        const int klen = chunk_len(ci.c), k0 = chunk_k0(ci.c);
        const uint32_t qbytes = (uint32_t)klen * T * 4;
        float* dst = St + (size_t)s * STAGE;
        // the block's row indices: from global memory at its first chunk (kept in shared
        // memory for the others -- issues are serialised, see the release protocol below)
        int r0, r1 = 0;
        if (ci.c == 0) {
            const int* seg = p.glist + ((long long)ci.w.w * BPT + ci.j) * TB;
            r0 = __ldg(seg + lane);
            if (TB == 64) r1 = __ldg(seg + lane + 32);
            if (lane < TB / 32) prefetch_l1(seg + TB + lane * 32);  // the next block's indices
            if (nkc > 1) {
                ridx[lane] = r0;
                if (TB == 64) ridx[lane + 32] = r1;
            }
        } else {
            r0 = ridx[lane];
            if (TB == 64) r1 = ridx[lane + 32];
        }
        if (lane == 0) {
            mbar_arrive_expect_tx(&full[s], qbytes);
            bulk_g2s(dst, p.Qp + (size_t)(ci.w.x - p.tq0) * T * Kpad + (size_t)k0 * T, qbytes, &full[s]);
        }
        const uint32_t tdst = smem_u32(dst + KC * T);
        const float* src0 = p.Ts + k0;
        auto piece = [&](int row, int pseg, int ridx) {
            const int slot = SWZ ? (pseg ^ (row & 7)) : pseg;
            cp_async16(tdst + (uint32_t)(row * LD + slot * 4) * 4u, src0 + (size_t)ridx * Kpad + pseg * 4);
        };
        {
            // rpp rows per pass over rpp * per_row lanes (two divisions per issue)
            const int per_row = klen / 4, rpp = 32 / per_row;
            const int prow = lane / per_row, pseg = lane - prow * per_row;
            const bool act = lane < rpp * per_row;
#pragma unroll 2
            for (int row0 = 0; row0 < TB; row0 += rpp) {
                const int row = row0 + prow;
                const int a0 = __shfl_sync(0xffffffffu, r0, row & 31);
                const int a1 = TB == 64 ? __shfl_sync(0xffffffffu, r1, row & 31) : 0;
                if (act && row < TB) piece(row, pseg, row < 32 ? a0 : a1);
            }
        }
        cp_async_mbar_arrive_noinc(&full[s]);
        if (PROF && lane == 0) issued_at[s] = clock64();
    };

    It cs;  // the chunk sequence every thread consumes: this CTA's cost-balanced block of items
    cs.it = balanced_begin(p.item_cum, n_items, total, blockIdx.x, gridDim.x);
    cs.end = balanced_begin(p.item_cum, n_items, total, blockIdx.x + 1, gridDim.x);
    cs.c = 0;
    if (cs.it < cs.end) {
        cs.w = p.items[cs.it];
        cs.j = cs.w.y;
    }
    if (tid < 32) {  // prologue: warp 0 fills every stage
        It pr = cs;
        for (long long gp = 0; gp < NSTAGE && valid(pr); ++gp) {
            issue(pr, gp);
            next(pr);
        }
    }

    float thr[TM];
    float acc[TM][TN];
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) acc[a][b] = 0.f;
    long long cur_item = -1;
    const long long tstart = PROF ? clock64() : 0;

    for (long long g = 0; valid(cs); ++g) {
        if (cs.it != cur_item) {
            cur_item = cs.it;
#pragma unroll
            for (int a = 0; a < TM; ++a) thr[a] = p.qs[(size_t)(cs.w.x - p.tq0) * T + ty * TM + a].w;
        }
        const int s = (int)(g % NSTAGE);
        if (PROF) {  // wait-time instrumentation (KGC_GT_PROF=1): by chunk kind
            const long long t0 = clock64();
            mbar_wait(&full[s], (uint32_t)(g / NSTAGE) & 1u);
            const long long t1 = clock64(), dt = t1 - t0;
            const int kind = cs.c != 0 ? 2 : (cs.j == cs.w.y ? 0 : 1);  // item start / block start / other
            if (lane == 0) {
                atomicAdd(p.prof + 2 * kind, (unsigned long long)dt);
                atomicAdd(p.prof + 2 * kind + 1, 1ull);
                if (g >= NSTAGE && dt > 200) {  // waited: issue -> ready latency
                    atomicAdd(p.prof + 8, (unsigned long long)(t1 - issued_at[s]));
                    atomicAdd(p.prof + 9, 1ull);
                }
            }
        } else {
            mbar_wait(&full[s], (uint32_t)(g / NSTAGE) & 1u);
        }
        const int klen = chunk_len(cs.c);
        const float* qk = St + (size_t)s * STAGE + ty * TM;
        const float* tk = St + (size_t)s * STAGE + KC * T + tx * LD;
#pragma unroll KUN
        for (int k4 = 0; k4 < klen; k4 += 4) {
            float4 tv[TN];
#pragma unroll
            for (int b = 0; b < TN; ++b)
                tv[b] = *reinterpret_cast<const float4*>(tk + b * GX * LD + (SWZ ? (((k4 >> 2) ^ tx) << 2) : k4));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                float qv[TM];
#pragma unroll
                for (int a = 0; a < TM; a += 4) {
                    const float4 v = *reinterpret_cast<const float4*>(qk + (k4 + kk) * T + a);
                    qv[a] = v.x; qv[a + 1] = v.y; qv[a + 2] = v.z; qv[a + 3] = v.w;
                }
#pragma unroll
                for (int a = 0; a < TM; ++a)
#pragma unroll
                    for (int b = 0; b < TN; ++b) {
                        const float t = kk == 0 ? tv[b].x : kk == 1 ? tv[b].y : kk == 2 ? tv[b].z : tv[b].w;
                        const float df = qv[a] - t;
                        if (NORM == 1) acc[a][b] += fabsf(df);
                        else acc[a][b] = fmaf(df, df, acc[a][b]);
                    }
            }
        }
        // Refill duty alternates with the chunk: warp (g & 1) refills stage s with chunk
        // g + NSTAGE once the other warp has released it (empty[s]); the other warp just
        // releases.  (A fixed "last releaser refills" rule made the refilling warp the
        // slower one for good, and its partner then waited on every chunk.)
        __syncwarp();
        int last = 0;
        if (NWARP == 1) {
            last = 1;  // the only reader refills its own stage
        } else if (DUTY) {
            const int warp = tid >> 5;
            if (warp == (int)(g & 1)) {
                mbar_wait(&empty[s], (uint32_t)(g / NSTAGE) & 1u);
                last = 1;
            } else if (lane == 0) {
                mbar_arrive(&empty[s]);
            }
        } else {
            if (lane == 0) {
                __threadfence_block();
                last = atomicAdd(&released[s], 1) == NT / 32 - 1;
                if (last) released[s] = 0;
            }
            last = __shfl_sync(0xffffffffu, last, 0);
        }
        if (last) {
            It nx = cs;
#pragma unroll 1
            for (int x = 0; x < NSTAGE && valid(nx); ++x) next(nx);
            if (valid(nx)) {
                fence_proxy_async_smem();
                issue(nx, g + NSTAGE);
            }
        }
        if (cs.c == nkc - 1) {
            unsigned long long hit = 0;
#pragma unroll
            for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TN; ++b) hit |= (unsigned long long)(acc[a][b] <= thr[a]) << (a * TN + b);
            if (__any_sync(0xffffffffu, hit != 0)) {
                const int* seg = p.glist + ((long long)cs.w.w * BPT + cs.j) * TB + tx;
#pragma unroll
                for (int b = 0; b < TN; ++b) {
                    const unsigned long long colm = 0x0101010101010101ull << b;  // column b of the micro-tile
                    if ((hit & colm) && __ldg(seg + b * GX) >= p.Nt) hit &= ~colm;  // sentinel padding
                }
                unsigned long long slot = warp_reserve(__popcll(hit), p.cand_count);
                while (hit) {
                    const int ab = __ffsll(hit) - 1;
                    if (slot < (unsigned long long)p.cand_cap)
                        p.cand[slot] = make_int2(cs.w.x * T + ty * TM + ab / TN, __ldg(seg + (ab % TN) * GX));
                    ++slot;
                    hit &= hit - 1;
                }
            }
#pragma unroll
            for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TN; ++b) acc[a][b] = 0.f;
        }
        next(cs);
    }
    if (PROF && lane == 0) {
        atomicAdd(p.prof + 6, (unsigned long long)(clock64() - tstart));
        atomicAdd(p.prof + 7, 1ull);
    }
}

template <int NORM, int KC, int NS, int SWZ = 0, int DUTY = 1, int MINB = 8, int KUN = 1, int TB = 64>
static void launch_gather_variant(const TileParams& p, int num_sms, long long max_items, cudaStream_t s) {
    constexpr int T = SIMT_T;
    const size_t smem = (size_t)NS * (KC * T + TB * (SWZ ? KC : KC + 4)) * 4 + 128 + TB * 4;
    static_assert(NS * 20 <= 128, "barriers and counters fit the 128-byte tail");
    auto kern = p.prof ? tiles_gather_kernel<NORM, KC, NS, SWZ, 1, DUTY, MINB, KUN, TB>
                       : tiles_gather_kernel<NORM, KC, NS, SWZ, 0, DUTY, MINB, KUN, TB>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TB, smem);
    if (per_sm < 1) per_sm = 1;
    long long g = (long long)num_sms * per_sm;
    if (g > max_items) g = max_items;
    if (g < 1) g = 1;
    kern<<<(unsigned)g, TB, smem, s>>>(p);
}

void launch_tiles_gather(const TileParams& p, int norm, int num_sms, long long max_items, cudaStream_t s) {
    if (max_items <= 0) return;
    const char* e = kgc_knob("KGC_GT_VAR");  // experiment knob: chunk / stage / refill-protocol variants
    const int v = e ? atoi(e) : 0;
    // measured on c2 L1 (tile-kernel ms, same session): KC 24 / 2 stages / alternating refill duty
    // 4.83; KC 32 4.93-5.07; KC 16 4.95; KC 24 with "last releaser refills" 4.93; KC 32 swizzled
    // 4.90; 3 stages 4.98-5.54; k-loop unrolled x2 at 6 CTAs/SM 4.99
    if (p.gb == 32) {  // one warp per CTA, 32-tail blocks
        if (norm == 1) {
            if (v == 1) launch_gather_variant<1, 32, 2, 0, 1, 8, 1, 32>(p, num_sms, max_items, s);
            else if (v == 2) launch_gather_variant<1, 24, 3, 0, 1, 8, 1, 32>(p, num_sms, max_items, s);
            else launch_gather_variant<1, 24, 2, 0, 1, 8, 1, 32>(p, num_sms, max_items, s);
        } else {
            launch_gather_variant<2, 24, 2, 0, 1, 8, 1, 32>(p, num_sms, max_items, s);
        }
        return;
    }
    if (norm == 1) {
        if (v == 1) launch_gather_variant<1, 32, 2>(p, num_sms, max_items, s);
        else if (v == 2) launch_gather_variant<1, 16, 2>(p, num_sms, max_items, s);
        else if (v == 3) launch_gather_variant<1, 32, 2, 1>(p, num_sms, max_items, s);
        else if (v == 4) launch_gather_variant<1, 24, 2, 0, 0>(p, num_sms, max_items, s);
        else launch_gather_variant<1, 24, 2>(p, num_sms, max_items, s);
    } else {
        launch_gather_variant<2, 24, 2>(p, num_sms, max_items, s);
    }
}

}  // namespace kgc
