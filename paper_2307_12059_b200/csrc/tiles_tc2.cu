// tiles_tc2.cu -- K4 on CTA pairs: the L2 surviving-tile contraction with
// tcgen05.mma.cta_group::2 (the M = 256 form of
// tiles_tc.cu).
//
// Same arithmetic and guard band as tiles_tc.cu (D^2 = ||q||^2 + ||t||^2 -
// 2 q.t; TF32 band + FP64 re-check keep the filter lossless,
// PAPER.md:349-351).  What changes is the data movement: a cluster of two
// CTAs on two SMs works on one 256-row query tile (128 rows per CTA, built
// in each CTA's shared memory) against the same 256-row tail tiles, and
// each CTA streams only HALF of every tail tile (its 128 rows; the tails
// are staged as two 128-row UMMA blocks per tile).  The even CTA issues
// M = 256, N = 256, K = 8 MMAs that read A and B from both CTAs' shared
// memory; each CTA's TMEM receives its own 128 x 256 accumulator.  Per SM,
// tail bytes per MAC halve relative to tiles_tc.cu -- the B-operand wait
// that bounds the 1-CTA kernel on large N.
//
// Cross-CTA signalling (all mbarriers live at the same offsets in both CTAs):
//   a_full   (even CTA: 256 arrivals) builders of both CTAs; odd-CTA
//            builders arrive remotely (release.cluster) after their
//            proxy fence.
//   b_full   (even CTA: 2 arrivals) its producer's expect_tx + a relay
//            thread of the odd CTA that waits for the odd CTA's own bulk
//            copy and forwards the completion (1-D bulk copies complete
//            only on a barrier of the destination CTA).
//   b_empty, a_empty, acc_full: tcgen05.commit multicast to both CTAs.
//   acc_empty (even CTA: 16 arrivals) the 8 epilogue warps of each CTA.
//
// GATHER (l2_engine 6): the tail operand is not a contiguous tail tile but a block
// of 256 gathered tails -- the tails of the query tile's surviving tiles whose own
// K pivot keys pass the L_inf test against the query tile's key box (Lemma 1 per
// tail, pivots.cu gather_tails_kernel<256>), at 3-4x fewer pairs than whole tiles.
// The producer WARP of each CTA gathers its 128 rows of the block with 16-byte
// cp.async pieces straight into a 128-byte-swizzled K-major operand (8 lanes per
// 128-byte row chunk: 4 rows = 512 contiguous bytes per instruction, the block's
// row indices in registers), keeps up to 3 chunks in flight, and signals a chunk after
// cp.async.wait_group + fence.proxy.async (generic-proxy writes made visible to
// tcgen05.mma).  The epilogue takes ||t||^2 / 2 per list entry and the block's
// guard-band maxima from the list build, and emits the list entry (sorted tail
// position) as the candidate column.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_build.cuh"

namespace kgc {

#ifdef KGC_PROF_TC
// debug build only: cycles each role spends blocked in each barrier wait
__device__ unsigned long long g_tc2_prof[16];
#define TC2_WAIT(slot, bar, par)                                   \
    do {                                                           \
        const long long t0_ = clock64();                           \
        mbar_wait(bar, par);                                       \
        atomicAdd(&g_tc2_prof[slot], (unsigned long long)(clock64() - t0_)); \
    } while (0)
#else
#define TC2_WAIT(slot, bar, par) mbar_wait(bar, par)
#endif

constexpr int TC2_THREADS = 448;  // same roles as tiles_tc.cu
constexpr int TC2_BUILDER_WARP0 = 10;
constexpr uint32_t LBO_A2 = (BM / 8) * 128;     // 128 query rows per CTA
constexpr int TC2_T2S_BYTES = 8 * 128 * 4;      // per epilogue warp: ||t||^2 / 2 of its 128 columns
constexpr uint32_t SBO2 = 128;
// tail tiles of BNT rows (256, or 128: finer tail tiles prune better, same B bytes per MAC);
// each CTA streams HALFT = BNT / 2 of them

int tc2_smem_bytes(int Kpad, int* a_stages, int* b_stages, int* kc, int bnt) {
    (void)bnt;  // 128-row tiles are streamed whole by one CTA: the same 128 rows per CTA and stage
    const int HALF = 128;
    const int budget = 227 * 1024 - 512 - 2 * BM * 16 - TC2_T2S_BYTES;
    const int A = BM * Kpad * 4;
    // prefer two A stages when the B ring still buffers >= 64 K-values
    // (experiment knob KGC_TC2_MINK: the minimum ring depth in K-values for two A stages)
    const char* e = kgc_knob("KGC_TC2_MINK");
    const int mink = e ? atoi(e) : 64;
    for (int as = 2; as >= 1; --as) {
        for (int KC : {32, 16, 8}) {
            const int B = HALF * KC * 4;
            const int rem = budget - as * A;
            if (rem <= 0) continue;
            int bs = rem / B;
            if (bs > 6) bs = 6;
            if (bs >= 2 && (bs * KC >= mink || as == 1)) {
                *a_stages = as;
                *b_stages = bs;
                *kc = KC;
                const int bytes = as * A + bs * B + 512 + as * BM * 16 + TC2_T2S_BYTES;
                return bytes < 117 * 1024 ? 117 * 1024 : bytes;  // one CTA per SM
            }
        }
    }
    return -1;
}

template <bool GATHER, int BNT>
__global__ void __launch_bounds__(TC2_THREADS, 1) tiles_tc2_kernel(TileParams p, int a_stages, int b_stages, int KC) {
    static_assert(!GATHER || BNT == BN_TC, "gathered blocks are 256 tails");
    // BNT = tail-tile rows.  256: each CTA streams one half of every tile.  128 (PAIRED): the
    // surviving tiles of an item are taken two at a time, CTA c streaming the whole of the
    // (2m + c)-th -- one M = 256, N = 256 MMA covers two 128-row tiles (an N = 128 MMA ran at
    // half the rate: c4 380 vs 700 TF/s), while the tile test prunes at 128-row granularity
    constexpr bool PAIRED = BNT == 128;
    constexpr int HALF = 128;                              // tail rows per CTA and MMA
    constexpr int TSTEP = PAIRED ? 2 : 1;                  // list entries per MMA tile
    constexpr uint32_t LBO_B2 = (HALF / 8) * 128;
    constexpr uint32_t IDESC2 = idesc_tf32(2 * BM, 2 * HALF);  // M = 256, N = 256
    extern __shared__ __align__(1024) uint8_t smem[];
    const int Kpad = p.Kpad;
    const uint32_t A_FLOATS = BM * Kpad;
    const int nkc = (Kpad + KC - 1) / KC;
    float* As = reinterpret_cast<float*>(smem);
    float* Bs = As + (size_t)a_stages * A_FLOATS;
    uint64_t* bars = reinterpret_cast<uint64_t*>(Bs + (size_t)b_stages * HALF * KC);
    uint64_t* a_full = bars;
    uint64_t* a_empty = bars + 2;
    uint64_t* acc_full = bars + 4;
    uint64_t* acc_empty = bars + 6;
    uint64_t* b_full = bars + 8;
    uint64_t* b_empty = b_full + b_stages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 40);
    float4* qrow = reinterpret_cast<float4*>(bars + 64);  // [a_stages][BM] {||q||^2, ||q||, ||q - tf32(q)||, 0}
    float* t2smem = reinterpret_cast<float*>(qrow + a_stages * BM);  // [8 epilogue warps][128]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = cluster_ctarank();
    const bool leader = crank == 0;
    const long long cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    // gathered: the item count was produced on the device (round-robin items)
    const long long n_items = GATHER ? *p.dn_items : p.n_items;
    const bool sched = !GATHER && p.sched;
    const long long it_begin = sched ? balanced_begin(p.item_cum, n_items, p.total_tiles, cid, ncl) : cid;
    const long long it_end = sched ? balanced_begin(p.item_cum, n_items, p.total_tiles, cid + 1, ncl) : n_items;
    const long long it_step = sched ? 1 : ncl;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&a_full[i], leader ? 2 * BM : BM);
            mbar_init(&a_empty[i], 1 + 8);
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 16);
        }
        for (int i = 0; i < b_stages; ++i) {
            // producer: one expect_tx arrival (bulk copy) or 32 lane arrivals (gathered); + the relay
            const uint32_t prod = GATHER ? 32u : 1u;
            mbar_init(&b_full[i], leader ? prod + 1 : prod);
            mbar_init(&b_empty[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
    tc_fence_before();
    cluster_sync_all();  // barrier inits + the TMEM address visible in both CTAs
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && GATHER) {
        // ------------------------------------------------ producer (gathered blocks): this CTA's 128 rows
        int bi = 0, npend = 0;
        uint32_t bph = 0;
        const int lag = b_stages - 1 < 3 ? b_stages - 1 : 3;  // chunks in flight (measured: 5 slower than 3)
        const int p8 = lane & 7, rsub = lane >> 3;            // 16-byte piece of a 128-byte row chunk; row in a quad
        auto signal_oldest = [&](int keep) {
            cp_async_wait_n(keep);
            fence_proxy_async_smem();  // generic-proxy smem writes -> visible to tcgen05.mma
            int s0 = bi - npend;
            if (s0 < 0) s0 += b_stages;
            mbar_arrive(&b_full[s0]);
            --npend;
        };
        for (long long it = it_begin; it < it_end; it += it_step) {
            const int4 w = p.items[it];
            for (int jj = w.y; jj <= w.z; ++jj) {
                // the block's 128 row indices of this CTA: lane l loads rows 4l..4l+3, then lane
                // l keeps the index of row 4u + rsub for every instruction u
                const int4 rv = __ldg(reinterpret_cast<const int4*>(p.glist + ((long long)w.w + jj) * BNT +
                                                                    crank * HALF) + lane);
                int idx[32];
#pragma unroll
                for (int u = 0; u < 32; ++u) {
                    const int a = __shfl_sync(0xffffffffu, rv.x, u), b = __shfl_sync(0xffffffffu, rv.y, u);
                    const int c2 = __shfl_sync(0xffffffffu, rv.z, u), d2 = __shfl_sync(0xffffffffu, rv.w, u);
                    idx[u] = rsub == 0 ? a : (rsub == 1 ? b : (rsub == 2 ? c2 : d2));
                }
                for (int c = 0; c < nkc; ++c) {
                    TC2_WAIT(0, &b_empty[bi], bph ^ 1);
                    const int klen = Kpad - c * KC < KC ? Kpad - c * KC : KC;
                    if (4 * p8 < klen) {
                        const uint32_t sbase = smem_u32(Bs + (size_t)bi * HALF * KC);
                        const float* src0 = p.Ts + (size_t)c * KC + 4 * p8;
#pragma unroll
                        for (int u = 0; u < 32; ++u) {
                            const int i = 4 * u + rsub;
                            // K-major, 128-byte swizzle: row i's 128-byte K-chunk at i * 128, its 16-byte
                            // piece p at (p ^ (i % 8)) * 16 -- the 4 rows of one instruction fill 512
                            // contiguous bytes (no bank conflicts; the no-swizzle layout put the 8 pieces of
                            // a row 2 KB apart: 8-way conflicts)
                            const uint32_t off = (uint32_t)(i * 128 + ((p8 ^ (i & 7)) << 4));
                            cp_async16(sbase + off, src0 + (size_t)idx[u] * Kpad);
                        }
                    }
                    cp_async_commit();
                    ++npend;
                    if (++bi == b_stages) { bi = 0; bph ^= 1; }
                    if (npend > lag) signal_oldest(lag);
                }
            }
        }
        while (npend > 0) signal_oldest(0);
        for (int k = 0; k < b_stages; ++k) {  // drain: the last commits have landed
            mbar_wait(&b_empty[bi], bph ^ 1);
            if (++bi == b_stages) { bi = 0; bph ^= 1; }
        }
    } else if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ producer: this CTA's half of each tail tile
            int bi = 0;
            uint32_t bph = 0;
            const uint64_t pol_keep = l2_policy_evict_last();
            for (long long it = it_begin; it < it_end; it += it_step) {
                const int4 w = p.items[it];
                for (int j = w.y; j <= w.z; j += TSTEP) {
                    // PAIRED: this CTA's tile is list entry j + crank (none past the item's end: the
                    // MMA half it feeds is ignored by the epilogue)
                    const bool have = !PAIRED || j + (int)crank <= w.z;
                    const float* tsrc = PAIRED ? p.Tp + (size_t)(have ? item_tile(w, j + crank, p.tile_list) : 0) * HALF * Kpad
                                               : p.Tp + ((size_t)item_tile(w, j, p.tile_list) * BNT + crank * HALF) * Kpad;
                    for (int c = 0; c < nkc; ++c) {
                        const int klen = Kpad - c * KC < KC ? Kpad - c * KC : KC;
                        const uint32_t bytes = (uint32_t)klen * HALF * 4;
                        TC2_WAIT(0, &b_empty[bi], bph ^ 1);
                        if (!have) {
                            mbar_arrive(&b_full[bi]);  // the stage's arrival, no bytes
                            if (++bi == b_stages) { bi = 0; bph ^= 1; }
                            continue;
                        }
                        mbar_arrive_expect_tx(&b_full[bi], bytes);
                        if (p.l2hint)  // the staged tails are re-read for every query tile: keep them in L2
                            bulk_g2s_hint(Bs + (size_t)bi * HALF * KC, tsrc + (size_t)c * KC * HALF, bytes, &b_full[bi],
                                          pol_keep);
                        else
                            bulk_g2s(Bs + (size_t)bi * HALF * KC, tsrc + (size_t)c * KC * HALF, bytes, &b_full[bi]);
                        if (++bi == b_stages) { bi = 0; bph ^= 1; }
                    }
                }
            }
            for (int k = 0; k < b_stages; ++k) {  // drain: the last commits have landed
                mbar_wait(&b_empty[bi], bph ^ 1);
                if (++bi == b_stages) { bi = 0; bph ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            // ------------------------------------------------ MMA issuer (even CTA)
            int ai = 0, bi = 0, acc = 0;
            uint32_t aph = 0, bph = 0, accph = 0;
            for (long long it = it_begin; it < it_end; it += it_step) {
                const int4 w = p.items[it];
                TC2_WAIT(1, &a_full[ai], aph);
                tc_fence_after();
                const uint64_t a_desc0 = umma_desc_kmajor(smem_u32(As + (size_t)ai * A_FLOATS), LBO_A2, SBO2);
                for (int j = w.y; j <= w.z; j += TSTEP) {
                    TC2_WAIT(2, &acc_empty[acc], accph ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem + (uint32_t)(acc * 2 * HALF);
                    for (int c = 0; c < nkc; ++c) {
                        TC2_WAIT(3, &b_full[bi], bph);
                        tc_fence_after();
                        const uint64_t b_desc0 = GATHER ? umma_desc_sw128(smem_u32(Bs + (size_t)bi * HALF * KC))
                                                        : umma_desc_kmajor(smem_u32(Bs + (size_t)bi * HALF * KC), LBO_B2, SBO2);
                        // descriptor units (16 B) per K = 8 step: 32 bytes in the swizzled rows, 2 core matrices otherwise
                        const uint32_t bstep = GATHER ? 2u : 2u * (LBO_B2 >> 4);
                        const int nsteps = (Kpad - c * KC < KC ? Kpad - c * KC : KC) / 8;
                        const uint64_t a_desc = a_desc0 + (uint64_t)((uint32_t)(c * KC / 4) * (LBO_A2 >> 4));
                        if (elect_one()) {
#pragma unroll
                            for (int s = 0; s < 4; ++s) {
                                if (s < nsteps)
                                    mma_tf32_pair(d_tmem, a_desc + (uint64_t)(2 * s * (LBO_A2 >> 4)),
                                                  b_desc0 + (uint64_t)(s * bstep), IDESC2, (c | s) != 0);
                            }
                            mma_commit_pair(&b_empty[bi], 3);
                        }
                        __syncwarp();
                        if (++bi == b_stages) { bi = 0; bph ^= 1; }
                    }
                    if (elect_one()) mma_commit_pair(&acc_full[acc], 3);
                    __syncwarp();
                    if (++acc == 2) { acc = 0; accph ^= 1; }
                }
                if (elect_one()) mma_commit_pair(&a_empty[ai], 3);
                __syncwarp();
                if (++ai == a_stages) { ai = 0; aph ^= 1; }
            }
            for (int k = 0; k < 2; ++k) {  // drain: both CTAs' epilogues released the accumulators
                mbar_wait(&acc_empty[acc], accph ^ 1);
                if (++acc == 2) { acc = 0; accph ^= 1; }
            }
        } else if (lane == 0) {
            // ------------------------------------------------ relay (odd CTA): forward B-chunk completions
            int bi = 0;
            uint32_t bph = 0;
            for (long long it = it_begin; it < it_end; it += it_step) {
                const int4 w = p.items[it];
                for (int j = w.y; j <= w.z; j += TSTEP) {
                    for (int c = 0; c < nkc; ++c) {
                        TC2_WAIT(7, &b_full[bi], bph);
                        mbar_arrive_cluster(&b_full[bi], 0);
                        if (++bi == b_stages) { bi = 0; bph ^= 1; }
                    }
                }
            }
        }
    } else if (warp < TC2_BUILDER_WARP0) {
        // ---------------------------------------------------- epilogue (both CTAs, own 128 rows)
        // Each warp's ||t||^2 / 2 slice (128 floats) and band maxima of the NEXT tile are loaded one
        // tile ahead (one float4 per lane) and parked in shared memory: read at use they were a
        // global-load latency per 32-column chunk, and on d = 128 (c5) the MMA waited on the
        // accumulator 38% of the time (ncu: the first FADD2 of each chunk stalled on them).
        const int q = warp & 3;
        const int hcol = (warp - 2) >> 2;       // column half of the 256-column accumulator
        const int col0 = hcol * HALF;           // its first TMEM column
        const int tcol = PAIRED ? 0 : col0;     // this warp's first column inside its tile
        const int i = q * 32 + lane;
        float* t2s = t2smem + (warp - 2) * 128;
        const float* t2base = GATHER ? p.gT2 : p.T2;
        auto tile_of = [&](const int4& w, int jj, int& j, bool& have) {
            // PAIRED: this warp's column half is list entry jj + hcol (absent past the item's end)
            have = !PAIRED || jj + hcol <= w.z;
            // gathered: j is the block (the tile list's offset + jj), else the tail tile
            j = GATHER ? w.w + jj : item_tile(w, PAIRED ? (have ? jj + hcol : jj) : jj, p.tile_list);
        };
        float4 nt2 = make_float4(0.f, 0.f, 0.f, 0.f);
        float2 ntv = make_float2(0.f, 0.f);
        auto load_ahead = [&](const int4& w, int jj) {
            int j;
            bool hv;
            tile_of(w, jj, j, hv);
            nt2 = __ldg(reinterpret_cast<const float4*>(t2base + (size_t)j * BNT + tcol) + lane);
            ntv = GATHER ? p.gtst[j] : p.tstile[j];
        };
        if (it_begin < it_end) {
            const int4 w0 = p.items[it_begin];
            load_ahead(w0, w0.y);
        }
        int acc = 0, ai = 0;
        uint32_t accph = 0, aph = 0;
        for (long long it = it_begin; it < it_end; it += it_step) {
            const int4 w = p.items[it];
            TC2_WAIT(4, &a_full[ai], aph);
            const float4 qv = qrow[ai * BM + i];
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_empty[ai]);
            if (++ai == a_stages) { ai = 0; aph ^= 1; }
            const float Q2 = qv.x, Qn = qv.y, Qd = qv.z;
            const int rowid = w.x * (2 * BM) + (int)crank * BM + i;
            const float thf = p.theta * (1.0f + 2.44140625e-04f) + 2.384185791015625e-07f * Qn;
            for (int jj = w.y; jj <= w.z; jj += TSTEP) {
                int j;
                bool have;
                tile_of(w, jj, j, have);
                // this tile's slice (loaded a tile ago) into shared memory, then the next tile's loads
                __syncwarp();
                reinterpret_cast<float4*>(t2s)[lane] = nt2;
                const float2 tv = ntv;
                __syncwarp();
                if (jj + TSTEP <= w.z) {
                    load_ahead(w, jj + TSTEP);
                } else if (it + it_step < it_end) {
                    const int4 wn = p.items[it + it_step];
                    load_ahead(wn, wn.y);
                }
                const float Tm = tv.x, Tdm = tv.y;
                // guard band exactly as tiles_tc.cu
                const float eb = Qd * Tm + Qn * Tdm + Qd * Tdm + p.eta * (Qn + Qd) * (Tm + Tdm);
                const float sl = 4.76837158203125e-07f * (Qn + Tm) * (Qn + Tm);
                const float R = thf * thf + 2.0f * eb + sl;
                const float c = Q2 - R - (float)(p.Kpad + 4) * 1.1920928955078125e-07f * Q2 - 9.5367431640625e-07f * (Q2 + R);
                TC2_WAIT(5, &acc_full[acc], accph);
                tc_fence_after();
                const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * 2 * HALF + col0);
                uint32_t ra[32], rb[32];
                const float ch2 = 0.5f * c;  // T2 holds ||t||^2 / 2 (stage kernel)
                auto process = [&](const uint32_t (&r)[32], int ch) {
                    if (!have) return;
                    const float4* t2 = reinterpret_cast<const float4*>(t2s + ch * 32);
                    const float m = epi_max32_s(r, t2);
                    if (__any_sync(0xffffffffu, m >= ch2)) {
                        uint32_t hit = epi_hits32_s(r, t2, ch2);
                        unsigned long long slot = warp_reserve(__popc(hit), p.cand_count);
                        const int colb = j * BNT + tcol + ch * 32;
                        while (hit) {
                            const int u = __ffs(hit) - 1;
                            // gathered: the list entry holds the sorted tail position
                            const int col = GATHER ? __ldg(p.glist + (size_t)colb + u) : colb + u;
                            if (slot < (unsigned long long)p.cand_cap) p.cand[slot] = make_int2(rowid, col);
                            ++slot;
                            hit &= hit - 1;
                        }
                    }
                };
                // software-pipelined TMEM loads: chunk ch + 1 is in flight while ch is tested
                tmem_ld32_nowait(tbase + 0, ra);
                tmem_wait_ld();
                tmem_ld32_nowait(tbase + 32, rb);
                process(ra, 0);
                tmem_wait_ld();
                tmem_ld32_nowait(tbase + 64, ra);
                process(rb, 1);
                tmem_wait_ld();
                tmem_ld32_nowait(tbase + 96, rb);
                process(ra, 2);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (leader) mbar_arrive(&acc_empty[acc]);
                    else mbar_arrive_cluster(&acc_empty[acc], 0);
                }
                process(rb, 3);
                if (++acc == 2) { acc = 0; accph ^= 1; }
            }
        }
    }
    if (warp >= TC2_BUILDER_WARP0) {
        // ---------------------------------------------------- builders (tc_build.cuh)
        const int wb = warp - TC2_BUILDER_WARP0;
        const bool vec4 = (p.d % 4 == 0) && ((reinterpret_cast<uintptr_t>(p.E) | reinterpret_cast<uintptr_t>(p.Rel)) % 16 == 0);
        const int i = wb * 32 + lane;  // the row whose next-item entity row this lane prefetches
        int ai = 0;
        uint32_t aph = 0;
        for (long long it = it_begin; it < it_end; it += it_step) {
            const int4 w = p.items[it];
            const int r = w.x / p.QT;
            TC2_WAIT(6, &a_empty[ai], aph ^ 1);
            build_query_rows(As + (size_t)ai * A_FLOATS, qrow + ai * BM, p.E, p.Rel, p.qperm, p.N, p.d, Kpad, r,
                             (long long)(w.x - r * p.QT) * (2 * BM) + crank * BM, wb, lane, vec4, p.l2hint);
            fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the pair's tcgen05.mma
            mbar_arrive(&a_full[ai]);
            if (!leader) mbar_arrive_cluster(&a_full[ai], 0);
            if (++ai == a_stages) { ai = 0; aph ^= 1; }
            if (a_stages == 1 && p.t2pf && it + it_step < it_end) {
                // one query-tile buffer: the next build waits for every MMA of this item, so pull
                // the next item's entity rows into L2 now (prefetch.global.L2, one per 128-B line)
                const int4 wn = p.items[it + it_step];
                const int rn = wn.x / p.QT;
                const long long posn = (long long)(wn.x - rn * p.QT) * (2 * BM) + crank * BM + i;
                if (posn < p.N) {
                    const char* rowp = reinterpret_cast<const char*>(p.E + (long long)p.qperm[(long long)rn * p.N + posn] * p.d);
                    for (int b = 0; b < p.d * 4; b += 128) prefetch_l2(rowp + b);
                }
            }
        }
        for (int k = 0; k < a_stages; ++k) {  // drain: the last a_empty commits have landed
            mbar_wait(&a_empty[ai], aph ^ 1);
            if (++ai == a_stages) { ai = 0; aph ^= 1; }
        }
    }
    tc_fence_before();
    cluster_sync_all();  // no CTA leaves while its partner may still signal it
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(tmem, 512);
    }
}

#ifdef KGC_PROF_TC
}  // namespace kgc
extern "C" __attribute__((visibility("default"))) void kgc_debug_tc2_prof(unsigned long long* out16, int reset) {
    if (out16) cudaMemcpyFromSymbol(out16, kgc::g_tc2_prof, 16 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(kgc::g_tc2_prof, z, sizeof z);
    }
}
namespace kgc {
#endif

template <bool GATHER, int BNT>
static void launch_tc2(const TileParams& p, int num_sms, cudaStream_t s) {
    if (p.n_items <= 0) return;
    int as, bs, kc;
    const int smem = tc2_smem_bytes(p.Kpad, &as, &bs, &kc, BNT);
    auto kern = tiles_tc2_kernel<GATHER, BNT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(TC2_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(num_sms & ~1);
    int max_clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters <= 0) {
        cudaGetLastError();
        max_clusters = num_sms / 2;
    }
    long long g = p.n_items < max_clusters ? p.n_items : max_clusters;  // gathered: n_items is a bound
    cfg.gridDim = dim3((unsigned)(2 * g));
    cudaLaunchKernelEx(&cfg, kern, p, as, bs, kc);
}

void launch_tiles_tc2(const TileParams& p, int num_sms, cudaStream_t s) {
    if (p.bn == 128) launch_tc2<false, 128>(p, num_sms, s);
    else launch_tc2<false, BN_TC>(p, num_sms, s);
}

// gathered tail blocks need 32-wide K-chunks (8 pieces of 16 bytes per row chunk)
int tc2_gather_ok(int Kpad) {
    int as, bs, kc;
    return tc2_smem_bytes(Kpad, &as, &bs, &kc, BN_TC) > 0 && kc == 32 && bs >= 2;
}
void launch_tiles_tc2_gather(const TileParams& p, int num_sms, cudaStream_t s) { launch_tc2<true, BN_TC>(p, num_sms, s); }

}  // namespace kgc
