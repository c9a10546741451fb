// tiles_tc.cu -- K4: the L2 surviving-tile contraction on the 5th-generation
// tensor cores.
//
// For a surviving (query tile, tail tile) pair, D^2(q, t) = ||q||^2 + ||t||^2
// - 2 q.t (TransE L2); the q.t block (128 x 256, K = d padded
// to 8) is one tcgen05 kind::tf32 GEMM tile.  TF32 rounds the operands, so
// the epilogue keeps every pair whose D^2 could be <= theta^2 under a
// rigorous bound on the TF32 + accumulation error (the guard band), and the
// FP64 re-check (verify.cu) decides -- the filtering stays lossless
// (PAPER.md:349-351).
//
// Persistent kernel, one CTA per SM, 448 threads:
//   warp 0      producer: 1-D bulk TMA (cp.async.bulk) of K-chunks of the
//               staged tail tiles
//   warps 10-13 builders: form the query tile q = fl32(h + r) of the next
//               work item in shared memory (UMMA layout) + its row scalars
//   warp 1      TMEM allocation + single-thread tcgen05.mma issue
//   warps 2..9  epilogue: tcgen05.ld 32x32b.x32 -> band test -> candidates
// TMEM holds two 128 x 256 FP32 accumulators (all 512 columns) so the
// epilogue of tile j overlaps the MMAs of tile j + 1.
#include <cstdio>

#include "common.cuh"
#include "tc_build.cuh"

namespace kgc {

#ifdef KGC_PROF_TC
// debug build only: cycles each role spends blocked in each barrier wait
__device__ unsigned long long g_tc_prof[16];
#define TC_WAIT(slot, bar, par)                                    \
    do {                                                           \
        const long long t0_ = clock64();                           \
        mbar_wait(bar, par);                                       \
        atomicAdd(&g_tc_prof[slot], (unsigned long long)(clock64() - t0_)); \
    } while (0)
#else
#define TC_WAIT(slot, bar, par) mbar_wait(bar, par)
#endif
constexpr int TC_THREADS = 448;  // 2 control warps + 8 epilogue warps + 4 builder warps
constexpr int TC_BUILDER_WARP0 = 10;
constexpr uint32_t LBO_A = (BM / 8) * 128;     // bytes between K-adjacent core matrices, query tile
constexpr uint32_t LBO_B = (BN_TC / 8) * 128;  // same, tail tile
constexpr uint32_t SBO = 128;                  // bytes between M/N-adjacent core matrices
constexpr uint32_t IDESC = idesc_tf32(BM, BN_TC);
constexpr int TC_T2S_BYTES = 8 * 128 * 4;       // per epilogue warp: ||t||^2 / 2 of its 128 columns

int tc_smem_bytes(int Kpad, int* a_stages, int* b_stages, int* kc) {
    const int budget = 227 * 1024 - 512 - 2 * BM * 16 - TC_T2S_BYTES;
    const int A = BM * Kpad * 4;
    for (int KC : {32, 16, 8}) {
        const int B = BN_TC * KC * 4;
        for (int as = 2; as >= 1; --as) {
            int rem = budget - as * A;
            if (rem <= 0) continue;
            int bs = rem / B;
            if (bs > 4) bs = 4;
            if (bs >= 2) {
                *a_stages = as;
                *b_stages = bs;
                *kc = KC;
                int bytes = as * A + bs * B + 256 + as * BM * 16 + TC_T2S_BYTES;
                // >= 117 KB keeps one CTA per SM, so the 512-column TMEM
                // allocation never waits on a co-resident CTA.
                return bytes < 117 * 1024 ? 117 * 1024 : bytes;
            }
        }
    }
    return -1;
}

// GATHER: tail blocks are the query tile's gathered surviving tails (pivots.cu,
// gather_tails_kernel<256>): the producer thread gathers their rows from the
// sorted row-major tails with TMA row gathers (cp.async.bulk.tensor ...
// tile::gather4, a 2-D tensor map over Ts with 128-byte swizzle), so each K-chunk
// of 32 arrives as a 128B-swizzled K-major operand (umma_desc_sw128); the
// epilogue takes ||t||^2/2 and the block's guard-band maxima from the list build.
// (A warp of 16-byte cp.async pieces was measured 4x slower than contiguous tiles
// on c3: one warp cannot keep enough scattered loads in flight.)
// MODE 2 (FACTORED): the relation-factored L2 join for low-pruning
// data.  D^2(h, r, t) = ||h + r||^2 + ||t||^2 - 2 h.t - 2 r.t (TransE), so a
// 128 x 256 tile of G = H T^T (heads in natural order, every tail tile, no relation)
// serves all R relations: per relation the epilogue adds r.t (table) and tests against
// (||h + r||^2 - theta^2) / 2 (table), widened by the TF32 band of G and the FP32
// rounding of the two additions.
template <int MODE>
__global__ void __launch_bounds__(TC_THREADS, 1) tiles_tc_kernel(TileParams p, int a_stages, int b_stages, int KC) {
    constexpr bool GATHER = MODE == 1, FACT = MODE == 2;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int Kpad = p.Kpad;
    const uint32_t A_FLOATS = BM * Kpad;
    const int nkc = (Kpad + KC - 1) / KC;
    float* As = reinterpret_cast<float*>(smem);
    float* Bs = As + (size_t)a_stages * A_FLOATS;
    uint64_t* bars = reinterpret_cast<uint64_t*>(Bs + (size_t)b_stages * BN_TC * KC);
    uint64_t* a_full = bars;
    uint64_t* a_empty = bars + 2;
    uint64_t* b_full = bars + 4;
    uint64_t* b_empty = b_full + b_stages;
    uint64_t* acc_full = b_empty + b_stages;
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    float4* qrow = reinterpret_cast<float4*>(bars + 32);  // [a_stages][BM] {||q||^2, ||q||, ||q - tf32(q)||, 0}
    float* t2smem = reinterpret_cast<float*>(qrow + a_stages * BM);  // [8 epilogue warps][128]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // this CTA's contiguous, cost-balanced block of work items (every role walks it)
    // gathered: the item count and block total were produced on the device
    const long long n_items = GATHER ? *p.dn_items : p.n_items, total = GATHER ? *p.dtotal : p.total_tiles;
    const long long it_begin = p.sched ? balanced_begin(p.item_cum, n_items, total, blockIdx.x, gridDim.x)
                                       : (long long)blockIdx.x;
    const long long it_end = p.sched ? balanced_begin(p.item_cum, n_items, total, blockIdx.x + 1, gridDim.x)
                                     : n_items;
    const long long it_step = p.sched ? 1 : gridDim.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&a_full[i], BM);        // one arrival per builder thread (one row each)
            mbar_init(&a_empty[i], 1 + 8);    // MMA commit + the 8 epilogue warps (row scalars read)
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 8);
        }
        for (int i = 0; i < b_stages; ++i) {
            mbar_init(&b_full[i], 1);
            mbar_init(&b_empty[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && GATHER) {
        // ------------------------------------------------ producer (gathered tail blocks)
        // 64 TMA row gathers of 4 rows x 128 bytes per K-chunk (KC = 32: one 128-byte
        // swizzle atom row; columns past Kpad are zero-filled by TMA).  The block's row
        // indices are loaded once per block, lane l holding gathers l and l + 32.
        int bi = 0;
        uint32_t bph = 0;
        for (long long it = it_begin; it < it_end; it += it_step) {
            const int4 w = p.items[it];
            for (int jj = w.y; jj <= w.z; ++jj) {
                const int4* seg = reinterpret_cast<const int4*>(p.glist + ((long long)w.w + jj) * BN_TC);
                const int4 ra = __ldg(seg + lane), rb = __ldg(seg + lane + 32);
                for (int c = 0; c < nkc; ++c) {
                    TC_WAIT(0, &b_empty[bi], bph ^ 1);
                    if (lane == 0) mbar_arrive_expect_tx(&b_full[bi], (uint32_t)BN_TC * 128u);
                    __syncwarp();
                    const uint32_t bbase = smem_u32(Bs + (size_t)bi * BN_TC * KC);
                    tma_gather4(bbase + (uint32_t)lane * 512u, p.tmap, c * KC, ra.x, ra.y, ra.z, ra.w, &b_full[bi]);
                    tma_gather4(bbase + (uint32_t)(lane + 32) * 512u, p.tmap, c * KC, rb.x, rb.y, rb.z, rb.w,
                                &b_full[bi]);
                    if (++bi == b_stages) { bi = 0; bph ^= 1; }
                }
            }
        }
    } else if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ producer (tail tiles)
            int bi = 0;
            uint32_t bph = 0;
            for (long long it = it_begin; it < it_end; it += it_step) {
                const int4 w = p.items[it];
                for (int j = w.y; j <= w.z; ++j) {
                    const float* tsrc = p.Tp + (size_t)item_tile(w, j, p.tile_list) * BN_TC * Kpad;
                    for (int c = 0; c < nkc; ++c) {
                        const int klen = Kpad - c * KC < KC ? Kpad - c * KC : KC;
                        const uint32_t bytes = (uint32_t)klen * BN_TC * 4;
                        TC_WAIT(0, &b_empty[bi], bph ^ 1);
                        mbar_arrive_expect_tx(&b_full[bi], bytes);
                        bulk_g2s(Bs + (size_t)bi * BN_TC * KC, tsrc + (size_t)c * KC * BN_TC, bytes, &b_full[bi]);
                        if (++bi == b_stages) { bi = 0; bph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------- MMA issuer
        // The whole warp walks the schedule (so every operand of tcgen05.mma is
        // warp-uniform and lives in uniform registers); one elected lane issues.
        int ai = 0, bi = 0, acc = 0;
        uint32_t aph = 0, bph = 0, accph = 0;
        for (long long it = it_begin; it < it_end; it += it_step) {
            const int4 w = p.items[it];
            TC_WAIT(1, &a_full[ai], aph);
            tc_fence_after();
            const uint64_t a_desc0 = umma_desc_kmajor(smem_u32(As + (size_t)ai * A_FLOATS), LBO_A, SBO);
            for (int j = w.y; j <= w.z; ++j) {
                TC_WAIT(2, &acc_empty[acc], accph ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + (uint32_t)(acc * BN_TC);
                for (int c = 0; c < nkc; ++c) {
                    TC_WAIT(3, &b_full[bi], bph);
                    tc_fence_after();
                    // gathered blocks arrive 128B-swizzled (TMA); a K step is 32 bytes there
                    const uint64_t b_desc0 = GATHER ? umma_desc_sw128(smem_u32(Bs + (size_t)bi * BN_TC * KC))
                                                    : umma_desc_kmajor(smem_u32(Bs + (size_t)bi * BN_TC * KC), LBO_B, SBO);
                    constexpr uint32_t BSTEP = GATHER ? 2u : 2u * (LBO_B >> 4);  // descriptor units per K = 8
                    const int nsteps = (Kpad - c * KC < KC ? Kpad - c * KC : KC) / 8;
                    // descriptor start address advances by 2 core matrices (K = 8) per step
                    const uint64_t a_desc = a_desc0 + (uint64_t)((uint32_t)(c * KC / 4) * (LBO_A >> 4));
                    if (elect_one()) {
#pragma unroll
                        for (int s = 0; s < 4; ++s) {
                            if (s < nsteps)
                                mma_tf32(d_tmem, a_desc + (uint64_t)(2 * s * (LBO_A >> 4)), b_desc0 + (uint64_t)(s * BSTEP),
                                         IDESC, (c | s) != 0);
                        }
                        for (int s = 4; s < nsteps; ++s)  // KC > 32 is not configured; kept for safety
                            mma_tf32(d_tmem, a_desc + (uint64_t)(2 * s * (LBO_A >> 4)), b_desc0 + (uint64_t)(s * BSTEP),
                                     IDESC, 1u);
                        mma_commit(&b_empty[bi]);
                    }
                    __syncwarp();
                    if (++bi == b_stages) { bi = 0; bph ^= 1; }
                }
                if (elect_one()) mma_commit(&acc_full[acc]);
                __syncwarp();
                if (++acc == 2) { acc = 0; accph ^= 1; }
            }
            if (elect_one()) mma_commit(&a_empty[ai]);
            __syncwarp();
            if (++ai == a_stages) { ai = 0; aph ^= 1; }
        }
    } else if (warp < TC_BUILDER_WARP0) {
        // ---------------------------------------------------- epilogue
        // 8 warps: warp w reads TMEM lane quadrant (w % 4) (hardware rule) and
        // column half (w - 2) / 4 of the 128 x 256 accumulator.
        const int q = warp & 3;
        const int col0 = ((warp - 2) >> 2) * (BN_TC / 2);
        const int i = q * 32 + lane;
        int acc = 0, ai = 0;
        uint32_t accph = 0, aph = 0;
        float* t2s = t2smem + (warp - 2) * 128;
        float4 nt2 = make_float4(0.f, 0.f, 0.f, 0.f);
        float2 ntv = make_float2(0.f, 0.f);
        auto load_ahead = [&](const int4& w, int jj) {
            const int j = GATHER ? w.w + jj : item_tile(w, jj, p.tile_list);
            nt2 = __ldg(reinterpret_cast<const float4*>((GATHER ? p.gT2 : p.T2) + (size_t)j * BN_TC + col0) + lane);
            ntv = GATHER ? p.gtst[j] : p.tstile[j];
        };
        if (!FACT && it_begin < it_end) {
            const int4 w0 = p.items[it_begin];
            load_ahead(w0, w0.y);
        }
        for (long long it = it_begin; it < it_end; it += it_step) {
            const int4 w = p.items[it];
            TC_WAIT(4, &a_full[ai], aph);
            const float4 qv = qrow[ai * BM + i];
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_empty[ai]);
            if (++ai == a_stages) { ai = 0; aph ^= 1; }
            const float Q2 = qv.x, Qn = qv.y, Qd = qv.z;
            const int rowid = w.x * BM + i;
            // theta_f covers q = fl32(h + r) vs the exact h + r (|dq_k| <= 2^-24 |q_k|)
            const float thf = p.theta * (1.0f + 2.44140625e-04f) + 2.384185791015625e-07f * Qn;
            if (FACT) {
                const long long h = (long long)w.x * BM + i;
                const bool hv = h < p.N;
                const long long rows_per_rel = (long long)p.QT * BM;
                for (int j = w.y; j <= w.z; ++j) {
                    const float2 tv = p.tstile[j];
                    const float Tm = tv.x, Tdm = tv.y;
                    const float eb = Qd * Tm + Qn * Tdm + Qd * Tdm + p.eta * (Qn + Qd) * (Tm + Tdm);
                    const float* t2row = p.T2 + (size_t)j * BN_TC + col0;
                    TC_WAIT(5, &acc_full[acc], accph);
                    tc_fence_after();
                    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN_TC + col0);
                    for (int ch = 0; ch < 4; ++ch) {
                        uint32_t ra[32];
                        tmem_ld32_nowait(tbase + 32 * ch, ra);
                        tmem_wait_ld();
                        if (ch == 3) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&acc_empty[acc]);
                        }
                        float v[32];  // acc - ||t||^2 / 2 (padding columns: -3e38)
                        const float4* t2 = reinterpret_cast<const float4*>(t2row + ch * 32);
#pragma unroll
                        for (int u4 = 0; u4 < 8; ++u4) {
                            const float4 tt = __ldg(t2 + u4);
                            v[4 * u4 + 0] = __uint_as_float(ra[4 * u4 + 0]) - tt.x;
                            v[4 * u4 + 1] = __uint_as_float(ra[4 * u4 + 1]) - tt.y;
                            v[4 * u4 + 2] = __uint_as_float(ra[4 * u4 + 2]) - tt.z;
                            v[4 * u4 + 3] = __uint_as_float(ra[4 * u4 + 3]) - tt.w;
                        }
                        const long long colb = (long long)j * BN_TC + col0 + ch * 32;
                        // relations FU at a time over FC-column slices: the table loads of FU relations
                        // are in flight together (one at a time, the loop waited on L2 per relation)
                        constexpr int FU = 4, FC = 16, FQ = FC / 4;  // measured: 4 x 16 best (8 x 8: 2.8x slower)
#pragma unroll
                        for (int hf = 0; hf < 32 / FC; ++hf) {
                            for (int rel0 = 0; rel0 < p.R; rel0 += FU) {
                                float zd[FU], rn[FU];
                                float4 rt[FU][FQ];
#pragma unroll
                                for (int u = 0; u < FU; ++u) {
                                    const int rel = rel0 + u;
                                    const bool rv = rel < p.R;
                                    zd[u] = (rv && hv) ? __ldg(p.fz + (size_t)rel * p.N + h) : 3e38f;
                                    rn[u] = rv ? __ldg(p.frn + rel) : 0.f;
                                    const float4* rt4 = reinterpret_cast<const float4*>(
                                                            p.frt + (size_t)(rv ? rel : 0) * p.ntpad + colb) + FQ * hf;
#pragma unroll
                                    for (int q4 = 0; q4 < FQ; ++q4) rt[u][q4] = __ldg(rt4 + q4);
                                }
#pragma unroll
                                for (int u = 0; u < FU; ++u) {
                                    // S' = fl(fl(acc - T2) + fl(r.t)) is within eb + 2^-21 (Hn + Rn + Tm)^2 of
                                    // h.t + r.t - ||t||^2/2; a hit has S >= Z = (||h + r||^2 - theta^2)/2 >= zd
                                    const float e2 = Qn + rn[u] + Tm;
                                    const float err = eb + 4.76837158203125e-07f * e2 * e2;
                                    const float c = zd[u] - err * 1.0000010f - 2.384185791015625e-07f * fabsf(zd[u]);
                                    float m0 = -3e38f, m1 = -3e38f;
#pragma unroll
                                    for (int q4 = 0; q4 < FQ; ++q4) {
                                        const int b0 = FC * hf + 4 * q4;
                                        m0 = max3_f32(m0, v[b0 + 0] + rt[u][q4].x, v[b0 + 1] + rt[u][q4].y);
                                        m1 = max3_f32(m1, v[b0 + 2] + rt[u][q4].z, v[b0 + 3] + rt[u][q4].w);
                                    }
                                    if (__any_sync(0xffffffffu, fmaxf(m0, m1) >= c)) {
                                        uint32_t hit = 0;
#pragma unroll
                                        for (int q4 = 0; q4 < FQ; ++q4) {
                                            const int b0 = FC * hf + 4 * q4;
                                            hit |= (uint32_t)(v[b0 + 0] + rt[u][q4].x >= c) << (4 * q4 + 0);
                                            hit |= (uint32_t)(v[b0 + 1] + rt[u][q4].y >= c) << (4 * q4 + 1);
                                            hit |= (uint32_t)(v[b0 + 2] + rt[u][q4].z >= c) << (4 * q4 + 2);
                                            hit |= (uint32_t)(v[b0 + 3] + rt[u][q4].w >= c) << (4 * q4 + 3);
                                        }
                                        unsigned long long slot = warp_reserve(__popc(hit), p.cand_count);
                                        while (hit) {
                                            const int bit = __ffs(hit) - 1;
                                            if (slot < (unsigned long long)p.cand_cap)
                                                p.cand[slot] = make_int2((int)((rel0 + u) * rows_per_rel + h),
                                                                         (int)(colb + FC * hf + bit));
                                            ++slot;
                                            hit &= hit - 1;
                                        }
                                    }
                                }
                            }
                        }
                    }
                    if (++acc == 2) { acc = 0; accph ^= 1; }
                }
            }
            if (!FACT) for (int jj = w.y; jj <= w.z; ++jj) {
                // gathered: j is the block (the tile list's offset + jj), else the tail tile
                const int j = GATHER ? w.w + jj : item_tile(w, jj, p.tile_list);
                // this tile's ||t||^2 / 2 slice and band maxima (loaded a tile ago: tiles_tc2.cu) into
                // shared memory, then the next tile's loads
                __syncwarp();
                reinterpret_cast<float4*>(t2s)[lane] = nt2;
                const float2 tv = ntv;
                __syncwarp();
                if (jj < w.z) {
                    load_ahead(w, jj + 1);
                } else if (it + it_step < it_end) {
                    const int4 wn = p.items[it + it_step];
                    load_ahead(wn, wn.y);
                }
                const float Tm = tv.x, Tdm = tv.y;
                // |acc - q.t| <= Qd Tm + Qn Tdm + Qd Tdm + eta (Qn + Qd)(Tm + Tdm)
                const float eb = Qd * Tm + Qn * Tdm + Qd * Tdm + p.eta * (Qn + Qd) * (Tm + Tdm);
                const float sl = 4.76837158203125e-07f * (Qn + Tm) * (Qn + Tm);  // 8u (Qn + Tm)^2, fp32 evaluation
                const float R = thf * thf + 2.0f * eb + sl;
                // candidate iff 2 acc - ||t||^2 >= c, tested as acc - ||t||^2/2 >= c/2 (T2 holds ||t||^2/2)
                // Q2 is an FP32 sum: |Q2 - ||q||^2| <= (Kpad + 4) 2^-23 Q2 (builder)
                const float c = Q2 - R - (float)(p.Kpad + 4) * 1.1920928955078125e-07f * Q2 - 9.5367431640625e-07f * (Q2 + R);
                TC_WAIT(5, &acc_full[acc], accph);
                tc_fence_after();
                const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN_TC + col0);
                uint32_t ra[32], rb[32];
                const float ch2 = 0.5f * c;  // T2 holds ||t||^2 / 2 (stage kernel)
                auto process = [&](const uint32_t (&r)[32], int ch) {
                    const float4* t2 = reinterpret_cast<const float4*>(t2s + ch * 32);
                    const float m = epi_max32_s(r, t2);
                    if (__any_sync(0xffffffffu, m >= ch2)) {
                        uint32_t hit = epi_hits32_s(r, t2, ch2);
                        unsigned long long slot = warp_reserve(__popc(hit), p.cand_count);
                        const int colb = j * BN_TC + col0 + ch * 32;
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
                if (lane == 0) mbar_arrive(&acc_empty[acc]);
                process(rb, 3);
                if (++acc == 2) { acc = 0; accph ^= 1; }
            }
        }
    }
    if (warp >= TC_BUILDER_WARP0) {
        // ---------------------------------------------------- builders (tc_build.cuh)
        const int wb = warp - TC_BUILDER_WARP0;
        const bool vec4 = (p.d % 4 == 0) && ((reinterpret_cast<uintptr_t>(p.E) | reinterpret_cast<uintptr_t>(p.Rel)) % 16 == 0);
        int ai = 0;
        uint32_t aph = 0;
        for (long long it = it_begin; it < it_end; it += it_step) {
            const int4 w = p.items[it];
            const int r = w.x / p.QT;
            TC_WAIT(6, &a_empty[ai], aph ^ 1);
            build_query_rows(As + (size_t)ai * A_FLOATS, qrow + ai * BM, p.E, p.Rel, p.qperm, p.N, p.d, Kpad, r,
                             (long long)(w.x - r * p.QT) * BM, wb, lane, vec4);
            fence_proxy_async_smem();  // generic-proxy smem writes -> visible to tcgen05.mma
            mbar_arrive(&a_full[ai]);
            if (++ai == a_stages) { ai = 0; aph ^= 1; }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

#ifdef KGC_PROF_TC
}  // namespace kgc
extern "C" __attribute__((visibility("default"))) void kgc_debug_tc_prof(unsigned long long* out16, int reset) {
    if (out16) cudaMemcpyFromSymbol(out16, kgc::g_tc_prof, 16 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(kgc::g_tc_prof, z, sizeof z);
    }
}
namespace kgc {
#endif

void launch_tiles_tc(const TileParams& p, int num_sms, cudaStream_t s) {
    if (p.n_items <= 0) return;
    int as, bs, kc;
    int smem = tc_smem_bytes(p.Kpad, &as, &bs, &kc);
    cudaFuncSetAttribute(tiles_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long g = p.n_items < num_sms ? p.n_items : num_sms;
    tiles_tc_kernel<0><<<(unsigned)g, TC_THREADS, smem, s>>>(p, as, bs, kc);
}

// Relation-factored L2 (MODE 2): items are (head tile, tail-tile range); p.R relations per tile.
void launch_tiles_tc_factored(const TileParams& p, int num_sms, cudaStream_t s) {
    if (p.n_items <= 0) return;
    int as, bs, kc;
    int smem = tc_smem_bytes(p.Kpad, &as, &bs, &kc);
    cudaFuncSetAttribute(tiles_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long g = p.n_items < num_sms ? p.n_items : num_sms;
    tiles_tc_kernel<2><<<(unsigned)g, TC_THREADS, smem, s>>>(p, as, bs, kc);
}

// Gathered tail blocks: items, their count and block total are on the device
// (p.items, *p.dn_items, *p.dtotal); p.n_items is an upper bound that sizes the grid.
int tc_gather_ok(int Kpad) {
    int as, bs, kc;
    return tc_smem_bytes(Kpad, &as, &bs, &kc) > 0 && kc == 32;
}

void launch_tiles_tc_gather(const TileParams& p, int num_sms, cudaStream_t s) {
    if (p.n_items <= 0) return;  // here: an upper bound of the device-side item count
    int as, bs, kc;
    int smem = tc_smem_bytes(p.Kpad, &as, &bs, &kc);
    cudaFuncSetAttribute(tiles_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long g = p.n_items < num_sms ? p.n_items : num_sms;
    tiles_tc_kernel<1><<<(unsigned)g, TC_THREADS, smem, s>>>(p, as, bs, kc);
}

}  // namespace kgc
