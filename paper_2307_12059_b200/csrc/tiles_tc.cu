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
// Persistent kernel, one CTA per SM, 320 threads:
//   warp 0      producer: 1-D bulk TMA (cp.async.bulk) of the staged query
//               tile (resident for a work item) and of K-chunks of tail tiles
//   warp 1      TMEM allocation + single-thread tcgen05.mma issue
//   warps 2..9  epilogue: tcgen05.ld 32x32b.x32 -> band test -> candidates
// TMEM holds two 128 x 256 FP32 accumulators (all 512 columns) so the
// epilogue of tile j overlaps the MMAs of tile j + 1.
#include <cstdio>

#include "common.cuh"

namespace kgc {

constexpr int TC_THREADS = 320;  // 2 control warps + 8 epilogue warps
constexpr uint32_t LBO_A = (BM / 8) * 128;     // bytes between K-adjacent core matrices, query tile
constexpr uint32_t LBO_B = (BN_TC / 8) * 128;  // same, tail tile
constexpr uint32_t SBO = 128;                  // bytes between M/N-adjacent core matrices
constexpr uint32_t IDESC = idesc_tf32(BM, BN_TC);

int tc_smem_bytes(int Kpad, int* a_stages, int* b_stages, int* kc) {
    const int budget = 227 * 1024 - 512;
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
                int bytes = as * A + bs * B + 256;
                // >= 117 KB keeps one CTA per SM, so the 512-column TMEM
                // allocation never waits on a co-resident CTA.
                return bytes < 117 * 1024 ? 117 * 1024 : bytes;
            }
        }
    }
    return -1;
}

__global__ void __launch_bounds__(TC_THREADS, 1) tiles_tc_kernel(TileParams p, int a_stages, int b_stages, int KC) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int Kpad = p.Kpad;
    const uint32_t A_FLOATS = BM * Kpad;
    const uint32_t A_BYTES = A_FLOATS * 4;
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

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
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

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ producer
            int ai = 0, bi = 0;
            uint32_t aph = 0, bph = 0;
            for (long long it = blockIdx.x; it < p.n_items; it += gridDim.x) {
                const int4 w = p.items[it];
                mbar_wait(&a_empty[ai], aph ^ 1);
                mbar_arrive_expect_tx(&a_full[ai], A_BYTES);
                const float* src = p.Qp + (size_t)(w.x - p.tq0) * A_FLOATS;
                float* dst = As + (size_t)ai * A_FLOATS;
                for (uint32_t off = 0; off < A_BYTES; off += 32768u) {
                    uint32_t n = A_BYTES - off < 32768u ? A_BYTES - off : 32768u;
                    bulk_g2s(dst + off / 4, src + off / 4, n, &a_full[ai]);
                }
                if (++ai == a_stages) { ai = 0; aph ^= 1; }
                for (int j = w.y; j <= w.z; ++j) {
                    const float* tsrc = p.Tp + (size_t)j * BN_TC * Kpad;
                    for (int c = 0; c < nkc; ++c) {
                        const int klen = Kpad - c * KC < KC ? Kpad - c * KC : KC;
                        const uint32_t bytes = (uint32_t)klen * BN_TC * 4;
                        mbar_wait(&b_empty[bi], bph ^ 1);
                        mbar_arrive_expect_tx(&b_full[bi], bytes);
                        bulk_g2s(Bs + (size_t)bi * BN_TC * KC, tsrc + (size_t)c * KC * BN_TC, bytes, &b_full[bi]);
                        if (++bi == b_stages) { bi = 0; bph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------ MMA issuer
            int ai = 0, bi = 0, acc = 0;
            uint32_t aph = 0, bph = 0, accph = 0;
            for (long long it = blockIdx.x; it < p.n_items; it += gridDim.x) {
                const int4 w = p.items[it];
                mbar_wait(&a_full[ai], aph);
                tc_fence_after();
                const uint32_t a_base = smem_u32(As + (size_t)ai * A_FLOATS);
                for (int j = w.y; j <= w.z; ++j) {
                    mbar_wait(&acc_empty[acc], accph ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem + (uint32_t)(acc * BN_TC);
                    for (int c = 0; c < nkc; ++c) {
                        mbar_wait(&b_full[bi], bph);
                        tc_fence_after();
                        const uint32_t b_base = smem_u32(Bs + (size_t)bi * BN_TC * KC);
                        const int klen = Kpad - c * KC < KC ? Kpad - c * KC : KC;
                        for (int s = 0; s < klen / 8; ++s) {
                            const uint64_t ad = umma_desc_kmajor(a_base + (uint32_t)(c * KC / 4 + 2 * s) * LBO_A, LBO_A, SBO);
                            const uint64_t bd = umma_desc_kmajor(b_base + (uint32_t)(2 * s) * LBO_B, LBO_B, SBO);
                            mma_tf32(d_tmem, ad, bd, IDESC, (c | s) != 0);
                        }
                        mma_commit(&b_empty[bi]);
                        if (++bi == b_stages) { bi = 0; bph ^= 1; }
                    }
                    mma_commit(&acc_full[acc]);
                    if (++acc == 2) { acc = 0; accph ^= 1; }
                }
                mma_commit(&a_empty[ai]);
                if (++ai == a_stages) { ai = 0; aph ^= 1; }
            }
        }
    } else {
        // ---------------------------------------------------- epilogue
        // 8 warps: warp w reads TMEM lane quadrant (w % 4) (hardware rule) and
        // column half (w - 2) / 4 of the 128 x 256 accumulator.
        const int q = warp & 3;
        const int col0 = ((warp - 2) >> 2) * (BN_TC / 2);
        const int i = q * 32 + lane;
        int acc = 0;
        uint32_t accph = 0;
        for (long long it = blockIdx.x; it < p.n_items; it += gridDim.x) {
            const int4 w = p.items[it];
            const float4 qv = p.qs[(size_t)(w.x - p.tq0) * BM + i];
            const float Q2 = qv.x, Qn = qv.y, Qd = qv.z;
            const int rowid = w.x * BM + i;
            // theta_f covers q = fl32(h + r) vs the exact h + r (|dq_k| <= 2^-24 |q_k|)
            const float thf = p.theta * (1.0f + 2.44140625e-04f) + 2.384185791015625e-07f * Qn;
            for (int j = w.y; j <= w.z; ++j) {
                const float2 tv = p.tstile[j];
                const float Tm = tv.x, Tdm = tv.y;
                // |acc - q.t| <= Qd Tm + Qn Tdm + Qd Tdm + eta (Qn + Qd)(Tm + Tdm)
                const float eb = Qd * Tm + Qn * Tdm + Qd * Tdm + p.eta * (Qn + Qd) * (Tm + Tdm);
                const float sl = 4.76837158203125e-07f * (Qn + Tm) * (Qn + Tm);  // 8u (Qn + Tm)^2, fp32 evaluation
                const float R = thf * thf + 2.0f * eb + sl;
                // candidate iff 2 acc - ||t||^2 >= c
                const float c = Q2 - R - 9.5367431640625e-07f * (Q2 + R);
                mbar_wait(&acc_full[acc], accph);
                tc_fence_after();
                const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN_TC + col0);
                const float* t2row = p.T2 + (size_t)j * BN_TC + col0;
                uint32_t ra[32], rb[32];
                auto process = [&](const uint32_t (&r)[32], int ch) {
                    const float4* t2 = reinterpret_cast<const float4*>(t2row + ch * 32);
                    float m0 = -3.0e38f, m1 = -3.0e38f, m2 = -3.0e38f, m3 = -3.0e38f;
#pragma unroll
                    for (int u4 = 0; u4 < 8; ++u4) {
                        const float4 tt = __ldg(t2 + u4);
                        m0 = fmaxf(m0, fmaf(2.0f, __uint_as_float(r[4 * u4 + 0]), -tt.x));
                        m1 = fmaxf(m1, fmaf(2.0f, __uint_as_float(r[4 * u4 + 1]), -tt.y));
                        m2 = fmaxf(m2, fmaf(2.0f, __uint_as_float(r[4 * u4 + 2]), -tt.z));
                        m3 = fmaxf(m3, fmaf(2.0f, __uint_as_float(r[4 * u4 + 3]), -tt.w));
                    }
                    const float m = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
                    if (__any_sync(0xffffffffu, m >= c)) {
                        uint32_t hit = 0;
#pragma unroll
                        for (int u4 = 0; u4 < 8; ++u4) {
                            const float4 tt = __ldg(t2 + u4);
                            hit |= (uint32_t)(fmaf(2.0f, __uint_as_float(r[4 * u4 + 0]), -tt.x) >= c) << (4 * u4 + 0);
                            hit |= (uint32_t)(fmaf(2.0f, __uint_as_float(r[4 * u4 + 1]), -tt.y) >= c) << (4 * u4 + 1);
                            hit |= (uint32_t)(fmaf(2.0f, __uint_as_float(r[4 * u4 + 2]), -tt.z) >= c) << (4 * u4 + 2);
                            hit |= (uint32_t)(fmaf(2.0f, __uint_as_float(r[4 * u4 + 3]), -tt.w) >= c) << (4 * u4 + 3);
                        }
                        unsigned long long slot = warp_reserve(__popc(hit), p.cand_count);
                        const int colb = j * BN_TC + col0 + ch * 32;
                        while (hit) {
                            const int u = __ffs(hit) - 1;
                            if (slot < (unsigned long long)p.cand_cap) p.cand[slot] = make_int2(rowid, colb + u);
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
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

void launch_tiles_tc(const TileParams& p, int num_sms, cudaStream_t s) {
    if (p.n_items <= 0) return;
    int as, bs, kc;
    int smem = tc_smem_bytes(p.Kpad, &as, &bs, &kc);
    cudaFuncSetAttribute(tiles_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long g = p.n_items < num_sms ? p.n_items : num_sms;
    tiles_tc_kernel<<<(unsigned)g, TC_THREADS, smem, s>>>(p, as, bs, kc);
}

}  // namespace kgc
