// tiles_simt.cu -- K5: surviving-tile distance reduction on the FP32 SIMT
// pipes (SURVEY §8(a) row a6, and the L2 "SIMT" control engine).
//
// L1 (TransE ||h + r - t||_1) has no dense-contraction form, so
// it runs as register-tiled |q - t| accumulation: a 128-query x 128-tail
// tile per CTA, 256 threads, an 8 x 8 micro-tile per thread (FADD + FADD|.|
// per element and k).  Query and tail K-chunks stream through a double
// buffer fed by 1-D bulk TMA copies (shared memory independent of d, two
// CTAs per SM).  A pair whose FP32 distance is within the row's
// rigorous bound (stage kernel) becomes a
// candidate; the FP64 re-check (verify.cu) decides.
#include "common.cuh"

namespace kgc {

constexpr int SIMT_KC = 32;

template <int NORM>
__global__ void __launch_bounds__(256, 2) tiles_simt_kernel(TileParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int Kpad = p.Kpad;
    const int nkc = (Kpad + SIMT_KC - 1) / SIMT_KC;
    // stage s: query chunk [SIMT_KC][BM] followed by tail chunk [SIMT_KC][BN]
    float* St = reinterpret_cast<float*>(smem);
    uint64_t* t_full = reinterpret_cast<uint64_t*>(St + 2 * SIMT_KC * (BM + BN_SIMT));

    const int tid = threadIdx.x;
    const int ty = tid >> 4, tx = tid & 15;
    if (tid == 0) {
        mbar_init(&t_full[0], 1);
        mbar_init(&t_full[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t tph0 = 0, tph1 = 0;

    // Both operands stream in K-chunks (the query chunk is re-read per tail
    // tile from L2), so shared memory does not grow with d.
    auto issue_chunk = [&](int tq, int j, int c, int buf) {
        const int klen = Kpad - c * SIMT_KC < SIMT_KC ? Kpad - c * SIMT_KC : SIMT_KC;
        const uint32_t qbytes = (uint32_t)klen * BM * 4, tbytes = (uint32_t)klen * BN_SIMT * 4;
        float* dst = St + (size_t)buf * SIMT_KC * (BM + BN_SIMT);
        mbar_arrive_expect_tx(&t_full[buf], qbytes + tbytes);
        bulk_g2s(dst, p.Qp + (size_t)(tq - p.tq0) * BM * Kpad + (size_t)c * SIMT_KC * BM, qbytes, &t_full[buf]);
        bulk_g2s(dst + SIMT_KC * BM, p.Tp + (size_t)j * BN_SIMT * Kpad + (size_t)c * SIMT_KC * BN_SIMT, tbytes,
                 &t_full[buf]);
    };

    for (long long it = blockIdx.x; it < p.n_items; it += gridDim.x) {
        const int4 w = p.items[it];
        const int ntile = w.z - w.y + 1;
        const int G = ntile * nkc;
        if (tid == 0) {
            fence_proxy_async_smem();
            issue_chunk(w.x, w.y, 0, 0);
        }
        float thr[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) thr[a] = p.qs[(size_t)(w.x - p.tq0) * BM + ty * 8 + a].w;

        float acc[8][8];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;

        for (int g = 0; g < G; ++g) {
            const int jt = g / nkc, c = g - jt * nkc, buf = g & 1;
            if (tid == 0 && g + 1 < G) {
                const int g1 = g + 1, jt1 = g1 / nkc;
                issue_chunk(w.x, w.y + jt1, g1 - jt1 * nkc, g1 & 1);
            }
            if (buf == 0) { mbar_wait(&t_full[0], tph0); tph0 ^= 1; }
            else          { mbar_wait(&t_full[1], tph1); tph1 ^= 1; }
            const int klen = Kpad - c * SIMT_KC < SIMT_KC ? Kpad - c * SIMT_KC : SIMT_KC;
            const float* qk = St + (size_t)buf * SIMT_KC * (BM + BN_SIMT) + ty * 8;
            const float* tk = St + (size_t)buf * SIMT_KC * (BM + BN_SIMT) + SIMT_KC * BM + tx * 8;
#pragma unroll 4
            for (int k = 0; k < klen; ++k) {
                const float4 qa = *reinterpret_cast<const float4*>(qk + k * BM);
                const float4 qb = *reinterpret_cast<const float4*>(qk + k * BM + 4);
                const float4 ta = *reinterpret_cast<const float4*>(tk + k * BN_SIMT);
                const float4 tb = *reinterpret_cast<const float4*>(tk + k * BN_SIMT + 4);
                const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
                const float tv[8] = {ta.x, ta.y, ta.z, ta.w, tb.x, tb.y, tb.z, tb.w};
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const float df = qv[a] - tv[b];
                        if (NORM == 1) acc[a][b] += fabsf(df);
                        else acc[a][b] = fmaf(df, df, acc[a][b]);
                    }
            }
            if (c == nkc - 1) {
                const int j = w.y + jt;
                unsigned long long hit = 0;
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int b = 0; b < 8; ++b) hit |= (unsigned long long)(acc[a][b] <= thr[a]) << (a * 8 + b);
                if (__any_sync(0xffffffffu, hit != 0)) {
                    // columns past the last tail are padding
                    const int colb = j * BN_SIMT + tx * 8;
#pragma unroll
                    for (int b = 0; b < 8; ++b)
                        if (colb + b >= p.N) hit &= ~(0x0101010101010101ull << b);
                    unsigned long long slot = warp_reserve(__popcll(hit), p.cand_count);
                    while (hit) {
                        const int ab = __ffsll(hit) - 1;
                        if (slot < (unsigned long long)p.cand_cap)
                            p.cand[slot] = make_int2(w.x * BM + ty * 8 + (ab >> 3), colb + (ab & 7));
                        ++slot;
                        hit &= hit - 1;
                    }
                }
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;
            }
            __syncthreads();
            if (tid == 0) fence_proxy_async_smem();
        }
    }
}

void launch_tiles_simt(const TileParams& p, int norm, int num_sms, cudaStream_t s) {
    if (p.n_items <= 0) return;
    const size_t smem = (size_t)2 * SIMT_KC * (BM + BN_SIMT) * 4 + 64;
    auto kern = norm == 1 ? tiles_simt_kernel<1> : tiles_simt_kernel<2>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
    if (per_sm < 1) per_sm = 1;
    long long g = (long long)num_sms * per_sm;
    if (g > p.n_items) g = p.n_items;
    kern<<<(unsigned)g, 256, smem, s>>>(p);
}

}  // namespace kgc
