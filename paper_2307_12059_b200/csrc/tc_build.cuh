// tc_build.cuh -- the builder warps of the tensor-core engines (tiles_tc.cu,
// tiles_tc2.cu): form a 128-row query tile q = fl32(E_h + Rel_r) (connector_1,
// PAPER.md:193) for the sorted queries of a work item directly in the UMMA
// K-major layout in shared memory, plus the row scalars the guard band needs.
#pragma once
#include "common.cuh"

namespace kgc {

// Builder warp wb (0..3) forms rows 32 wb .. 32 wb + 31 of the tile, one row per thread:
// sorted position pos0 + i of relation r (h = qperm[r N + pos]; positions >= N are padding
// rows).  A: element (i, k) at ((k / 4) (BM / 8) + i / 8) 32 + (i % 8) 4 floats (8-row x
// 16-byte core matrices), so for a fixed K-quad the 32 rows of a warp are 512 contiguous
// bytes.  With 16-byte rows (d % 4 == 0, aligned E) the row's K-quads of E go straight into
// their places in A by cp.async -- every piece of the tile in flight at once -- and a second
// pass adds the relation row in place (each thread re-reads only its own pieces, visible
// after its cp.async.wait_group).  Loading through registers kept ~8 loads in flight per
// thread and the build (~15 us per item on c4) left the MMA waiting 19% of the time with one
// query-tile buffer.  qrow[i] = {||q||^2, ||q|| up, ||q - tf32(q)|| up, 0} (3e38 / 0 for
// padding rows): FP32 sums whose error the epilogue covers with (Kpad + 4) 2^-23.
__device__ __forceinline__ void build_query_rows(float* __restrict__ A, float4* __restrict__ qrow,
                                                 const float* __restrict__ E, const float* __restrict__ Rel,
                                                 const int* __restrict__ qperm, long long N, int d, int Kpad, int r,
                                                 long long pos0, int wb, int lane, bool vec4, int l2hint = 0) {
    const int i = 32 * wb + lane;
    const long long pos = pos0 + i;
    const bool valid = pos < N;
    const long long h = valid ? __ldg(qperm + (long long)r * N + pos) : 0;
    const float* e = E + h * d;
    const float* rr = Rel + (long long)r * d;
    const int nq = Kpad >> 2;
    float* Ai = A + (size_t)(i >> 3) * 32 + (i & 7) * 4;  // K-quad kq of row i at Ai + kq (BM / 8) 32
    float s2 = 0.f, sd2 = 0.f;
    auto stats = [&](const float4& q) {
        const float* qq = reinterpret_cast<const float*>(&q);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float rd = qq[c] - __uint_as_float(__float_as_uint(qq[c]) & 0xFFFFE000u);  // exact
            s2 = fmaf(qq[c], qq[c], s2);
            sd2 = fmaf(rd, rd, sd2);
        }
    };
    if (vec4) {
        const int dq = d >> 2;
        // l2hint: the entity rows are read once per item -- evict them first, so the staged
        // tail tiles (re-read for every query tile) keep the L2
        const uint64_t pol = l2hint ? l2_policy_evict_first() : 0;
        for (int kq = 0; kq < nq; ++kq) {
            float* dst = Ai + (size_t)kq * (BM / 8) * 32;
            if (valid && kq < dq) {
                if (l2hint) cp_async16_hint(smem_u32(dst), e + 4 * kq, pol);
                else cp_async16(smem_u32(dst), e + 4 * kq);
            } else {
                *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        cp_async_commit();
        cp_async_wait_n(0);
        if (valid) {
#pragma unroll 4
            for (int kq = 0; kq < dq; ++kq) {
                float4* dst = reinterpret_cast<float4*>(Ai + (size_t)kq * (BM / 8) * 32);
                const float4 a = *dst;
                const float4 b = __ldg(reinterpret_cast<const float4*>(rr + 4 * kq));  // same row for all lanes
                const float4 q = make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                                             __fadd_rn(a.w, b.w));
                *dst = q;
                stats(q);
            }
        }
    } else {
        // unaligned or d % 4 != 0: through registers, 8 K-quads in flight
        for (int kq0 = 0; kq0 < nq; kq0 += 8) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int kq = kq0 + u, k = kq * 4;
                v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (valid && kq < nq) {
                    float* vv = reinterpret_cast<float*>(&v[u]);
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (k + c < d) vv[c] = __fadd_rn(__ldg(e + k + c), __ldg(rr + k + c));
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int kq = kq0 + u;
                if (kq < nq) {
                    stats(v[u]);
                    *reinterpret_cast<float4*>(Ai + (size_t)kq * (BM / 8) * 32) = v[u];
                }
            }
        }
    }
    const float gam = 1.0f + (float)(Kpad + 4) * 1.1920928955078125e-07f;
    qrow[i] = valid ? make_float4(s2, __fsqrt_ru(__fmul_ru(s2, gam)), __fsqrt_ru(__fmul_ru(sd2, gam)), 0.f)
                    : make_float4(3e38f, 0.f, 0.f, 0.f);
}

}  // namespace kgc
