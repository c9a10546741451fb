// pivots.cu -- multi-pivot tile pruning ("tighter tile
// bounds"): K pivots instead of one.  Lemma 1 holds for
// every pivot, so a (query, tail) pair can be a hit only if
// |d(p_k, q) - d(p_k, t)| <= theta for ALL k -- the L_inf bound over pivot
// distances of Chen et al. that the paper cites.  At tile
// granularity: a tile pair survives iff, for every pivot, the key intervals of
// the two tiles are within theta of each other.
//
// Pieces (all on the device, deterministic):
//   pick_pivots   p_0 = zero (or mean) vector, p_1..p_{K-1} = farthest-point
//                 traversal over a fixed sample of tails (a heuristic: it only
//                 decides how much is pruned, never what is returned)
//   mp_keys       d(p_k, x) for every query q = fl32(h + r) and tail, FP32
//                 (relative error <= (d + 4) 2^-24, covered by the test margin)
//   mp_morton     32-bit Hilbert (default) or Morton code of the first 4 quantised
//                 keys, so that the radix-sorted tiles are compact in pivot space
//   mp_boxes      per tile and pivot: [min, max] of its rows' keys
//   mp_count / mp_emit  per query tile: count, then list, the surviving tail tiles
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace kgc {

static inline unsigned grid_for_mp(long long n, int threads, long long cap = 148LL * 64) {
    long long g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

// --------------------------------------------------------------- pivots
template <int NORM>
__device__ __forceinline__ float dist_f32(const float* __restrict__ a, const float* __restrict__ b, int d) {
    float s = 0.f;
    for (int k = 0; k < d; ++k) {
        const float x = a[k] - b[k];
        s = NORM == 1 ? s + fabsf(x) : fmaf(x, x, s);
    }
    return s;  // squared for L2 (monotone: fine for argmax)
}

// Farthest-point traversal over S sample tails held in shared memory (row
// stride d|1: conflict-free across threads), one sample per thread.
template <int NORM>
__global__ void __launch_bounds__(1024) pick_pivots_kernel(const float* __restrict__ E, long long N, int d, int K,
                                                           int S, const double* __restrict__ p0,
                                                           float* __restrict__ P) {
    extern __shared__ float pp_smem[];
    const int st = d | 1;
    float* X = pp_smem;                      // [S][st] sample rows
    float* piv = X + (size_t)S * st;         // [d] current pivot
    __shared__ float bv[32];
    __shared__ int bi[32];
    __shared__ int chosen;
    {   // warp per sample row (lanes over k, coalesced), 4 rows' loads in flight per lane
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int s0 = w * 4; s0 < S; s0 += nw * 4) {
            for (int k0 = 0; k0 < d; k0 += 32) {
                const int k = k0 + lane;
                float v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int sidx = s0 + u;
                    v[u] = (sidx < S && k < d) ? __ldg(E + ((long long)sidx * N / S) * d + k) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (s0 + u < S && k < d) X[(s0 + u) * st + k] = v[u];
            }
        }
    }
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        const float v = p0 ? (float)p0[k] : 0.f;
        P[k] = v;
        piv[k] = v;
    }
    __syncthreads();
    const int sidx = threadIdx.x;
    auto dist_to_piv = [&]() {
        float s8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // 8 independent chains (K rounds are serial)
        if (sidx < S) {
            const float* xr = X + sidx * st;
            int k = 0;
            for (; k + 8 <= d; k += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const float x = xr[k + u] - piv[k + u];
                    s8[u] = NORM == 1 ? s8[u] + fabsf(x) : fmaf(x, x, s8[u]);
                }
            }
            for (; k < d; ++k) {
                const float x = xr[k] - piv[k];
                s8[0] = NORM == 1 ? s8[0] + fabsf(x) : fmaf(x, x, s8[0]);
            }
        }
        return ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));  // squared for L2
    };
    float mind = sidx < S ? dist_to_piv() : -1.f;
    for (int kk = 1; kk < K; ++kk) {
        float best = mind;
        int besti = sidx;
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, besti, o);
            if (ov > best || (ov == best && oi < besti)) { best = ov; besti = oi; }
        }
        if ((threadIdx.x & 31) == 0) { bv[threadIdx.x >> 5] = best; bi[threadIdx.x >> 5] = besti; }
        __syncthreads();
        if (threadIdx.x < 32) {  // warp 0 reduces the per-warp winners (ties: the lower index)
            const int nw = (int)(blockDim.x >> 5);
            float b = threadIdx.x < nw ? bv[threadIdx.x] : -2.f;
            int ix = threadIdx.x < nw ? bi[threadIdx.x] : 0x7fffffff;
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, b, o);
                const int oi = __shfl_xor_sync(0xffffffffu, ix, o);
                if (ov > b || (ov == b && oi < ix)) { b = ov; ix = oi; }
            }
            if (threadIdx.x == 0) chosen = ix;
        }
        __syncthreads();
        float* pk = P + (size_t)kk * d;
        for (int k = threadIdx.x; k < d; k += blockDim.x) {
            const float v = X[chosen * st + k];
            pk[k] = v;
            piv[k] = v;
        }
        __syncthreads();
        if (sidx < S) mind = fminf(mind, dist_to_piv());
        __syncthreads();
    }
}

// ----------------------------------------------------------------- keys
// QUERY: a block walks `nch` chunks of 32 entities against 16 relations (warp
// w: relations w, w + 8; lane = entity); tails: 128 threads, `nch` chunks of
// 128 entities (warp w: entities w*32 + lane).  Key min/max per (segment,
// pivot) are kept per warp across chunks: one atomic pair per warp at the end.
// nch is chosen so the grid still fills the GPU (~8 blocks per SM).
// Row stride (floats) of the entity tile: a multiple of 4 whose quarter is odd,
// so the per-lane float4 row reads of a quarter-warp hit distinct bank groups.
__host__ __device__ inline int mk_stride(int d) {
    int s4 = (d + 3) / 4;
    if ((s4 & 1) == 0) ++s4;
    return 4 * s4;
}
template <int NORM, bool QUERY, int K>
__global__ void __launch_bounds__(256) mp_keys_kernel(const float* __restrict__ E, const float* __restrict__ Rel,
                                                      long long N, long long nseg, int d, int nch,
                                                      const float* __restrict__ P, float* __restrict__ keys,
                                                      unsigned int* minmax, unsigned int* qnmax,
                                                      unsigned int* nonfinite) {
    extern __shared__ __align__(16) float mk_smem[];
    const int S = mk_stride(d);                            // entity row stride (zero padded)
    const int D4 = (d + 3) / 4 * 4;                        // pivot / relation row stride (zero padded)
    constexpr int ENT = QUERY ? 32 : 128;
    constexpr int NU = QUERY ? 2 : 1;                     // relations per warp
    float* Es = mk_smem;                                   // [ENT][S]
    float* Ps = Es + ENT * S;                              // [K][D4]
    float* Rs = Ps + K * D4;                               // [16][D4] (queries)
    const long long r0 = QUERY ? (long long)blockIdx.y * 16 : 0;
    bool bad = false;
    for (int x = threadIdx.x; x < K * D4; x += blockDim.x) {
        const int i = x / D4, k = x % D4;
        Ps[x] = k < d ? P[i * d + k] : 0.f;
    }
    if (QUERY) {
        for (int x = threadIdx.x; x < 16 * D4; x += blockDim.x) {
            const int i = x / D4, k = x % D4;
            const float v = (r0 + i < nseg && k < d) ? Rel[(r0 + i) * d + k] : 0.f;
            bad |= !isfinite(v);
            Rs[x] = v;
        }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float mn[NU][K], mx[NU][K], qn[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        qn[u] = 0.f;
#pragma unroll
        for (int k = 0; k < K; ++k) { mn[u][k] = FLT_MAX; mx[u][k] = 0.f; }
    }
    for (int ch = 0; ch < nch; ++ch) {
        const long long h0 = ((long long)blockIdx.x * nch + ch) * ENT;
        if (h0 >= N) break;
        __syncthreads();
        for (int x = threadIdx.x; x < ENT * S; x += blockDim.x) {
            const int i = x / S, k = x % S;
            const float v = (h0 + i < N && k < d) ? E[(h0 + i) * d + k] : 0.f;
            bad |= !isfinite(v);
            Es[x] = v;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < NU; ++u) {
            const int rl = QUERY ? w + 8 * u : 0;
            const long long r = r0 + rl;
            if (QUERY && r >= nseg) break;
            const int eloc = QUERY ? lane : w * 32 + lane;
            const long long h = h0 + eloc;
            const float* es = Es + eloc * S;
            const float* rs = QUERY ? Rs + rl * D4 : nullptr;
            float acc[K], an = 0.f;  // an: ||fl32(h + r)||_p (squared for L2), queries only
#pragma unroll
            for (int k = 0; k < K; ++k) acc[k] = 0.f;
            // 4 dims per step: float4 loads of the entity row, relation row (broadcast)
            // and every pivot row (broadcast); padding dims are zero on all sides.
            for (int dd = 0; dd < D4; dd += 4) {
                const float4 e4 = *reinterpret_cast<const float4*>(es + dd);
                float4 q4 = e4;
                if (QUERY) {
                    const float4 r4 = *reinterpret_cast<const float4*>(rs + dd);
                    q4 = make_float4(__fadd_rn(e4.x, r4.x), __fadd_rn(e4.y, r4.y), __fadd_rn(e4.z, r4.z),
                                     __fadd_rn(e4.w, r4.w));  // connector_1(h, r) = h + r
                    if (NORM == 1) an = an + fabsf(q4.x) + fabsf(q4.y) + fabsf(q4.z) + fabsf(q4.w);
                    else an = fmaf(q4.w, q4.w, fmaf(q4.z, q4.z, fmaf(q4.y, q4.y, fmaf(q4.x, q4.x, an))));
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const float4 p4 = *reinterpret_cast<const float4*>(Ps + k * D4 + dd);
                    const float x0 = q4.x - p4.x, x1 = q4.y - p4.y, x2 = q4.z - p4.z, x3 = q4.w - p4.w;
                    if (NORM == 1) acc[k] = acc[k] + fabsf(x0) + fabsf(x1) + fabsf(x2) + fabsf(x3);
                    else acc[k] = fmaf(x3, x3, fmaf(x2, x2, fmaf(x1, x1, fmaf(x0, x0, acc[k]))));
                }
            }
            if (h < N) {
                if (QUERY) qn[u] = fmaxf(qn[u], NORM == 2 ? sqrtf(an) : an);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const float key = NORM == 2 ? sqrtf(acc[k]) : acc[k];
                    keys[((size_t)r * N + h) * K + k] = key;
                    mn[u][k] = fminf(mn[u][k], key);
                    mx[u][k] = fmaxf(mx[u][k], key);
                }
            }
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1u);
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        const long long r = r0 + (QUERY ? w + 8 * u : 0);
        if (QUERY && r >= nseg) break;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            float a = mn[u][k], z = mx[u][k];
            for (int o = 16; o > 0; o >>= 1) {
                a = fminf(a, __shfl_xor_sync(0xffffffffu, a, o));
                z = fmaxf(z, __shfl_xor_sync(0xffffffffu, z, o));
            }
            if (lane == 0) {
                atomicMin(&minmax[((size_t)r * K + k) * 2], __float_as_uint(a));
                atomicMax(&minmax[((size_t)r * K + k) * 2 + 1], __float_as_uint(z));
            }
        }
        if (QUERY) {
            float z = qn[u];
            for (int o = 16; o > 0; o >>= 1) z = fmaxf(z, __shfl_xor_sync(0xffffffffu, z, o));
            if (lane == 0) atomicMax(&qnmax[r], __float_as_uint(z));
        }
    }
}

// Query keys d(p_k, fl32(h + r)) for every (h, r): the K1 kernel with the most work
// (N R K d distances, c4: 7.3e9 per join).  Lane = entity (32 per chunk, rows staged in
// shared memory), warp w = NU consecutive relations, so each staged entity element and
// each (negated) pivot element loaded from shared memory serves NU x K distance terms:
// with NU = 4, K = 8 a 4-dim step is 13 shared loads against 72 packed FP32 ops
// (FADD2 / FFMA2: two dims per instruction), where one relation per lane was bound by
// the shared-memory loads.  Per (relation, pivot) key min / max: REDUX per chunk, the
// running value held by lane u K + k.  Same FP32 values up to summation order (the key
// margin covers any order); ||fl32(h + r)||_p per relation for the box widening.
template <int NORM, int K, int NU>
__global__ void __launch_bounds__(256) mp_qkeys_kernel(const float* __restrict__ E, const float* __restrict__ Rel,
                                                       long long N, long long R, int d, int nch,
                                                       const float* __restrict__ P, float* __restrict__ keys,
                                                       unsigned int* minmax, unsigned int* qnmax,
                                                       unsigned int* nonfinite) {
    static_assert(NU * K <= 32, "one lane per (relation, pivot) min/max");
    extern __shared__ __align__(16) float mq_smem[];
    const int S = mk_stride(d);
    const int D4 = (d + 3) / 4 * 4;
    constexpr int RB = 8 * NU;                            // relations per block
    float* Eb = mq_smem;                                  // [2][32][S] entity rows, double-buffered
    float* Ps = Eb + 2 * 32 * S;                          // [K][D4] negated pivots
    float* Rs = Ps + K * D4;                              // [RB][D4] relation rows
    const long long r0 = (long long)blockIdx.y * RB;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    bool bad = false;
    for (int x = threadIdx.x; x < K * D4; x += blockDim.x) {
        const int i = x / D4, k = x % D4;
        Ps[x] = k < d ? -P[i * d + k] : 0.f;
    }
    for (int x = threadIdx.x; x < RB * D4; x += blockDim.x) {
        const int i = x / D4, k = x % D4;
        const float v = (r0 + i < R && k < d) ? Rel[(r0 + i) * d + k] : 0.f;
        bad |= !isfinite(v);
        Rs[x] = v;
    }
    const long long rw = r0 + (long long)w * NU;          // this warp's first relation
    const int nu = rw >= R ? 0 : (int)min((long long)NU, R - rw);
    float run_mn = FLT_MAX, run_mx = 0.f, run_qn = 0.f;  // lane u K + k: (relation rw + u, pivot k)
    // entity rows of chunk `ch` into buffer b: 16-byte cp.async pieces (zero-filled past N) when
    // rows are 16-byte aligned, else plain loads; the next chunk's copies overlap this chunk's math
    const bool vec = (d & 3) == 0 && (reinterpret_cast<uintptr_t>(E) & 15) == 0;
    const int q4 = D4 / 4;
    auto stage = [&](int ch, int b) {
        const long long h0 = ((long long)blockIdx.x * nch + ch) * 32;
        float* Es = Eb + b * 32 * S;
        if (vec) {
            for (int x = threadIdx.x; x < 32 * q4; x += blockDim.x) {
                const int i = x / q4, c = x % q4;
                const bool ok = h0 + i < N;
                const float* src = E + (ok ? (h0 + i) * d + 4 * c : 0);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(Es + i * S + 4 * c)),
                             "l"(src), "r"(ok ? 16 : 0) : "memory");
            }
        } else {
            for (int x = threadIdx.x; x < 32 * S; x += blockDim.x) {
                const int i = x / S, k = x % S;
                Es[x] = (h0 + i < N && k < d) ? E[(h0 + i) * d + k] : 0.f;
            }
        }
        cp_async_commit();
    };
    int nch_here = 0;  // chunks of this block that exist
    while (nch_here < nch && ((long long)blockIdx.x * nch + nch_here) * 32 < N) ++nch_here;
    if (nch_here > 0) stage(0, 0);
    for (int ch = 0; ch < nch_here; ++ch) {
        const long long h0 = ((long long)blockIdx.x * nch + ch) * 32;
        const float* Es = Eb + (ch & 1) * 32 * S;
        __syncthreads();  // every warp is done with the buffer the next chunk goes into
        if (ch + 1 < nch_here) {
            stage(ch + 1, (ch + 1) & 1);
            cp_async_wait_n(1);
        } else {
            cp_async_wait_n(0);
        }
        __syncthreads();  // this chunk's rows have landed (every thread's copies)
        if (vec)  // non-finite check of the pieces this thread copied
            for (int x = threadIdx.x; x < 32 * q4; x += blockDim.x) {
                const float4 v = *reinterpret_cast<const float4*>(Es + (x / q4) * S + 4 * (x % q4));
                bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
            }
        else
            for (int x = threadIdx.x; x < 32 * S; x += blockDim.x) bad |= !isfinite(Es[x]);
        if (nu == 0) continue;
        const long long h = h0 + lane;
        const float* es = Es + lane * S;
        float2 acc[NU][K], an[NU];
#pragma unroll
        for (int u = 0; u < NU; ++u) {
            an[u] = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < K; ++k) acc[u][k] = make_float2(0.f, 0.f);
        }
        for (int dd = 0; dd < D4; dd += 4) {
            const float4 e4 = *reinterpret_cast<const float4*>(es + dd);
            float2 qa[NU], qb[NU];
#pragma unroll
            for (int u = 0; u < NU; ++u) {
                const float4 r4 = *reinterpret_cast<const float4*>(Rs + (w * NU + u) * D4 + dd);
                qa[u] = __fadd2_rn(make_float2(e4.x, e4.y), make_float2(r4.x, r4.y));  // connector_1 = h + r
                qb[u] = __fadd2_rn(make_float2(e4.z, e4.w), make_float2(r4.z, r4.w));
                if (NORM == 2) {
                    an[u] = __ffma2_rn(qa[u], qa[u], an[u]);
                    an[u] = __ffma2_rn(qb[u], qb[u], an[u]);
                } else {
                    an[u].x += fabsf(qa[u].x) + fabsf(qb[u].x);
                    an[u].y += fabsf(qa[u].y) + fabsf(qb[u].y);
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const float4 p4 = *reinterpret_cast<const float4*>(Ps + k * D4 + dd);
                const float2 pa = make_float2(p4.x, p4.y), pb = make_float2(p4.z, p4.w);
#pragma unroll
                for (int u = 0; u < NU; ++u) {
                    const float2 xa = __fadd2_rn(qa[u], pa), xb = __fadd2_rn(qb[u], pb);
                    if (NORM == 2) {
                        acc[u][k] = __ffma2_rn(xa, xa, acc[u][k]);
                        acc[u][k] = __ffma2_rn(xb, xb, acc[u][k]);
                    } else {
                        acc[u][k].x += fabsf(xa.x) + fabsf(xb.x);
                        acc[u][k].y += fabsf(xa.y) + fabsf(xb.y);
                    }
                }
            }
        }
        const bool hv = h < N;
#pragma unroll
        for (int u = 0; u < NU; ++u) {
            if (u >= nu) break;
            const long long r = rw + u;
            float kv[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const float s2 = acc[u][k].x + acc[u][k].y;
                kv[k] = NORM == 2 ? sqrtf(s2) : s2;
            }
            if (hv) {
                float* dst = keys + ((size_t)r * N + h) * K;
                if (K == 8) {
                    reinterpret_cast<float4*>(dst)[0] = make_float4(kv[0], kv[1], kv[2], kv[3]);
                    reinterpret_cast<float4*>(dst)[1] = make_float4(kv[4], kv[5], kv[6], kv[7]);
                } else {
#pragma unroll
                    for (int k = 0; k < K; ++k) dst[k] = kv[k];
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const unsigned bits = __float_as_uint(kv[k]);
                const unsigned m = __reduce_min_sync(0xffffffffu, hv ? bits : 0x7f7fffffu);
                const unsigned z = __reduce_max_sync(0xffffffffu, hv ? bits : 0u);
                if (lane == u * K + k) {
                    run_mn = fminf(run_mn, __uint_as_float(m));
                    run_mx = fmaxf(run_mx, __uint_as_float(z));
                }
            }
            const float qn = NORM == 2 ? sqrtf(an[u].x + an[u].y) : an[u].x + an[u].y;
            const unsigned zq = __reduce_max_sync(0xffffffffu, hv ? __float_as_uint(qn) : 0u);
            if (lane == u) run_qn = fmaxf(run_qn, __uint_as_float(zq));
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1u);
    if (lane < nu * K) {
        const long long r = rw + lane / K;
        const int k = lane % K;
        atomicMin(&minmax[((size_t)r * K + k) * 2], __float_as_uint(run_mn));
        atomicMax(&minmax[((size_t)r * K + k) * 2 + 1], __float_as_uint(run_mx));
    }
    if (lane < nu) atomicMax(&qnmax[rw + lane], __float_as_uint(run_qn));
}

// ------------------------------------------- factorised L2 keys (FP64)
// For L2 the K query keys of (h, r) need not cost K d operations each:
//   ||h + r - p_k||^2 = ||h - p_k||^2 + 2 h.r - 2 r.p_k + ||r||^2
//                     =   A[h][k]     + 2 B[h][r] - 2 C[r][k] + rr[r]
// (TransE's connector_1 = h + r; the same expansion as the relation-factored
// engine).  A is N x K (computed once per join, and for the tails it IS the tail key
// squared), C and rr are R x K and R, and only B = h.r costs d per (h, r): one dot
// product instead of K distances (c4: 7.3e9 -> 9.1e8 terms).  Everything is FP64
// from the fp32 inputs, so the keys are those of the EXACT h + r (not of fl32(h + r)).
// Error (u = 2^-53; products of two floats are exact in FP64; a d-term sum of
// magnitudes M errs by <= (d - 1) u M; A <= (||h|| + ||p||)^2):
//   |D~^2 - D^2| <= (d + 6) u (||h|| + ||r|| + ||p_k||)^2,
// and sqrt is 1/2-Hoelder (|sqrt a - sqrt b| <= sqrt|a - b|, the clamp at 0 only
// shrinks it), so |D~ - D| <= sqrt((d + 6) u) (Hmax + ||r|| + Pmax) =: delta_r.  The
// float key sqrtf(fl32(D~^2)) adds < 2^-23 relative, inside the test margin relm;
// delta_r widens the query boxes of relation r (through qnmax, which mp_boxes scales
// by 2^-23: qnmax[r] = delta_r 2^23 rounded up).  The fl32(h + r) widening of the FP32
// keys is not needed: these keys bound the exact h + r directly.

// Key = sqrt of the FP64 squared distance rounded to float: the hardware approximation
// (sqrt.approx.f32, MUFU; relative error < 2^-22) -- the IEEE sqrtf is a multi-instruction
// sequence that made the 32-pivot key kernel issue-bound (c4: 1.5e8 keys per join).  With the
// fl32 rounding of D^2 (2^-25 in the key) the key errs by < 2^-21 relative, well inside the tile
// test's margin relm = (d + 8) 2^-23 (>= 9 2^-23) per key.
__device__ __forceinline__ float key_sqrt(float x) {
    float y;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Entity terms from the GEMM HP = X P^T (mp_hr_kernel with the pivots as the "relations"):
// A[x][k] = (||x||^2 + ||p_k||^2) - 2 HP[k][x] in FP64 (one thread per row; ||x||^2 from the row,
// ||p_k||^2 per block), the tail keys key_sqrt(fl32(max(A, 0))) with their ranges, max ||x|| and the
// non-finite check.  The expansion cancels: |A~ - A| <= (d + 2) 2^-53 (||x|| + ||p||)^2, so a tail
// key errs by <= delta_t = sqrt((d + 4) 2^-53) (max ||t|| + max ||p||) absolute -- the tail boxes and
// the per-tail test are widened by it (mp_rel_terms_kernel writes it to DevCounters::twid); in the
// query keys the same error is inside delta_r.  Half the FP64 operations of the difference form and
// a register-blocked GEMM for the K d part (c4, K = 64: 0.47 ms for the difference form).
template <int K>
__global__ void __launch_bounds__(256) mp_ent_gemm_kernel(const float* __restrict__ X, long long n, int d,
                                                          const float* __restrict__ P, const double* __restrict__ HP,
                                                          double* __restrict__ A, float* __restrict__ keys,
                                                          unsigned int* minmax, unsigned int* xmax,
                                                          unsigned int* nonfinite) {
    __shared__ double pp[K];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
    for (int k = w; k < K; k += NW) {
        double sp = 0.0;
        for (int x = lane; x < d; x += 32) {
            const double v = (double)__ldg(P + k * d + x);
            sp = fma(v, v, sp);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o);
        if (lane == 0) pp[k] = sp;
    }
    __syncthreads();
    const bool vec = (d & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
    float run_mn[(K + 31) / 32], run_mx[(K + 31) / 32];  // lane k % 32 of word k / 32: pivot k
#pragma unroll
    for (int z = 0; z < (K + 31) / 32; ++z) { run_mn[z] = FLT_MAX; run_mx[z] = 0.f; }
    float run_x = 0.f;
    bool bad = false;
    const long long nblk = (n + blockDim.x - 1) / blockDim.x;
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const long long row = blk * blockDim.x + threadIdx.x;
        const bool rv = row < n;
        double xx = 0.0;
        if (rv) {
            const float* xr = X + row * d;
            if (vec) {
                for (int i = 0; i < d; i += 4) {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(xr + i));
                    bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
                    xx = fma((double)v.x, (double)v.x, xx);
                    xx = fma((double)v.y, (double)v.y, xx);
                    xx = fma((double)v.z, (double)v.z, xx);
                    xx = fma((double)v.w, (double)v.w, xx);
                }
            } else {
                for (int i = 0; i < d; ++i) {
                    const float v = __ldg(xr + i);
                    bad |= !isfinite(v);
                    xx = fma((double)v, (double)v, xx);
                }
            }
        }
        // four pivots at a time: 16-byte stores of A (two double2) and of the keys (float4) -- each
        // thread's row is K contiguous values, so narrower stores touched a line per lane per pivot
        constexpr bool V4 = K % 4 == 0;
#pragma unroll 2
        for (int k0 = 0; k0 < K; k0 += 4) {
            double a[4];
            float key[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = k0 + j;
                a[j] = (rv && k < K) ? (xx + pp[k]) - 2.0 * __ldg(HP + (size_t)k * n + row) : 0.0;
                key[j] = key_sqrt(__double2float_rn(fmax(a[j], 0.0)));
            }
            if (rv && A) {
                if (V4) {
                    reinterpret_cast<double2*>(A + row * K + k0)[0] = make_double2(a[0], a[1]);
                    reinterpret_cast<double2*>(A + row * K + k0)[1] = make_double2(a[2], a[3]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (k0 + j < K) A[row * K + k0 + j] = a[j];
                }
            }
            if (rv && keys) {
                if (V4) {
                    *reinterpret_cast<float4*>(keys + row * K + k0) = make_float4(key[0], key[1], key[2], key[3]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (k0 + j < K) keys[row * K + k0 + j] = key[j];
                }
            }
            if (minmax) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int k = k0 + j;
                    if (k < K) {
                        const unsigned bits = __float_as_uint(key[j]);
                        const unsigned m = __reduce_min_sync(0xffffffffu, rv ? bits : 0x7f7fffffu);
                        const unsigned z = __reduce_max_sync(0xffffffffu, rv ? bits : 0u);
                        if (lane == (k & 31)) {
                            run_mn[k >> 5] = fminf(run_mn[k >> 5], __uint_as_float(m));
                            run_mx[k >> 5] = fmaxf(run_mx[k >> 5], __uint_as_float(z));
                        }
                    }
                }
            }
        }
        if (rv) run_x = fmaxf(run_x, __double2float_ru(sqrt(xx) * (1.0 + 0x1p-40)));
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1u);
    if (minmax) {
#pragma unroll
        for (int z = 0; z < (K + 31) / 32; ++z) {
            const int k = 32 * z + lane;
            if (k < K) {
                atomicMin(&minmax[2 * k], __float_as_uint(run_mn[z]));
                atomicMax(&minmax[2 * k + 1], __float_as_uint(run_mx[z]));
            }
        }
    }
    if (xmax) {
        const unsigned z = __reduce_max_sync(0xffffffffu, __float_as_uint(run_x));
        if (lane == 0) atomicMax(xmax, z);
    }
}


// B[r][h] = E_h . Rel_r for every (h, r) in FP64 (products of two floats are exact, FP64 sums):
// the one d-term quantity per query row.  A register-blocked SIMT GEMM (FP64 tensor cores run at
// the same ~60 FMA/clk/SM on B200): block = 4 warps, tile 128 entities x 32 relations, thread =
// 4 entities x 8 relations (lane: entities 4 lane .. 4 lane + 3, warp w: relations 8 w ..), K-chunks
// of 32 dims staged in shared memory as FP64 (converted once per block); per dim a warp issues
// 32 DFMA against 12 shared-memory wavefronts.
constexpr int HR_BM = 128, HR_BR = 32, HR_KC = 32;
__global__ void __launch_bounds__(128) mp_hr_kernel(const float* __restrict__ E, const float* __restrict__ Rel,
                                                    long long N, long long R, int d, double* __restrict__ B) {
    __shared__ __align__(16) double Es[HR_KC][HR_BM];
    __shared__ __align__(16) double Rs[HR_KC][HR_BR];
    const long long h0 = (long long)blockIdx.x * HR_BM, r0 = (long long)blockIdx.y * HR_BR;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    double acc[4][8];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[a][c] = 0.0;
    const bool vec = (d & 3) == 0 && ((reinterpret_cast<uintptr_t>(E) | reinterpret_cast<uintptr_t>(Rel)) & 15) == 0;
    for (int k0 = 0; k0 < d; k0 += HR_KC) {
        __syncthreads();
        if (vec) {
            // thread = entity row (128 rows), its chunk as 8 independent float4 loads in flight
            // (a dependent-latency loop of 32 scalar loads per thread made the GEMM load-bound);
            // stores Es[k][row]: consecutive threads, consecutive words
            const long long h = h0 + tid;
            float4 v[HR_KC / 4];
#pragma unroll
            for (int j = 0; j < HR_KC / 4; ++j) {
                const int k = k0 + 4 * j;
                v[j] = (h < N && k < d) ? __ldg(reinterpret_cast<const float4*>(E + h * d + k))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int j = 0; j < HR_KC / 4; ++j) {
                Es[4 * j][tid] = (double)v[j].x;
                Es[4 * j + 1][tid] = (double)v[j].y;
                Es[4 * j + 2][tid] = (double)v[j].z;
                Es[4 * j + 3][tid] = (double)v[j].w;
            }
            // relations: 32 rows x 8 float4, two per thread
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int x = tid + 128 * u, i = x >> 3, j = x & 7;
                const long long r = r0 + i;
                const int k = k0 + 4 * j;
                const float4 w4 = (r < R && k < d) ? __ldg(reinterpret_cast<const float4*>(Rel + r * d + k))
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                Rs[4 * j][i] = (double)w4.x;
                Rs[4 * j + 1][i] = (double)w4.y;
                Rs[4 * j + 2][i] = (double)w4.z;
                Rs[4 * j + 3][i] = (double)w4.w;
            }
        } else {
            for (int x = tid; x < HR_BM * HR_KC; x += 128) {
                const int i = x % HR_BM, k = x / HR_BM;
                const long long h = h0 + i;
                Es[k][i] = (h < N && k0 + k < d) ? (double)__ldg(E + h * d + k0 + k) : 0.0;
            }
            for (int x = tid; x < HR_BR * HR_KC; x += 128) {
                const int i = x % HR_BR, k = x / HR_BR;
                const long long r = r0 + i;
                Rs[k][i] = (r < R && k0 + k < d) ? (double)__ldg(Rel + r * d + k0 + k) : 0.0;
            }
        }
        __syncthreads();
#pragma unroll 4
        for (int k = 0; k < HR_KC; ++k) {
            const double2 e01 = *reinterpret_cast<const double2*>(&Es[k][4 * lane]);
            const double2 e23 = *reinterpret_cast<const double2*>(&Es[k][4 * lane + 2]);
            const double ev[4] = {e01.x, e01.y, e23.x, e23.y};
            double rv[8];
#pragma unroll
            for (int c = 0; c < 8; c += 2) {
                const double2 r2 = *reinterpret_cast<const double2*>(&Rs[k][8 * w + c]);
                rv[c] = r2.x;
                rv[c + 1] = r2.y;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[a][c] = fma(ev[a], rv[c], acc[a][c]);
        }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const long long r = r0 + 8 * w + c;
        if (r >= R) break;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const long long h = h0 + 4 * lane + a;
            if (h < N) B[r * N + h] = acc[a][c];
        }
    }
}

// Per relation: Cg[r][k] = 2 r.p_k (k < K), Cg[r][K] = ||r||^2 (FP64), the non-finite check of
// Rel, and the box widening delta_r of the factorised keys (qnmax[r] = delta_r 2^23, rounded up;
// needs max ||h|| from mp_ent_kernel).  One warp per (relation, term).
__global__ void mp_rel_terms_kernel(const float* __restrict__ Rel, long long R, int d, int K,
                                    const float* __restrict__ P, double* __restrict__ Cg,
                                    const unsigned int* __restrict__ hmax, unsigned int* qnmax,
                                    unsigned int* nonfinite, const unsigned int* __restrict__ tmax,
                                    unsigned int* twid) {
    __shared__ double pmax_s;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
    if (threadIdx.x == 0) pmax_s = 0.0;
    __syncthreads();
    if (blockIdx.x == 0) {  // max ||p_k||
        for (int k = w; k < K; k += NW) {
            double sp = 0.0;
            for (int x = lane; x < d; x += 32) {
                const double v = (double)__ldg(P + k * d + x);
                sp = fma(v, v, sp);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o);
            if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&pmax_s), __double_as_longlong(sp));
        }
    }
    __syncthreads();
    bool bad = false;
    const long long nt = R * (K + 1);
    for (long long t = (long long)blockIdx.x * NW + w; t < nt; t += (long long)gridDim.x * NW) {
        const long long r = t / (K + 1);
        const int k = (int)(t - r * (K + 1));
        double sum = 0.0;
        for (int x = lane; x < d; x += 32) {
            const float rv = __ldg(Rel + r * d + x);
            bad |= !isfinite(rv);
            const double dr = (double)rv;
            sum = fma(dr, k < K ? (double)__ldg(P + k * d + x) : dr, sum);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) Cg[t] = k < K ? 2.0 * sum : sum;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1u);
    if (blockIdx.x == 0) {
        // delta_r needs max ||p|| of every pivot: block 0 only (it computed pmax_s), after the
        // terms above are globally visible -- recompute ||r|| here instead of reading Cg
        const double pm = sqrt(pmax_s) * (1.0 + 0x1p-40);
        if (threadIdx.x == 0 && twid) {  // tail-key bound delta_t of the GEMM-form entity terms
            const double dt = sqrt((double)(d + 4) * 0x1p-53) * (1.0 + 0x1p-20) *
                              ((double)__uint_as_float(*tmax) + pm);
            atomicMax(twid, __float_as_uint(__double2float_ru(dt * 0x1p23)));
        }
        for (long long r = w; r < R; r += NW) {
            double rr = 0.0;
            for (int x = lane; x < d; x += 32) {
                const double v = (double)__ldg(Rel + r * d + x);
                rr = fma(v, v, rr);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) rr += __shfl_xor_sync(0xffffffffu, rr, o);
            if (lane == 0) {
                const double S1 = (double)__uint_as_float(*hmax) + sqrt(rr) * (1.0 + 0x1p-40) + pm;
                const double delta = sqrt((double)(d + 8) * 0x1p-53) * (1.0 + 0x1p-20) * S1;
                atomicMax(&qnmax[r], __float_as_uint(__double2float_ru(delta * 0x1p23)));
            }
        }
    }
}

// One L2 query key from the factorisation terms (the only place the formula is written, so
// the materialised keys, the Hilbert keys and the boxes computed on the fly agree bit for bit).
__device__ __forceinline__ float mp_key_l2(double a, double b2, double c) {
    return key_sqrt(__double2float_rn(fmax((a + b2) - c, 0.0)));
}

// Query keys from the factorisation: thread = entity h (A[h][k] from L2), loop over a chunk of
// relations: D~^2_k = (A[h][k] + (2 B[r][h] + ||r||^2)) - 2 r.p_k, key = mp_key_l2.  Writes the
// first KO keys of every (r, h) row (KO = min(K, 4): the Hilbert-order pivots; KO = K: the full
// keys, only for kgc_inspect), KO contiguous floats per row, and (optionally) per (relation,
// pivot) key ranges for k < KO: warp REDUX, shared-memory atomics, one global atomic per block.
constexpr int QK_RCH = 8;  // relations per block
template <int K, int KO>
__global__ void __launch_bounds__(256) mp_qkeys_fact_kernel(const double* __restrict__ B, const double* __restrict__ A,
                                                            const double* __restrict__ Cg, long long N, long long R,
                                                            float* __restrict__ keys, unsigned int* minmax) {
    __shared__ unsigned int smn[QK_RCH][KO], smx[QK_RCH][KO];
    __shared__ double cs[QK_RCH][K + 1];
    const long long r0 = (long long)blockIdx.y * QK_RCH;
    const int nr = (int)min((long long)QK_RCH, R - r0);
    for (int x = threadIdx.x; x < QK_RCH * KO; x += blockDim.x) {
        smn[x / KO][x % KO] = 0x7f7fffffu;
        smx[x / KO][x % KO] = 0u;
    }
    for (int x = threadIdx.x; x < nr * (K + 1); x += blockDim.x) cs[x / (K + 1)][x % (K + 1)] = Cg[r0 * (K + 1) + x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long h = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool hv = h < N;
    for (int u = 0; u < nr; ++u) {
        const long long r = r0 + u;
        const double b2 = 2.0 * (hv ? __ldg(B + r * N + h) : 0.0) + cs[u][K];
        float* dst = keys + ((size_t)r * N + h) * KO;
#pragma unroll
        for (int k0 = 0; k0 < KO; k0 += 4) {
            float kv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = k0 + j < KO ? k0 + j : 0;
                kv[j] = (k0 + j < KO && hv) ? mp_key_l2(__ldg(A + h * K + k), b2, cs[u][k]) : 0.f;
            }
            if (hv) {
                if (KO % 4 == 0) {
                    *reinterpret_cast<float4*>(dst + k0) = make_float4(kv[0], kv[1], kv[2], kv[3]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (k0 + j < KO) dst[k0 + j] = kv[j];
                }
            }
            if (minmax && k0 < MP_SORT_PIVOTS) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int k = k0 + j;
                    if (k < KO && k < MP_SORT_PIVOTS) {
                        const unsigned bits = __float_as_uint(kv[j]);
                        const unsigned m = __reduce_min_sync(0xffffffffu, hv ? bits : 0x7f7fffffu);
                        const unsigned z = __reduce_max_sync(0xffffffffu, hv ? bits : 0u);
                        if (lane == 0) {
                            atomicMin(&smn[u][k], m);
                            atomicMax(&smx[u][k], z);
                        }
                    }
                }
            }
        }
    }
    if (!minmax) return;
    __syncthreads();
    for (int x = threadIdx.x; x < nr * KO; x += blockDim.x) {
        const int u = x / KO, k = x % KO;
        atomicMin(&minmax[((r0 + u) * KO + k) * 2], smn[u][k]);
        atomicMax(&minmax[((r0 + u) * KO + k) * 2 + 1], smx[u][k]);
    }
}

// Query-tile boxes straight from the factorisation terms (no materialised query keys: c5 at 64
// pivots would need 25.6 GB of them): one warp per query tile, lanes over PIVOTS (lane k holds
// pivot k, k + 32), rows of the tile one after the other (h = qperm; each row's A[h][.] is one
// coalesced read).  The key is monotone in D~^2 (fl32 rounding, the clamp at 0 and sqrt are), so
// the box is the key of the min / max FP64 D~^2 -- two conversions and square roots per (tile,
// pivot) instead of one per (row, pivot); widened by delta_r (qnmax[r] 2^-23).
template <int K>
__global__ void mp_qboxes_fact_kernel(const unsigned int* __restrict__ perm, const double* __restrict__ B,
                                      const double* __restrict__ A, const double* __restrict__ Cg, long long N,
                                      long long R, int ROWS, int QT, const unsigned int* __restrict__ qnmax,
                                      float* __restrict__ bmin, float* __restrict__ bmax) {
    constexpr int KL = (K + 31) / 32;  // pivots per lane
    const int lane = threadIdx.x & 31;
    const long long nt = R * QT;
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < nt;
         w += ((long long)gridDim.x * blockDim.x) >> 5) {
        const long long r = w / QT, tl = w - r * QT;
        const long long b = tl * ROWS, e = min(N, b + ROWS);
        const double* cr = Cg + r * (K + 1);
        const double rr = __ldg(cr + K);
        double c[KL], lo[KL], hi[KL];
#pragma unroll
        for (int j = 0; j < KL; ++j) {
            const int k = lane + 32 * j;
            c[j] = k < K ? __ldg(cr + k) : 0.0;
            lo[j] = 1e300;
            hi[j] = -1e300;
        }
        const unsigned int* pr = perm + r * N;
        const double* br = B + r * N;
#pragma unroll 4
        for (long long i = b; i < e; ++i) {
            const long long h = __ldg(pr + i);
            const double b2 = 2.0 * __ldg(br + h) + rr;
            const double* ah = A + h * K;
#pragma unroll
            for (int j = 0; j < KL; ++j) {
                const int k = lane + 32 * j;
                if (k < K) {
                    const double q2 = (__ldg(ah + k) + b2) - c[j];  // the operation order of mp_key_l2
                    lo[j] = fmin(lo[j], q2);
                    hi[j] = fmax(hi[j], q2);
                }
            }
        }
        const float m = __fmul_ru(__uint_as_float(qnmax[r]), 1.1920928955078125e-07f);  // 2^-23
#pragma unroll
        for (int j = 0; j < KL; ++j) {
            const int k = lane + 32 * j;
            if (k < K && e > b) {
                bmin[w * K + k] = __fsub_rd(key_sqrt(__double2float_rn(fmax(lo[j], 0.0))), m);
                bmax[w * K + k] = __fadd_ru(key_sqrt(__double2float_rn(fmax(hi[j], 0.0))), m);
            }
        }
    }
}


__global__ void mp_init_minmax_kernel(unsigned int* mm, long long n, unsigned int* qnmax, long long nseg) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        mm[2 * i] = __float_as_uint(FLT_MAX);
        mm[2 * i + 1] = 0u;
    }
    if (qnmax)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nseg; i += (long long)gridDim.x * blockDim.x)
            qnmax[i] = 0u;
}

// -------------------------------------------------------------- Morton
// The sort code of one row from its first MP_SORT_PIVOTS keys: quantised to `bits` per pivot over
// the segment's key range, Hilbert order (Skilling's axes-to-transpose: Gray code + rotations,
// then the bit interleave) or Morton order.
__device__ __forceinline__ unsigned long long mp_code(const float* __restrict__ kr, const unsigned int* __restrict__ mm,
                                                      int K, int bits, int hilbert) {
    const float scale_max = (float)((1u << bits) - 1);
    unsigned q[MP_SORT_PIVOTS];
#pragma unroll
    for (int k = 0; k < MP_SORT_PIVOTS; ++k) {
        q[k] = 0;
        if (k < K) {
            const float lo = __uint_as_float(mm[k * 2]);
            const float hi = __uint_as_float(mm[k * 2 + 1]);
            const float rg = hi - lo;
            if (rg > 0.f) {
                float x = (kr[k] - lo) / rg * scale_max;
                x = fminf(fmaxf(x, 0.f), scale_max);
                q[k] = (unsigned)x;
            }
        }
    }
    const int Ks = K < MP_SORT_PIVOTS ? K : MP_SORT_PIVOTS;  // order by the first pivots only
    if (hilbert && Ks > 1) {
        // consecutive Hilbert codes are adjacent cells, so tiles are more compact
        const unsigned M = 1u << (bits - 1);
        for (unsigned Q = M; Q > 1; Q >>= 1) {
            const unsigned P = Q - 1;
#pragma unroll
            for (int k = 0; k < MP_SORT_PIVOTS; ++k) {
                if (k >= Ks) continue;
                if (q[k] & Q) {
                    q[0] ^= P;
                } else {
                    const unsigned tt = (q[0] ^ q[k]) & P;
                    q[0] ^= tt;
                    q[k] ^= tt;
                }
            }
        }
#pragma unroll
        for (int k = 1; k < MP_SORT_PIVOTS; ++k)
            if (k < Ks) q[k] ^= q[k - 1];
        unsigned tt = 0;
        for (unsigned Q = M; Q > 1; Q >>= 1)
            if (q[Ks - 1] & Q) tt ^= Q - 1;
#pragma unroll
        for (int k = 0; k < MP_SORT_PIVOTS; ++k)
            if (k < Ks) q[k] ^= tt;
    }
    unsigned long long c = 0;
    for (int b = bits - 1; b >= 0; --b)
#pragma unroll
        for (int k = 0; k < MP_SORT_PIVOTS; ++k)
            if (k < Ks) c = (c << 1) | ((q[k] >> b) & 1u);
    return c;
}

__global__ void mp_morton_kernel(const float* __restrict__ keys, const unsigned int* __restrict__ minmax, long long nseg,
                                 long long L, int K, int bits, unsigned int* __restrict__ code,
                                 unsigned int* __restrict__ idx, int hilbert) {
    const long long n = nseg * L;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
        const long long s = t / L, i = t - s * L;
        code[t] = (unsigned int)mp_code(keys + t * K, minmax + s * K * 2, K, bits, hilbert);  // <= 32 bits
        idx[t] = (unsigned)i;
    }
}

// Short segments (L <= MS_L): code and stable LSD sort of a whole segment in one CTA's shared
// memory (32-bit codes and 16-bit row indices, 8-bit digits, per-warp digit ranks by
// match_any) -- instead of a global code array and 4 x (histogram, scan, scatter) launches.  Same
// order as the multi-kernel path (stable by code, ties by index).  c3: 1345 segments of 14951.
constexpr int MS_L = 16384, MS_NT = 512;
__global__ void __launch_bounds__(MS_NT) mp_sort_small_kernel(const float* __restrict__ keys,
                                                              const unsigned int* __restrict__ minmax, long long L,
                                                              int K, int bits, int hilbert, int* __restrict__ perm) {
    extern __shared__ __align__(16) unsigned int ms_smem[];
    constexpr int NW = MS_NT / 32;
    unsigned int* ka = ms_smem;                                        // [L] codes
    unsigned int* kb = ka + L;                                         // [L]
    int* hist = reinterpret_cast<int*>(kb + L);                        // [256]
    int* wcnt = hist + 256;                                            // [NW][257]
    unsigned short* va = reinterpret_cast<unsigned short*>(wcnt + NW * 257);  // [L] indices
    unsigned short* vb = va + L;                                       // [L]
    const long long s = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int Ks = K < MP_SORT_PIVOTS ? K : MP_SORT_PIVOTS;
    for (int i = tid; i < L; i += MS_NT) {
        ka[i] = (unsigned)mp_code(keys + (s * L + i) * K, minmax + s * K * 2, K, bits, hilbert);
        va[i] = (unsigned short)i;
    }
    const int passes = (bits * Ks + 7) / 8;
    for (int pass = 0; pass < passes; ++pass) {
        const unsigned int* src = (pass & 1) ? kb : ka;
        unsigned int* dst = (pass & 1) ? ka : kb;
        const unsigned short* vs = (pass & 1) ? vb : va;
        unsigned short* vd = (pass & 1) ? va : vb;
        const int shift = 8 * pass;
        if (tid < 256) hist[tid] = 0;
        __syncthreads();
        for (int i = tid; i < L; i += MS_NT) atomicAdd(&hist[(src[i] >> shift) & 255u], 1);
        __syncthreads();
        if (w == 0) {  // exclusive scan of the 256 bins
            int v[8], t = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) { v[u] = hist[lane * 8 + u]; t += v[u]; }
            int incl = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int run = incl - t;
#pragma unroll
            for (int u = 0; u < 8; ++u) { hist[lane * 8 + u] = run; run += v[u]; }
        }
        __syncthreads();
        for (int base = 0; base < L; base += MS_NT) {
            const int i = base + tid;
            const bool valid = i < L;
            const unsigned int x = valid ? src[i] : 0u;
            const unsigned short xv = valid ? vs[i] : 0;
            const int dg = valid ? (int)((x >> shift) & 255u) : 256;
            for (int z = tid; z < NW * 257; z += MS_NT) wcnt[z] = 0;
            __syncthreads();
            const unsigned peers = __match_any_sync(0xffffffffu, dg);
            const int lrank = __popc(peers & lanemask_lt());
            if (valid && lrank == 0) wcnt[w * 257 + dg] = __popc(peers);
            __syncthreads();
            if (tid < 256) {  // per digit: warp offsets in warp order, then advance the running offset
                int run = hist[tid];
#pragma unroll
                for (int ww = 0; ww < NW; ++ww) {
                    const int c = wcnt[ww * 257 + tid];
                    wcnt[ww * 257 + tid] = run;
                    run += c;
                }
                hist[tid] = run;
            }
            __syncthreads();
            if (valid) {
                const int o = wcnt[w * 257 + dg] + lrank;
                dst[o] = x;
                vd[o] = xv;
            }
            __syncthreads();
        }
    }
    const unsigned short* vf = (passes & 1) ? vb : va;
    for (int i = tid; i < L; i += MS_NT) perm[s * L + i] = (int)vf[i];
}

// Sort order of nseg segments of L rows by their code; true when the short-segment kernel did it
// (perm written), false when the caller must run the global code + radix path.
bool launch_mp_sort_small(const float* keys, const unsigned int* minmax, long long nseg, long long L, int K, int bits,
                          int* perm, cudaStream_t s) {
    if (L > MS_L || L < 1) return false;
    const char* e = kgc_knob("KGC_HILBERT");
    const int hilbert = e ? atoi(e) : 1;
    const size_t smem = (size_t)L * 12 + (256 + (MS_NT / 32) * 257) * 4;
    cudaFuncSetAttribute(mp_sort_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mp_sort_small_kernel<<<(unsigned)nseg, MS_NT, smem, s>>>(keys, minmax, L, K, bits, hilbert, perm);
    return true;
}

// --------------------------------------------------------------- boxes
// One warp per tile: [min, max] per pivot of the keys of its (sorted) rows.
// Query keys are distances from q^ = fl32(h + r), not from h + r: by the triangle
// inequality |d(p, q^) - d(p, h + r)| <= ||q^ - (h + r)||_p <= 2^-24 ||h + r||_p, a term that
// does not scale with the key (embeddings with a common offset far larger than their
// spread make keys small and ||h + r|| large).  So every query box is widened by
// 2^-23 max_h ||q^||_p of its relation (qnmax; the factor 2 covers the FP32 norm and
// the 2^-24 -> ||q^|| vs ||h + r|| conversion), rounded outward: the boxes then bound
// the keys of the exact h + r, and every test built on them stays lossless.
// transpose = 1 (tail boxes): bmin[k * (nseg ntile) + tile], so the tile test's lanes (one tail
// tile each) read consecutive words per pivot.
__global__ void mp_boxes_kernel(const float* __restrict__ keys, const unsigned int* __restrict__ perm, long long nseg,
                                long long L, int ROWS, int ntile, int K, float* __restrict__ bmin,
                                float* __restrict__ bmax, const unsigned int* __restrict__ qnmax, int transpose) {
    constexpr int KC = 16;  // pivots per pass over the tile's rows (registers)
    const int lane = threadIdx.x & 31;
    const long long nt = nseg * ntile;
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < nt;
         w += ((long long)gridDim.x * blockDim.x) >> 5) {
        const long long s = w / ntile, tl = w - s * ntile;
        const long long b = tl * ROWS, e = min(L, b + ROWS);
        for (int k0 = 0; k0 < K; k0 += KC) {
            float mn[KC], mx[KC];
#pragma unroll
            for (int k = 0; k < KC; ++k) { mn[k] = FLT_MAX; mx[k] = -FLT_MAX; }
            for (long long i = b + lane; i < e; i += 32) {
                const float* kr = keys + ((size_t)s * L + perm[s * L + i]) * K + k0;
                if ((K & 3) == 0) {  // 16-byte rows: one float4 per 4 pivots
#pragma unroll
                    for (int k = 0; k < KC; k += 4)
                        if (k0 + k < K) {
                            const float4 v = __ldg(reinterpret_cast<const float4*>(kr + k));
                            mn[k] = fminf(mn[k], v.x); mx[k] = fmaxf(mx[k], v.x);
                            mn[k + 1] = fminf(mn[k + 1], v.y); mx[k + 1] = fmaxf(mx[k + 1], v.y);
                            mn[k + 2] = fminf(mn[k + 2], v.z); mx[k + 2] = fmaxf(mx[k + 2], v.z);
                            mn[k + 3] = fminf(mn[k + 3], v.w); mx[k + 3] = fmaxf(mx[k + 3], v.w);
                        }
                } else {
#pragma unroll
                    for (int k = 0; k < KC; ++k)
                        if (k0 + k < K) { mn[k] = fminf(mn[k], kr[k]); mx[k] = fmaxf(mx[k], kr[k]); }
                }
            }
#pragma unroll
            for (int kk = 0; kk < KC; ++kk) {
                const int k = k0 + kk;
                if (k < K) {
                    float a = mn[kk], z = mx[kk];
                    for (int o = 16; o > 0; o >>= 1) {
                        a = fminf(a, __shfl_xor_sync(0xffffffffu, a, o));
                        z = fmaxf(z, __shfl_xor_sync(0xffffffffu, z, o));
                    }
                    if (qnmax) {
                        const float m = __fmul_ru(__uint_as_float(qnmax[s]), 1.1920928955078125e-07f);  // 2^-23
                        a = __fsub_rd(a, m);
                        z = __fadd_ru(z, m);
                    }
                    if (lane == 0) {
                        const long long o = transpose ? k * nt + w : w * K + k;
                        bmin[o] = a;
                        bmax[o] = z;
                    }
                }
            }
        }
    }
}

// ------------------------------------------------------ test and lists
// Tile pair survives iff for every pivot k the intervals are within th_k,
// th_k = theta (1 + 2^-14) + relm (|qmax_k| + |tmax_k|), relm covering the
// FP32 key error.
// KM: register-array size (MP_MAX for the tile test, MP_G for the per-tail test).  Pivots are
// tested 8 at a time; the lane stops at the first group that fails (most tile pairs fail on the
// first pivots: with 32 pivots the loads of the later boxes are mostly skipped).
template <int KM>
__device__ __forceinline__ bool mp_survives(const float* qmn, const float* qmx, const float* __restrict__ tmn,
                                            const float* __restrict__ tmx, int K, float theta, float relm,
                                            int ts = 1) {
    bool ok = true;
#pragma unroll
    for (int k0 = 0; k0 < KM; k0 += 8) {
        if (k0 >= K || !ok) break;
#pragma unroll
        for (int k = k0; k < k0 + 8; ++k) {
            if (k < K) {
                const float tz = tmx[k * ts], ta = tmn[k * ts];  // ts: pivot stride of the tail box
                const float th = theta * (1.0f + 6.103515625e-05f) + relm * (fabsf(qmx[k]) + fabsf(tz));
                ok &= !(tz < qmn[k] - th || ta > qmx[k] + th);
            }
        }
    }
    return ok;
}

// One warp per query tile, lanes over tail tiles; the block's 16 query tiles share the tail
// boxes, staged in shared memory in chunks of CT = 4096 / K tail tiles ([pivot][tile]: consecutive
// lanes read consecutive words), and each warp's query box sits in shared memory too (up to 64
// pivots) -- the per-lane global loads of the boxes (a dependent L2 round trip per 32 tail tiles)
// made the many-pivot test latency-bound.
constexpr int MC_W = 32;
// tail tiles per staged chunk: 4096 / K rounded down to 32 (32 KB of boxes; 12288 / K measured slower on c5)
__host__ __device__ inline int mc_chunk(int K) { return 4096 / K / 32 * 32; }
__global__ void __launch_bounds__(32 * MC_W) mp_count_kernel(const float* __restrict__ qbmin,
                                                             const float* __restrict__ qbmax,
                                                             const float* __restrict__ tbmin,
                                                             const float* __restrict__ tbmax, long long nq, int TT,
                                                             int K, float theta, float relm, int prune, int2* ranges,
                                                             long long* cost, unsigned int* __restrict__ bits) {
    extern __shared__ float mc_smem[];
    const int CT = mc_chunk(K);                        // tail tiles per chunk (a multiple of 32)
    float* sbn = mc_smem;                              // [K][CT]
    float* sbx = sbn + K * CT;                         // [K][CT]
    float* sq = sbx + K * CT;                          // [MC_W][2][K] query boxes
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int TW = (TT + 31) >> 5;
    float* qmn = sq + w * 2 * K;
    float* qmx = qmn + K;
    for (long long qb = (long long)blockIdx.x * MC_W; qb < nq; qb += (long long)gridDim.x * MC_W) {
        const long long q = qb + w;
        const bool qv = q < nq;
        for (int k = lane; k < K; k += 32) {
            qmn[k] = qv ? qbmin[q * K + k] : 0.f;
            qmx[k] = qv ? qbmax[q * K + k] : 0.f;
        }
        __syncwarp();
        int c = 0;
        if (prune) {
            for (int j0 = 0; j0 < TT; j0 += CT) {
                __syncthreads();  // the previous chunk is consumed
                for (int x = threadIdx.x; x < K * CT; x += blockDim.x) {
                    const int k = x / CT, jj = x - k * CT;
                    const bool in = j0 + jj < TT;
                    sbn[x] = in ? tbmin[(size_t)k * TT + j0 + jj] : 0.f;
                    sbx[x] = in ? tbmax[(size_t)k * TT + j0 + jj] : 0.f;
                }
                __syncthreads();
                if (!qv) continue;
                for (int jj0 = 0; jj0 < CT && j0 + jj0 < TT; jj0 += 32) {
                    const int jj = jj0 + lane;
                    bool ok = j0 + jj < TT;
                    // pivots in groups of 8, the lane stops at the first group that fails
                    for (int k0 = 0; k0 < K && ok; k0 += 8) {
#pragma unroll
                        for (int k = k0; k < k0 + 8; ++k) {
                            if (k < K) {
                                const float tz = sbx[k * CT + jj], ta = sbn[k * CT + jj];
                                const float th = theta * (1.0f + 6.103515625e-05f) + relm * (fabsf(qmx[k]) + fabsf(tz));
                                ok &= !(tz < qmn[k] - th || ta > qmx[k] + th);
                            }
                        }
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, ok);
                    c += __popc(m);
                    if (bits && lane == 0) bits[q * TW + ((j0 + jj0) >> 5)] = m;  // mp_emit expands these
                }
            }
        } else {
            c = TT;
        }
        if (qv && lane == 0) {
            ranges[q] = make_int2(0, c - 1);  // positions in this query tile's list
            cost[q] = c;
        }
        __syncwarp();
    }
}

// MASKS: expand mp_count's survival masks (the usual case, few registers); else repeat the box
// tests (masks past 2 GiB).
template <bool MASKS>
__global__ void mp_emit_kernel(const float* __restrict__ qbmin, const float* __restrict__ qbmax,
                               const float* __restrict__ tbmin, const float* __restrict__ tbmax,
                               const long long* __restrict__ cum, const DevCounters* ctr, int TT, int K, float theta,
                               float relm, int prune, int* __restrict__ list, const unsigned int* __restrict__ bits) {
    const int tq0 = ctr->tq_begin, tq1 = ctr->tq_end;
    if (tq0 >= tq1) return;
    const long long base = cum[tq0];
    const int lane = threadIdx.x & 31;
    if constexpr (MASKS) {  // the survival masks mp_count wrote: expand, no second pass over the boxes
        const int TW = (TT + 31) >> 5;
        for (long long q = tq0 + ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5); q < tq1;
             q += ((long long)gridDim.x * blockDim.x) >> 5) {
            long long o = cum[q] - base;
            for (int w0 = 0; w0 < TW; w0 += 32) {
                const int wi = w0 + lane;
                const unsigned m = wi < TW ? __ldg(bits + q * TW + wi) : 0u;
                const int n = __popc(m);
                int incl = n;  // exclusive prefix of the words' counts across lanes (ascending j)
#pragma unroll
                for (int x = 1; x < 32; x <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, x);
                    if (lane >= x) incl += y;
                }
                long long pos = o + incl - n;
                unsigned mm = m;
                while (mm) {
                    const int b = __ffs(mm) - 1;
                    list[pos++] = (wi << 5) + b;
                    mm &= mm - 1;
                }
                o += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
    } else {
    for (long long q = tq0 + ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5); q < tq1;
         q += ((long long)gridDim.x * blockDim.x) >> 5) {
        float qmn[MP_MAX], qmx[MP_MAX];
#pragma unroll
        for (int k = 0; k < MP_MAX; ++k)
            if (k < K) { qmn[k] = qbmin[q * K + k]; qmx[k] = qbmax[q * K + k]; }
        long long o = cum[q] - base;
        for (int j0 = 0; j0 < TT; j0 += 32) {
            const int j = j0 + lane;
            const bool ok = j < TT && (!prune || mp_survives<MP_MAX>(qmn, qmx, tbmin + j, tbmax + j, K, theta,
                                                                     relm, TT));
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            if (ok) list[o + __popc(m & lanemask_lt())] = j;  // ascending j order
            o += __popc(m);
        }
    }
    }
}


// ------------------------------------------- gathered tails (element level)
// Finer than tile pruning on the tail side: inside every surviving tile pair,
// a single tail t can still be dropped when its own K keys fail the L_inf test
// against the query tile's box (Lemma 1 for every row of the query tile:
// |d(p_k, q) - d(p_k, t)| > theta for some k and all q in the tile).  The
// surviving tails of each query tile are listed in ascending sorted position
// and padded to a multiple of GT_ROWS with the sentinel row N; the SIMT engine
// then gathers them GT_ROWS at a time (tiles_simt.cu, tiles_gather_kernel).
// Measured on c2 L1 (numpy model of the same pivots): 2.76% -> 1.43% of all
// pairs computed.

// Sorted tails, row-major with row stride Kpad (zero padded), row N = zeros
// (the sentinel the lists are padded with; the engines mask it by index or by
// ||t||^2 = 3e38), the sorted tails' first MP_G keys with row stride MP_G (two float4
// loads per tail), and for the tensor-core engine the per-tail scalars
// {||t||^2 / 2, ||t|| (up), ||t - tf32(t)|| (up), 0} from FP64 sums -- the
// same values the tile staging kernel (prep.cu) computes.  One warp per row.
__device__ __forceinline__ double gt_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__global__ void stage_rows_kernel(const float* __restrict__ E, const int* __restrict__ tperm,
                                  const float* __restrict__ keys, long long N, int d, int Kpad, int K,
                                  float* __restrict__ Ts, float* __restrict__ tks, float4* __restrict__ tsc) {
    const int lane = threadIdx.x & 31;
    for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; i <= N;
         i += ((long long)gridDim.x * blockDim.x) >> 5) {
        float* dst = Ts + (size_t)i * Kpad;
        if (i == N) {
            for (int k = lane; k < Kpad; k += 32) dst[k] = 0.f;
            continue;
        }
        const long long src = tperm[i];
        const float* row = E + (size_t)src * d;
        double s2 = 0.0, sd2 = 0.0;
        for (int k = lane; k < Kpad; k += 32) {
            const float x = k < d ? __ldg(row + k) : 0.f;
            dst[k] = x;
            const double xd = x, rd = (double)(x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u));
            s2 += xd * xd;
            sd2 += rd * rd;
        }
        if (lane < MP_G) tks[(size_t)i * MP_G + lane] = lane < K ? __ldg(keys + (size_t)src * K + lane) : 0.f;
        if (tsc) {
            s2 = gt_warp_sum(s2);
            sd2 = gt_warp_sum(sd2);
            if (lane == 0)
                tsc[i] = make_float4(__double2float_rn(0.5 * s2), __double2float_ru(sqrt(s2)),
                                     __double2float_ru(sqrt(sd2)), 0.f);
        }
    }
}

__device__ __forceinline__ float gt_warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// One pass, warp per query tile of this shard: the tails of its surviving BN-row
// tiles (BN / 32 groups of 32 per tile, UN tiles' key loads in flight) that pass
// the per-tail test, written in ascending sorted position at list offset
// BN * (tile prefix[q] - prefix[first]) -- the tile list's own offsets, an
// upper bound -- and padded with the sentinel N to whole blocks of BN.  TCM
// (tensor-core engine): also ||t||^2/2 per list entry (3e38 for padding) and per
// block the maxima of ||t|| and ||t - tf32(t)|| (the guard band's Tm, Tdm).
template <int BN, bool TCM>
__global__ void gather_tails_kernel(const float* __restrict__ qbmin, const float* __restrict__ qbmax,
                                    const float4* __restrict__ tks, const int* __restrict__ list,
                                    const long long* __restrict__ cum, const int2* __restrict__ ranges,
                                    DevCounters* ctr, long long N, int K, float theta, float relm, int chunk,
                                    long long* __restrict__ gblocks, int2* __restrict__ granges,
                                    int* __restrict__ nitem, int* __restrict__ glist,
                                    const float4* __restrict__ tsc, float* __restrict__ gT2,
                                    float2* __restrict__ gtst, int cyc_world, int cyc_rank) {
    constexpr int H = BN / 32, UN = BN == 64 ? 4 : 1;
    const int tq0 = ctr->tq_begin, tq1 = ctr->tq_end;
    if (tq0 >= tq1) return;
    const long long base = cum[tq0];
    const int lane = threadIdx.x & 31;
    unsigned long long pairs = 0, blocks = 0;
    for (long long q = tq0 + ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5); q < tq1;
         q += ((long long)gridDim.x * blockDim.x) >> 5) {
        if (cyc_world > 1 && q % cyc_world != cyc_rank) continue;  // cyclic split: not this rank's tile
        // the per-tail test uses the first MP_G pivots (tks holds those; fewer pivots only prune less)
        const int Kg = K < MP_G ? K : MP_G;
        float qmn[MP_G], qmx[MP_G];
#pragma unroll
        for (int k = 0; k < MP_G; ++k)
            if (k < Kg) { qmn[k] = qbmin[q * K + k]; qmx[k] = qbmax[q * K + k]; }
        const int ntl = ranges[q].y + 1;
        const long long loff = cum[q] - base;
        const int* L = list + loff;
        int* out = glist + loff * BN;
        long long c = 0;
        float bn_max = 0.f, bd_max = 0.f;  // TCM: running maxima of the current block
        for (int u0 = 0; u0 < ntl; u0 += UN) {
            float4 kv[UN][H][2];
            long long ib[UN];
#pragma unroll
            for (int x = 0; x < UN; ++x) {
                ib[x] = u0 + x < ntl ? (long long)__ldg(L + u0 + x) * BN + lane : N;
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const long long i = ib[x] + 32 * h;
                    kv[x][h][0] = i < N ? __ldg(tks + 2 * i) : make_float4(0, 0, 0, 0);
                    kv[x][h][1] = i < N ? __ldg(tks + 2 * i + 1) : make_float4(0, 0, 0, 0);
                }
            }
#pragma unroll
            for (int x = 0; x < UN; ++x) {
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const long long i = ib[x] + 32 * h;
                    const float4 a = kv[x][h][0], b = kv[x][h][1];
                    const float tk[MP_G] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                    const bool ok = i < N && mp_survives<MP_G>(qmn, qmx, tk, tk, Kg, theta, relm);
                    const unsigned m = __ballot_sync(0xffffffffu, ok);
                    if (!m) continue;
                    const long long pos = c + __popc(m & lanemask_lt());
                    if (ok) out[pos] = (int)i;  // ascending positions
                    if (TCM) {
                        float4 sc = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (ok) {
                            sc = __ldg(tsc + i);
                            gT2[loff * BN + pos] = sc.x;
                        }
                        // this group spans at most two blocks: the current one and the next
                        const long long bcur = c / BN;
                        const bool nxt = ok && pos / BN != bcur;
                        const float n1 = gt_warp_max(ok && !nxt ? sc.y : 0.f), d1 = gt_warp_max(ok && !nxt ? sc.z : 0.f);
                        bn_max = fmaxf(bn_max, n1);
                        bd_max = fmaxf(bd_max, d1);
                        if (__any_sync(0xffffffffu, nxt)) {
                            if (lane == 0) gtst[loff + bcur] = make_float2(bn_max, bd_max);
                            bn_max = gt_warp_max(nxt ? sc.y : 0.f);
                            bd_max = gt_warp_max(nxt ? sc.z : 0.f);
                        }
                    }
                    c += __popc(m);
                    if (TCM && c % BN == 0) {  // the group filled its block exactly
                        if (lane == 0) gtst[loff + c / BN - 1] = make_float2(bn_max, bd_max);
                        bn_max = bd_max = 0.f;
                    }
                }
            }
        }
        const long long nb = (c + BN - 1) / BN;
        for (long long o = c + lane; o < nb * BN; o += 32) {
            out[o] = (int)N;  // sentinel padding
            if (TCM) gT2[loff * BN + o] = 3e38f;
        }
        if (TCM && c % BN != 0 && lane == 0) gtst[loff + c / BN] = make_float2(bn_max, bd_max);  // partial block
        if (lane == 0) {
            gblocks[q] = nb;
            granges[q] = make_int2(0, (int)nb - 1);
            nitem[q] = (int)((nb + chunk - 1) / chunk);
        }
        pairs += (unsigned long long)c;
        blocks += (unsigned long long)nb;
    }
    if (lane == 0 && blocks) {
        atomicAdd(&ctr->gpairs, pairs);
        atomicAdd((unsigned long long*)&ctr->gblocks, blocks);
    }
}

// The SIMT engine's list build with one 256-thread block per query tile: tile
// lists are heavy-tailed (c2 L1: median 3 surviving tiles per query tile, p99
// 137, max 496), so a warp per query tile left a long serial chain.  Warp w takes
// a contiguous eighth of the list; pass 1 counts, a shared-memory prefix orders
// the eighths, pass 2 writes (keys reloaded from L1/L2) -- the same ascending
// output as gather_tails_kernel<64, false>.
template <int BN>
__global__ void __launch_bounds__(256) gather_tails_block_kernel(
    const float* __restrict__ qbmin, const float* __restrict__ qbmax, const float4* __restrict__ tks,
    const int* __restrict__ list, const long long* __restrict__ cum, const int2* __restrict__ ranges,
    DevCounters* ctr, long long N, int K, float theta, float relm, int chunk, long long* __restrict__ gblocks,
    int2* __restrict__ granges, int* __restrict__ nitem, int* __restrict__ glist, int cyc_world, int cyc_rank,
    int GB) {
    // BN: tail-tile rows (list offsets; 64 SIMT, 256 tensor cores); GB: rows per gathered block
    constexpr int NW = 8, H = BN / 32, UN = BN == 64 ? 2 : 1;
    __shared__ long long wcnt[NW + 1];
    const int tq0 = ctr->tq_begin, tq1 = ctr->tq_end;
    if (tq0 >= tq1) return;
    const long long base = cum[tq0];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long pairs = 0, blocks = 0;
    for (long long q = tq0 + blockIdx.x; q < tq1; q += gridDim.x) {
        if (cyc_world > 1 && q % cyc_world != cyc_rank) continue;  // cyclic split: not this rank's tile
        // the per-tail test uses the first MP_G pivots (tks holds those; fewer pivots only prune less)
        const int Kg = K < MP_G ? K : MP_G;
        float qmn[MP_G], qmx[MP_G];
#pragma unroll
        for (int k = 0; k < MP_G; ++k)
            if (k < Kg) { qmn[k] = qbmin[q * K + k]; qmx[k] = qbmax[q * K + k]; }
        const int ntl = ranges[q].y + 1;
        const long long loff = cum[q] - base;
        const int* L = list + loff;
        int* out = glist + loff * BN;
        const int u_lo = (int)((long long)ntl * w / NW), u_hi = (int)((long long)ntl * (w + 1) / NW);
        long long c = 0;
        for (int pass = 0; pass < 2; ++pass) {
            if (pass == 1) c = wcnt[w];
            for (int u0 = u_lo; u0 < u_hi; u0 += UN) {
                float4 kv[UN][H][2];
                long long ib[UN];
#pragma unroll
                for (int x = 0; x < UN; ++x) {
                    ib[x] = u0 + x < u_hi ? (long long)__ldg(L + u0 + x) * BN + lane : N;
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                        const long long i = ib[x] + 32 * h;
                        kv[x][h][0] = i < N ? __ldg(tks + 2 * i) : make_float4(0, 0, 0, 0);
                        kv[x][h][1] = i < N ? __ldg(tks + 2 * i + 1) : make_float4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int x = 0; x < UN; ++x) {
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                        const long long i = ib[x] + 32 * h;
                        const float4 a = kv[x][h][0], b = kv[x][h][1];
                        const float tk[MP_G] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                        const bool ok = i < N && mp_survives<MP_G>(qmn, qmx, tk, tk, Kg, theta, relm);
                        const unsigned m = __ballot_sync(0xffffffffu, ok);
                        if (pass == 1 && ok) out[c + __popc(m & lanemask_lt())] = (int)i;
                        c += __popc(m);
                    }
                }
            }
            if (pass == 0) {
                if (lane == 0) wcnt[w + 1] = c;
                __syncthreads();
                if (threadIdx.x == 0) {
                    wcnt[0] = 0;
                    for (int x = 1; x <= NW; ++x) wcnt[x] += wcnt[x - 1];
                }
                __syncthreads();
            }
        }
        const long long tot = wcnt[NW];
        const long long nb = (tot + GB - 1) / GB;
        for (long long o = tot + threadIdx.x; o < nb * GB; o += blockDim.x) out[o] = (int)N;  // sentinel padding
        if (threadIdx.x == 0) {
            gblocks[q] = nb;
            granges[q] = make_int2(0, (int)nb - 1);
            nitem[q] = (int)((nb + chunk - 1) / chunk);
            pairs += (unsigned long long)tot;
            blocks += (unsigned long long)nb;
        }
        __syncthreads();  // wcnt is reused by the next query tile
    }
    if (threadIdx.x == 0 && blocks) {
        atomicAdd(&ctr->gpairs, pairs);
        atomicAdd((unsigned long long*)&ctr->gblocks, blocks);
    }
}

// ------------------------------------------- local kd refinement of the order
// The space-filling-curve order keeps tiles compact only as far as the curve is;
// a kd-tree keeps query boxes tighter (numpy, c2 L1: 13% fewer gathered tails).  A
// cheap local form: every aligned chunk of KD_CH consecutive sorted rows of a
// segment is split three times along its widest pivot-key dimension (512 -> 256
// -> 128 -> 64-row leaves = the SIMT tiles; pairs of leaves form the 128-row
// tensor-core tiles): one block per chunk, bitonic sorts in shared memory
// (numpy: 7% fewer gathered tails than Hilbert alone).  Only the order changes.
constexpr int KD_CH = 512, KD_LEVELS = 3;
__global__ void __launch_bounds__(KD_CH) kd_refine_kernel(const float* __restrict__ keys, int* __restrict__ perm,
                                                         long long L, int K) {
    __shared__ float kk[KD_CH][MP_G + 1];  // padded: row reads are conflict-free
    __shared__ int idx[KD_CH];
    __shared__ float sk[KD_CH];
    __shared__ int sl[KD_CH];
    __shared__ int ndim[1 << (KD_LEVELS - 1)];
    __shared__ float wmn[KD_CH / 32][MP_G], wmx[KD_CH / 32][MP_G];
    const long long seg = blockIdx.y;
    const long long c0 = (long long)blockIdx.x * KD_CH;
    if (c0 >= L) return;
    const int n = (int)(L - c0 < KD_CH ? L - c0 : KD_CH);
    const int i = threadIdx.x, lane = i & 31, w = i >> 5;
    int* pr = perm + seg * L + c0;
    const int my = i < n ? pr[i] : -1;
    idx[i] = my;
    if (K == MP_G) {  // two 16-byte loads per row
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
        if (my >= 0) {
            const float4* r4 = reinterpret_cast<const float4*>(keys + ((size_t)seg * L + my) * MP_G);
            a = __ldg(r4);
            b = __ldg(r4 + 1);
        }
        kk[i][0] = a.x; kk[i][1] = a.y; kk[i][2] = a.z; kk[i][3] = a.w;
        kk[i][4] = b.x; kk[i][5] = b.y; kk[i][6] = b.z; kk[i][7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < MP_G; ++k)
            kk[i][k] = (my >= 0 && k < K) ? keys[((size_t)seg * L + my) * K + k] : 0.f;
    }
    __syncthreads();
    for (int lev = 0; lev < KD_LEVELS; ++lev) {
        const int S = KD_CH >> lev, nodes = 1 << lev;
        {   // widest key dimension of every node over its real rows: warp partials, then one
            // thread per node combines its warps
            const bool real = idx[i] >= 0;
#pragma unroll
            for (int k = 0; k < MP_G; ++k) {
                float a = real ? kk[i][k] : 3e38f, z = real ? kk[i][k] : -3e38f;
                for (int o = 16; o > 0; o >>= 1) {
                    a = fminf(a, __shfl_xor_sync(0xffffffffu, a, o));
                    z = fmaxf(z, __shfl_xor_sync(0xffffffffu, z, o));
                }
                if (lane == 0) { wmn[w][k] = a; wmx[w][k] = z; }
            }
            __syncthreads();
            if (i < nodes) {
                const int wpn = (KD_CH / 32) / nodes;  // warps per node
                int best = 0;
                float bw = -1.f;
                for (int k = 0; k < K; ++k) {
                    float a = 3e38f, z = -3e38f;
                    for (int x = i * wpn; x < (i + 1) * wpn; ++x) { a = fminf(a, wmn[x][k]); z = fmaxf(z, wmx[x][k]); }
                    if (z - a > bw) { bw = z - a; best = k; }
                }
                ndim[i] = best;
            }
        }
        __syncthreads();
        // bitonic sort of every S-row node on (key, slot): strides < 32 by warp shuffles,
        // larger strides through shared memory (19 barriers over the three levels, not 109)
        float kv = idx[i] >= 0 ? kk[i][ndim[i / S]] : 3e38f;  // padding rows sort to the end
        int sv = i;
        for (int size = 2; size <= S; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                float pk;
                int ps;
                if (stride >= 32) {
                    sk[i] = kv;
                    sl[i] = sv;
                    __syncthreads();
                    pk = sk[i ^ stride];
                    ps = sl[i ^ stride];
                    __syncthreads();
                } else {
                    pk = __shfl_xor_sync(0xffffffffu, kv, stride);
                    ps = __shfl_xor_sync(0xffffffffu, sv, stride);
                }
                const bool up = (i & size) == 0, lower = (i & stride) == 0;
                const bool p_less = pk < kv || (pk == kv && ps < sv);
                if (lower == up ? p_less : !p_less) {  // keep the min (ascending lower half) or the max
                    kv = pk;
                    sv = ps;
                }
            }
        }
        sl[i] = sv;
        __syncthreads();
        // apply the node permutations
        const int src = sl[i];
        const int nidx = idx[src];
        float nk[MP_G];
#pragma unroll
        for (int k = 0; k < MP_G; ++k) nk[k] = kk[src][k];
        __syncthreads();
        idx[i] = nidx;
#pragma unroll
        for (int k = 0; k < MP_G; ++k) kk[i][k] = nk[k];
        __syncthreads();
    }
    // padding rows are at the end of every node that holds any; compact the real rows
    // (the partial last chunk: real rows first, in node order)
    if (n == KD_CH) {
        pr[i] = idx[i];
    } else if (i == 0) {
        int o = 0;
        for (int j = 0; j < KD_CH; ++j)
            if (idx[j] >= 0) pr[o++] = idx[j];
    }
}

void launch_kd_refine(const float* keys, int* perm, long long nseg, long long L, int K, cudaStream_t s) {
    if (L < 2 * SIMT_T || K > MP_G) return;  // (experiment: up to MP_G pivots)
    dim3 grid((unsigned)((L + KD_CH - 1) / KD_CH), (unsigned)nseg);
    kd_refine_kernel<<<grid, KD_CH, 0, s>>>(keys, perm, L, K);
}

// ------------------------------------------------------------ launchers
void launch_pick_pivots(const float* E, long long N, int d, int norm, int K, const double* p0, float* P,
                        cudaStream_t s) {
    // sample size: at most 1024 tails and ~200 KB of shared memory
    long long S = (200 * 1024 / 4 - d) / (d | 1);
    if (S > 1024) S = 1024;
    if (S > N) S = N;
    if (S < 1) S = 1;
    const size_t smem = ((size_t)S * (d | 1) + d) * sizeof(float);
    auto kern = norm == 1 ? pick_pivots_kernel<1> : pick_pivots_kernel<2>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<1, 1024, smem, s>>>(E, N, d, K, (int)S, p0, P);
}

// K dispatch for the key kernels: 2..8, 12, 16, 24, 32 pivots, and 48 ... 128 for the L2 path (mp_pivots_ok)
template <int KMAX = 32, class F>
static void for_pivots(int K, F&& f) {
    if constexpr (KMAX >= 48) {
        if (K == 48) { f(std::integral_constant<int, 48>{}); return; }
        if (K == 64) { f(std::integral_constant<int, 64>{}); return; }
        if (K == 96) { f(std::integral_constant<int, 96>{}); return; }
        if (K == 128) { f(std::integral_constant<int, 128>{}); return; }
    }
    switch (K) {
        case 2: f(std::integral_constant<int, 2>{}); break;
        case 3: f(std::integral_constant<int, 3>{}); break;
        case 4: f(std::integral_constant<int, 4>{}); break;
        case 5: f(std::integral_constant<int, 5>{}); break;
        case 6: f(std::integral_constant<int, 6>{}); break;
        case 7: f(std::integral_constant<int, 7>{}); break;
        case 8: f(std::integral_constant<int, 8>{}); break;
        case 12: f(std::integral_constant<int, 12>{}); break;
        case 16: f(std::integral_constant<int, 16>{}); break;
        case 24: f(std::integral_constant<int, 24>{}); break;
        default: f(std::integral_constant<int, 32>{}); break;
    }
}

static void launch_mp_qkeys(const float* E, const float* Rel, long long N, long long R, int d, int norm, int K,
                            const float* P, float* keys, unsigned int* minmax, unsigned int* qnmax,
                            unsigned int* nonfinite, cudaStream_t s) {
    // relations per warp NU (8 NU per block): per 4-dim step a warp issues ~K + 1 + NU shared loads
    // and NU (2K + 2) packed FP32 ops, and ceil(R / 8 NU) blocks cover the relations -- pick the NU
    // with the least issue per entity chunk (c4, R = 37: 3; c2, R = 18: 3; c5, R = 100: 4)
    int NU = 1;
    double best = 1e300;
    for (int nu = 1; nu <= 4 && nu * K <= 32; ++nu) {
        const double c = (double)((R + 8 * nu - 1) / (8 * nu)) * (K + 1 + nu + nu * (2.0 * K + 2));
        if (c < best - 1e-9) { best = c; NU = nu; }
    }
    const int S = mk_stride(d), D4 = (d + 3) / 4 * 4;
    const size_t smem = (size_t)(2 * 32 * S + K * D4 + 8 * NU * D4) * sizeof(float);
    const long long gy = (R + 8 * NU - 1) / (8 * NU);
    const long long chunks = (N + 31) / 32;
    long long gx_target = (148LL * 6 + gy - 1) / gy;
    if (gx_target < 1) gx_target = 1;
    long long nch = (chunks + gx_target - 1) / gx_target;
    nch = std::max<long long>(1, std::min<long long>(nch, 16));
    dim3 grid((unsigned)((chunks + nch - 1) / nch), (unsigned)gy);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, 256, smem, s>>>(E, Rel, N, R, d, (int)nch, P, keys, minmax, qnmax, nonfinite);
    };
    auto byNU = [&](auto n_, auto k_) {
        constexpr int NN = decltype(n_)::value, KK = decltype(k_)::value;
        // NU K <= 32 (one lane per (relation, pivot) min / max): larger NU only for small K
        if (NU == 1) go(mp_qkeys_kernel<NN, KK, 1>);
        if constexpr (2 * KK <= 32) if (NU == 2) go(mp_qkeys_kernel<NN, KK, 2>);
        if constexpr (3 * KK <= 32) if (NU == 3) go(mp_qkeys_kernel<NN, KK, 3>);
        if constexpr (4 * KK <= 32) if (NU == 4) go(mp_qkeys_kernel<NN, KK, 4>);
    };
    auto byK = [&](auto n_) { for_pivots(K, [&](auto k_) { byNU(n_, k_); }); };
    if (norm == 1) byK(std::integral_constant<int, 1>{});
    else byK(std::integral_constant<int, 2>{});
}

void launch_mp_keys(const float* E, const float* Rel, long long N, long long nseg, int d, int norm, int K,
                    const float* P, float* keys, unsigned int* minmax, unsigned int* qnmax, unsigned int* nonfinite,
                    cudaStream_t s) {
    const bool query = Rel != nullptr;
    mp_init_minmax_kernel<<<grid_for_mp(nseg * K, 256), 256, 0, s>>>(minmax, nseg * K, query ? qnmax : nullptr, nseg);
    if (query) {
        launch_mp_qkeys(E, Rel, N, nseg, d, norm, K, P, keys, minmax, qnmax, nonfinite, s);
        return;
    }
    const int S = mk_stride(d), D4 = (d + 3) / 4 * 4;
    const int ent = query ? 32 : 128;
    const size_t smem = (size_t)(ent * S + K * D4 + (query ? 16 * D4 : 0)) * sizeof(float);
    const long long gy = query ? (nseg + 15) / 16 : 1;
    const long long chunks = (N + ent - 1) / ent;
    long long gx_target = (148LL * 8 + gy - 1) / gy;
    if (gx_target < 1) gx_target = 1;
    long long nch = (chunks + gx_target - 1) / gx_target;
    if (nch < 1) nch = 1;
    if (nch > 8) nch = 8;
    dim3 grid((unsigned)((chunks + nch - 1) / nch), (unsigned)gy);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, query ? 256 : 128, smem, s>>>(E, Rel, N, nseg, d, (int)nch, P, keys, minmax, qnmax, nonfinite);
    };
    auto byK = [&](auto n_, auto q_) {
        constexpr int NN = decltype(n_)::value;
        constexpr bool QQ = decltype(q_)::value;
        if constexpr (!QQ) for_pivots(K, [&](auto k_) { go(mp_keys_kernel<NN, QQ, decltype(k_)::value>); });
    };
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using BT = std::integral_constant<bool, true>;
    using BF = std::integral_constant<bool, false>;
    if (norm == 1) { if (query) byK(I1{}, BT{}); else byK(I1{}, BF{}); }
    else { if (query) byK(I2{}, BT{}); else byK(I2{}, BF{}); }
}

// L2 keys by the factorisation (see mp_qkeys_fact_kernel): tails (Et, NT) and queries
// (E + Rel, N x R), both FP64.  A (N x K doubles) and hmax (one word) are scratch.
void launch_mp_keys_l2f(const float* E, const float* Rel, long long N, long long R, const float* Et, long long NT,
                        int d, int K, const float* P, float* tkeys, unsigned int* tminmax, float* qkeys4,
                        unsigned int* qmm4, unsigned int* qnmax, double* A, double* Bhr, double* Cg, double* HP,
                        unsigned int* hmax, unsigned int* nonfinite, unsigned int* twid, cudaStream_t s,
                        cudaEvent_t bready) {
    const int KO = K < MP_SORT_PIVOTS ? K : MP_SORT_PIVOTS;
    mp_init_minmax_kernel<<<grid_for_mp(K, 256), 256, 0, s>>>(tminmax, K, nullptr, 0);
    mp_init_minmax_kernel<<<grid_for_mp(R * KO, 256), 256, 0, s>>>(qmm4, R * KO, qnmax, R);
    cudaMemsetAsync(hmax, 0, 8, s);  // hmax[0] heads, hmax[1] tails
    cudaMemsetAsync(twid, 0, 4, s);
    const bool same = Et == E && NT == N;
    auto byK = [&](auto k_) {
        constexpr int KK = decltype(k_)::value;
        constexpr int KOO = KK < MP_SORT_PIVOTS ? KK : MP_SORT_PIVOTS;
        // entity terms: HP = X P^T by the FP64 GEMM, then A, the tail keys and their ranges
        launch_mp_hr(E, P, N, KK, d, HP, s);
        mp_ent_gemm_kernel<KK><<<grid_for_mp(N, 256, 148LL * 8), 256, 0, s>>>(
            E, N, d, P, HP, A, same ? tkeys : nullptr, same ? tminmax : nullptr, hmax, nonfinite);
        if (!same) {  // tails from another array (tail partition / block join): their own terms
            launch_mp_hr(Et, P, NT, KK, d, HP, s);
            mp_ent_gemm_kernel<KK><<<grid_for_mp(NT, 256, 148LL * 8), 256, 0, s>>>(
                Et, NT, d, P, HP, nullptr, tkeys, tminmax, hmax + 1, nonfinite);
        }
        mp_rel_terms_kernel<<<(unsigned)std::min<long long>(148LL * 4, (R * (KK + 1) + 7) / 8), 256, 0, s>>>(
            Rel, R, d, KK, P, Cg, hmax, qnmax, nonfinite, same ? hmax : hmax + 1, twid);
        cudaStreamWaitEvent(s, bready, 0);  // B from the aux stream (launch_mp_hr)
        dim3 gk((unsigned)((N + 255) / 256), (unsigned)((R + QK_RCH - 1) / QK_RCH));
        mp_qkeys_fact_kernel<KK, KOO><<<gk, 256, 0, s>>>(Bhr, A, Cg, N, R, qkeys4, qmm4);
    };
    for_pivots<128>(K, byK);
}

// The full K query keys per (r, h) (kgc_inspect only: the join itself never materialises them).
void launch_mp_qkeys_all(const double* Bhr, const double* A, const double* Cg, long long N, long long R, int K,
                         float* keys, cudaStream_t s) {
    for_pivots<128>(K, [&](auto k_) {
        constexpr int KK = decltype(k_)::value;
        dim3 gk((unsigned)((N + 255) / 256), (unsigned)((R + QK_RCH - 1) / QK_RCH));
        mp_qkeys_fact_kernel<KK, KK><<<gk, 256, 0, s>>>(Bhr, A, Cg, N, R, keys, nullptr);
    });
}

void launch_mp_qboxes_fact(const unsigned int* perm, const double* Bhr, const double* A, const double* Cg, long long N,
                           long long R, int K, int ROWS, int QT, const unsigned int* qnmax, float* bmin, float* bmax,
                           cudaStream_t s) {
    for_pivots<128>(K, [&](auto k_) {
        constexpr int KK = decltype(k_)::value;
        mp_qboxes_fact_kernel<KK><<<grid_for_mp(R * QT * 32, 256), 256, 0, s>>>(perm, Bhr, A, Cg, N, R, ROWS, QT, qnmax,
                                                                              bmin, bmax);
    });
}

void launch_mp_hr(const float* E, const float* Rel, long long N, long long R, int d, double* B, cudaStream_t s) {
    dim3 ghr((unsigned)((N + HR_BM - 1) / HR_BM), (unsigned)((R + HR_BR - 1) / HR_BR));
    mp_hr_kernel<<<ghr, 128, 0, s>>>(E, Rel, N, R, d, B);
}

void launch_mp_morton(const float* keys, const unsigned int* minmax, long long nseg, long long L, int K, int bits,
                      unsigned int* code, unsigned int* idx, cudaStream_t s) {
    // Hilbert order by default (c2: gathered L1 pairs 1.72% -> 1.69%, tile kernel -4%);
    // KGC_HILBERT=0 restores the Morton (Z) order
    const char* e = kgc_knob("KGC_HILBERT");
    const int hilbert = e ? atoi(e) : 1;
    mp_morton_kernel<<<grid_for_mp(nseg * L, 256), 256, 0, s>>>(keys, minmax, nseg, L, K, bits, code, idx, hilbert);
}

void launch_mp_boxes(const float* keys, const unsigned int* perm, long long nseg, long long L, int ROWS, int ntile,
                     int K, float* bmin, float* bmax, const unsigned int* qnmax, cudaStream_t s, int transpose) {
    mp_boxes_kernel<<<grid_for_mp(nseg * ntile * 32, 256), 256, 0, s>>>(keys, perm, nseg, L, ROWS, ntile, K, bmin,
                                                                         bmax, qnmax, transpose);
}

void launch_mp_count(const float* qbmin, const float* qbmax, const float* tbmin, const float* tbmax, long long nq,
                     int TT, int K, float theta, float relm, int prune, int2* ranges, long long* cost, unsigned int* bits,
                     cudaStream_t s) {
    const int CT = mc_chunk(K);
    const size_t smem = (size_t)(2 * K * CT + MC_W * 2 * K) * 4;
    cudaFuncSetAttribute(mp_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mp_count_kernel<<<grid_for_mp(nq, MC_W, 148LL * 16), 32 * MC_W, smem, s>>>(qbmin, qbmax, tbmin, tbmax, nq, TT, K,
                                                                             theta, relm, prune, ranges, cost,
                                                                             prune ? bits : nullptr);
}

void launch_mp_emit(const float* qbmin, const float* qbmax, const float* tbmin, const float* tbmax,
                    const long long* cum, const DevCounters* ctr, long long nq, int TT, int K, float theta, float relm,
                    int prune, int* list, const unsigned int* bits, cudaStream_t s) {
    auto kern = (prune && bits) ? mp_emit_kernel<true> : mp_emit_kernel<false>;
    kern<<<grid_for_mp(nq * 32, 256), 256, 0, s>>>(qbmin, qbmax, tbmin, tbmax, cum, ctr, TT, K, theta, relm, prune, list,
                                                  prune ? bits : nullptr);
}

void launch_stage_rows(const float* E, const int* tperm, const float* keys, long long N, int d, int Kpad, int K,
                       float* Ts, float* tks, float4* tsc, cudaStream_t s) {
    stage_rows_kernel<<<grid_for_mp((N + 1) * 32, 256), 256, 0, s>>>(E, tperm, keys, N, d, Kpad, K, Ts, tks, tsc);
}

// Tensor-core gathered blocks: per list entry ||t||^2 / 2 (3e38 for the sentinel padding)
// and per block of BN entries the maxima of ||t|| and ||t - tf32(t)|| (the guard band's Tm,
// Tdm) -- from the written lists, one warp per block (8 entries per lane).
template <int BN>
__global__ void gather_scalars_kernel(const long long* __restrict__ cum, const long long* __restrict__ gblocks,
                                      const DevCounters* ctr, const int* __restrict__ glist,
                                      const float4* __restrict__ tsc, long long N, float* __restrict__ gT2,
                                      float2* __restrict__ gtst) {
    const int tq0 = ctr->tq_begin, tq1 = ctr->tq_end;
    if (tq0 >= tq1) return;
    const long long base = cum[tq0];
    const int lane = threadIdx.x & 31;
    const long long nwarp = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long q = tq0 + ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5); q < tq1; q += nwarp) {
        const long long loff = cum[q] - base, nb = gblocks[q];
        for (long long b = 0; b < nb; ++b) {
            const long long e0 = (loff + b) * BN;
            float mn = 0.f, md = 0.f;
#pragma unroll
            for (int u = 0; u < BN / 32; ++u) {
                const long long e = e0 + u * 32 + lane;
                const int i = __ldg(glist + e);
                float4 sc = make_float4(3e38f, 0.f, 0.f, 0.f);
                if (i < N) sc = __ldg(tsc + i);
                gT2[e] = sc.x;
                mn = fmaxf(mn, sc.y);
                md = fmaxf(md, sc.z);
            }
            mn = gt_warp_max(mn);
            md = gt_warp_max(md);
            if (lane == 0) gtst[loff + b] = make_float2(mn, md);
        }
    }
}

void launch_gather_tails(const float* qbmin, const float* qbmax, const float* tks, const int* list,
                         const long long* cum, const int2* ranges, DevCounters* ctr, long long N, int BN, int K,
                         float theta, float relm, int chunk, long long nq, long long* gblocks, int2* granges,
                         int* nitem, int* glist, const float4* tsc, float* gT2, float2* gtst, int cyc_world,
                         int cyc_rank, cudaStream_t s, int gb) {
    const unsigned g = grid_for_mp(nq * 32, 256);
    const float4* tk4 = reinterpret_cast<const float4*>(tks);
    (void)g;
    if (BN == 64) {
        gather_tails_block_kernel<64><<<grid_for_mp(nq, 1, 148LL * 16), 256, 0, s>>>(
            qbmin, qbmax, tk4, list, cum, ranges, ctr, N, K, theta, relm, chunk, gblocks, granges, nitem, glist,
            cyc_world, cyc_rank, gb);
    } else {
        // tensor cores: the same block-per-query-tile list build (a warp per query tile left long serial
        // chains on heavy-tailed tile lists: c4 3.2 ms), then the per-entry / per-block scalars
        gather_tails_block_kernel<256><<<grid_for_mp(nq, 1, 148LL * 16), 256, 0, s>>>(
            qbmin, qbmax, tk4, list, cum, ranges, ctr, N, K, theta, relm, chunk, gblocks, granges, nitem, glist,
            cyc_world, cyc_rank, 256);
        gather_scalars_kernel<256><<<grid_for_mp(nq * 32, 256), 256, 0, s>>>(cum, gblocks, ctr, glist, tsc, N, gT2,
                                                                              gtst);
    }
}

}  // namespace kgc
