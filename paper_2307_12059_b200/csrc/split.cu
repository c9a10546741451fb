// Spatial block-cyclic head split (kgc_options.split = 3; SURVEY §8(e)
// "we create a block which can be processed in parallel").
//
// The query side is split by HEADS: rank k of W joins the queries h + r of its own heads h,
// every relation r, against all N tails (replicated).  The heads are ordered along a
// space-filling curve (Morton order of the distances to 4 pivots), the order is cut into
// W * m chunks of ~N / (W m) consecutive heads, and chunk c goes to rank c mod W.  A chunk is
// spatially compact, so its queries h + r (a translated copy of the chunk) still form tight
// query tiles -- the pruning power of the one-GPU join is kept -- while every rank holds a
// stratified sample of the whole space, so dense and empty query regions spread evenly over
// the ranks with no cost estimate (measured on one GPU, emulated shards: DESIGN.md §8).
//
// Every rank computes the same order from the same inputs: the pivots, keys and codes are
// deterministic and the radix sort is stable, so the chunks partition the heads exactly.
// The order only steers which GPU joins which head; it never changes what is computed.
#include <cfloat>

#include "common.cuh"

namespace kgc {

static inline unsigned sp_grid(long long n, int threads, long long cap = 148LL * 64) {
    long long g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    return (unsigned)(g < cap ? g : cap);
}

constexpr int SP_K = 4;     // pivots of the space-filling curve
constexpr int SP_BITS = 8;  // bits per pivot key (32-bit codes)

// warp per 4 entities: the SP_K FP32 distances to the pivots (lanes over k, float4 loads of the 4
// rows in flight when d % 4 == 0), min / max per pivot as float bits (distances are >= 0, so the
// unsigned order is the float order)
constexpr int SP_R = 4;  // rows per warp step
__global__ void __launch_bounds__(256) sp_keys_kernel(const float* __restrict__ E, long long N, int d,
                                                      const float* __restrict__ P, float* __restrict__ keys,
                                                      unsigned int* __restrict__ mm) {
    const int lane = threadIdx.x & 31;
    const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const bool vec = (d & 3) == 0 && (reinterpret_cast<uintptr_t>(E) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(P) & 15) == 0;
    float mn[SP_K], mx[SP_K];
#pragma unroll
    for (int j = 0; j < SP_K; ++j) { mn[j] = FLT_MAX; mx[j] = 0.f; }
    for (long long i0 = w0 * SP_R; i0 < N; i0 += nw * SP_R) {
        float acc[SP_R][SP_K] = {};
        if (vec) {
            for (int k = 4 * lane; k < d; k += 128) {
                float4 v[SP_R];
#pragma unroll
                for (int u = 0; u < SP_R; ++u)
                    v[u] = i0 + u < N ? __ldg(reinterpret_cast<const float4*>(E + (i0 + u) * d + k))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int j = 0; j < SP_K; ++j) {
                    const float4 p = __ldg(reinterpret_cast<const float4*>(P + j * d + k));
#pragma unroll
                    for (int u = 0; u < SP_R; ++u) {
                        const float a = v[u].x - p.x, b = v[u].y - p.y, c = v[u].z - p.z, e = v[u].w - p.w;
                        acc[u][j] = fmaf(a, a, fmaf(b, b, fmaf(c, c, fmaf(e, e, acc[u][j]))));
                    }
                }
            }
        } else {
            for (int k = lane; k < d; k += 32) {
#pragma unroll
                for (int u = 0; u < SP_R; ++u) {
                    const float v = i0 + u < N ? E[(i0 + u) * d + k] : 0.f;
#pragma unroll
                    for (int j = 0; j < SP_K; ++j) {
                        const float t = v - P[j * d + k];
                        acc[u][j] = fmaf(t, t, acc[u][j]);
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < SP_R; ++u) {
            if (i0 + u >= N) break;
#pragma unroll
            for (int j = 0; j < SP_K; ++j) {
                float a = acc[u][j];
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                a = sqrtf(a);
                if (lane == j) keys[(i0 + u) * SP_K + j] = a;
                mn[j] = fminf(mn[j], a);
                mx[j] = fmaxf(mx[j], a);
            }
        }
    }
    if (lane < SP_K) {
        float a = mn[0], b = mx[0];
#pragma unroll
        for (int j = 1; j < SP_K; ++j)
            if (lane == j) { a = mn[j]; b = mx[j]; }
        atomicMin(&mm[2 * lane], __float_as_uint(a));
        atomicMax(&mm[2 * lane + 1], __float_as_uint(b));
    }
}

__global__ void sp_init_kernel(unsigned int* mm) {
    if (threadIdx.x < SP_K) {
        mm[2 * threadIdx.x] = 0x7f7fffffu;  // FLT_MAX
        mm[2 * threadIdx.x + 1] = 0u;
    }
}

// Morton code of the SP_K keys quantised to SP_BITS bits each; value = entity index
__global__ void sp_code_kernel(const float* __restrict__ keys, long long N, const unsigned int* __restrict__ mm,
                               unsigned int* __restrict__ code, unsigned int* __restrict__ idx) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned int c = 0;
#pragma unroll
        for (int j = 0; j < SP_K; ++j) {
            const float lo = __uint_as_float(mm[2 * j]), hi = __uint_as_float(mm[2 * j + 1]);
            const float sc = hi > lo ? (float)(1 << SP_BITS) / (hi - lo) : 0.f;
            int q = (int)((keys[i * SP_K + j] - lo) * sc);
            q = q < 0 ? 0 : (q > (1 << SP_BITS) - 1 ? (1 << SP_BITS) - 1 : q);
#pragma unroll
            for (int b = 0; b < SP_BITS; ++b) c |= (unsigned int)((q >> b) & 1) << (b * SP_K + j);
        }
        code[i] = c;
        idx[i] = (unsigned int)i;
    }
}

// grid (row blocks, owned chunks): owned chunk i of this rank is c = k + W i, positions
// [c N / nch, (c + 1) N / nch) of the order, local rows from the sizes of the chunks before
// it; hidx[dst + j] = order[src + j] and Eh[dst + j] = E[order[src + j]] (warp per row)
__global__ void __launch_bounds__(256) sp_gather_kernel(const float* __restrict__ E, int d,
                                                        const unsigned int* __restrict__ order, long long N,
                                                        long long nch, long long W, long long k,
                                                        int* __restrict__ hidx, float* __restrict__ Eh) {
    const long long i = blockIdx.y, c = k + W * i;
    const long long src = c * N / nch, len = (c + 1) * N / nch - src;
    long long dst = 0;
    for (long long p = 0; p < i; ++p) {
        const long long cp = k + W * p;
        dst += (cp + 1) * N / nch - cp * N / nch;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (long long j = blockIdx.x * 8LL + w; j < len; j += gridDim.x * 8LL) {
        const long long h = order[src + j];
        if (lane == 0) hidx[dst + j] = (int)h;
        for (int kk = lane; kk < d; kk += 32) Eh[(dst + j) * d + kk] = E[h * d + kk];
    }
}

void launch_sp_order(const float* E, long long N, int d, const float* P, float* keys, unsigned int* mm,
                     unsigned int* code, unsigned int* idx, cudaStream_t s) {
    sp_init_kernel<<<1, 32, 0, s>>>(mm);
    sp_keys_kernel<<<sp_grid((N + SP_R - 1) / SP_R * 32, 256, 148 * 8), 256, 0, s>>>(E, N, d, P, keys, mm);
    sp_code_kernel<<<sp_grid(N, 256), 256, 0, s>>>(keys, N, mm, code, idx);
}

void launch_sp_gather(const float* E, int d, const unsigned int* order, long long N, long long nch, long long W,
                      long long k, long long owned, long long max_len, int* hidx, float* Eh, cudaStream_t s) {
    if (owned <= 0 || max_len <= 0) return;
    long long bx = (max_len + 7) / 8;
    if (bx > 1184) bx = 1184;
    sp_gather_kernel<<<dim3((unsigned)bx, (unsigned)owned), 256, 0, s>>>(E, d, order, N, nch, W, k, hidx, Eh);
}

}  // namespace kgc
