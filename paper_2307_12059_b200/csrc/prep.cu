// prep.cu -- the preprocessing steps of the join:
//   K1  pivot distances of every query q = h + r and every tail t
//       (Fig. algo1 lines 3-6; connector_1 = h + r)
//   K2  per-relation sort of the query keys and one sort of the tail keys
//       (lines 7-10; "the sorting is not heavy"; tails once)
//   K3  per query tile, the contiguous range of surviving tail tiles
//       (Lemma 1 PAPER.md:202-210 + Lemma 2 PAPER.md:282-305 at tile granularity)
//   and the staging of operand tiles in the layouts the tile engines read.
#include <cfloat>
#include <climits>
#include <cstdio>

#include <cuda_fp16.h>

#include "common.cuh"

namespace kgc {

static inline unsigned grid_for(long long n, int threads, long long cap = 148LL * 64) {
    long long g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

// ============================================================== K1: keys
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_min_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__global__ void init_minmax_kernel(unsigned int* mm, long long nseg) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nseg; i += (long long)gridDim.x * blockDim.x) {
        mm[2 * i] = __float_as_uint(FLT_MAX);
        mm[2 * i + 1] = 0u;
    }
}

// d(t, p) = ||t - p||_norm in FP64, stored RN to float.  One warp per tail.
template <int NORM, bool PIV>
__global__ void tail_keys_kernel(const float* __restrict__ E, long long N, int d, const double* __restrict__ pivot,
                                 float* __restrict__ kt, unsigned int* minmax_seg, unsigned int* nonfinite) {
    const int lane = threadIdx.x & 31;
    long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    float kmin = FLT_MAX, kmax = 0.f;
    bool bad = false;
    for (long long row = warp; row < N; row += nwarps) {
        double s = 0.0;
        const float* e = E + row * d;
        for (int k = lane; k < d; k += 32) {
            float v = e[k];
            bad |= !isfinite(v);
            double x = (double)v - (PIV ? pivot[k] : 0.0);
            s += NORM == 1 ? fabs(x) : x * x;
        }
        s = warp_sum_d(s);
        float key = __double2float_rn(NORM == 2 ? sqrt(s) : s);
        if (lane == 0) kt[row] = key;
        kmin = fminf(kmin, key);
        kmax = fmaxf(kmax, key);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(nonfinite, 1u);
    if (lane == 0) {
        atomicMin(&minmax_seg[0], __float_as_uint(kmin));
        atomicMax(&minmax_seg[1], __float_as_uint(kmax));
    }
}

// d(h + r, p) for every (h, r): a block walks `nch` chunks of 32 entity rows
// (in shared memory, fp32) against 32 relation rows (shared memory, FP64:
// converted once per block); warp w handles relations w, w + 8, w + 16,
// w + 24 with lane = entity, so each entity value is converted to FP64 once
// per 4 relations.  Per-relation key min/max are kept per warp across the
// chunks (one atomic pair per relation per warp).
constexpr int QK_ENT = 32, QK_RPW = 4;  // relations per block: 8 * rpw, rpw <= QK_RPW (shared memory for large d)
template <int NORM, bool PIV>
__global__ void __launch_bounds__(256) query_keys_kernel(const float* __restrict__ E, const float* __restrict__ Rel,
                                                         long long N, long long R, int d, int nch, int rpw,
                                                         const double* __restrict__ pivot, float* __restrict__ kq,
                                                         unsigned int* minmax, unsigned int* nonfinite) {
    extern __shared__ double qk_smem_d[];
    const int QK_REL = 8 * rpw;
    double* Rs = qk_smem_d;                                 // [QK_REL][d] relation rows (FP64, exact)
    double* Ps = Rs + (size_t)QK_REL * d;                   // [d] pivot (PIV)
    const int S = (d & 1) ? d : d + 1;                      // odd row stride: conflict-free column reads
    float* Es = reinterpret_cast<float*>(Ps + (PIV ? d : 0));  // [QK_ENT][S]
    const long long r0 = (long long)blockIdx.y * QK_REL;
    bool bad = false;
    for (int x = threadIdx.x; x < QK_REL * d; x += blockDim.x) {
        const int i = x / d, k = x % d;
        const float v = (r0 + i < R) ? Rel[(r0 + i) * d + k] : 0.f;
        bad |= !isfinite(v);
        Rs[x] = (double)v;
    }
    if (PIV)
        for (int k = threadIdx.x; k < d; k += blockDim.x) Ps[k] = pivot[k];
    if (blockIdx.x == 0 && __syncthreads_or(bad)) {
        if (threadIdx.x == 0) atomicOr(nonfinite, 1u);
    }
    bad = false;  // from here: the entity rows (a tail partition does not cover every head)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float mn[QK_RPW], mx[QK_RPW];
#pragma unroll
    for (int u = 0; u < QK_RPW; ++u) { mn[u] = FLT_MAX; mx[u] = 0.f; }
    for (int ch = 0; ch < nch; ++ch) {
        const long long h0 = ((long long)blockIdx.x * nch + ch) * QK_ENT;
        if (h0 >= N) break;
        __syncthreads();  // previous chunk fully consumed (and Rs / Ps written)
        for (int x = threadIdx.x; x < QK_ENT * d; x += blockDim.x) {
            const int i = x / d, k = x % d;
            const float v = (h0 + i < N) ? E[(h0 + i) * d + k] : 0.f;
            bad |= !isfinite(v);
            Es[i * S + k] = v;
        }
        __syncthreads();
        const long long h = h0 + lane;
        const float* es = Es + lane * S;
        double s[QK_RPW];
#pragma unroll
        for (int u = 0; u < QK_RPW; ++u) s[u] = 0.0;
        for (int k = 0; k < d; ++k) {
            const double e = (double)es[k];
#pragma unroll
            for (int u = 0; u < QK_RPW; ++u) {
                if (u >= rpw) break;
                double x = e + Rs[(w + 8 * u) * d + k];  // connector_1(h, r) = h + r
                if (PIV) x -= Ps[k];
                s[u] += NORM == 1 ? fabs(x) : x * x;
            }
        }
#pragma unroll
        for (int u = 0; u < QK_RPW; ++u) {
            const long long r = r0 + w + 8 * u;
            const float key = __double2float_rn(NORM == 2 ? sqrt(s[u]) : s[u]);
            if (u < rpw && h < N && r < R) {
                kq[r * N + h] = key;
                mn[u] = fminf(mn[u], key);
                mx[u] = fmaxf(mx[u], key);
            }
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1u);
#pragma unroll
    for (int u = 0; u < QK_RPW; ++u) {
        const long long r = r0 + w + 8 * u;
        if (u >= rpw || r >= R) break;
        const float a = warp_min_f(mn[u]), z = warp_max_f(mx[u]);
        if (lane == 0) {
            atomicMin(&minmax[2 * r], __float_as_uint(a));
            atomicMax(&minmax[2 * r + 1], __float_as_uint(z));
        }
    }
}

// Column means of E in FP64 (pivot option "mean of tails").
__global__ void pivot_mean_kernel(const float* __restrict__ E, long long N, int d, double* pivot) {
    int k = blockIdx.x;
    double s = 0.0;
    for (long long i = threadIdx.x; i < N; i += blockDim.x) s += (double)E[i * d + k];
    __shared__ double red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) pivot[k] = N > 0 ? red[0] / (double)N : 0.0;
}

void launch_pivot_mean(const float* E, long long N, int d, double* pivot, cudaStream_t s) {
    pivot_mean_kernel<<<d, 256, 0, s>>>(E, N, d, pivot);
}

void launch_tail_keys(const float* E, long long N, int d, int norm, const double* pivot, float* kt,
                      unsigned int* minmax_seg, unsigned int* nonfinite, cudaStream_t s) {
    init_minmax_kernel<<<1, 32, 0, s>>>(minmax_seg, 1);
    unsigned g = grid_for(N * 32, 256);
    if (norm == 1) {
        if (pivot) tail_keys_kernel<1, true><<<g, 256, 0, s>>>(E, N, d, pivot, kt, minmax_seg, nonfinite);
        else tail_keys_kernel<1, false><<<g, 256, 0, s>>>(E, N, d, pivot, kt, minmax_seg, nonfinite);
    } else {
        if (pivot) tail_keys_kernel<2, true><<<g, 256, 0, s>>>(E, N, d, pivot, kt, minmax_seg, nonfinite);
        else tail_keys_kernel<2, false><<<g, 256, 0, s>>>(E, N, d, pivot, kt, minmax_seg, nonfinite);
    }
}

void launch_query_keys(const float* E, const float* Rel, long long N, long long R, int d, int norm,
                       const double* pivot, float* kq, unsigned int* minmax, unsigned int* nonfinite,
                       cudaStream_t s) {
    init_minmax_kernel<<<grid_for(R, 256), 256, 0, s>>>(minmax, R);
    const int S = (d & 1) ? d : d + 1;
    int rpw = QK_RPW;
    auto smem_for = [&](int rp) {
        return (size_t)(8 * rp * d + (pivot ? d : 0)) * sizeof(double) + (size_t)QK_ENT * S * sizeof(float);
    };
    while (rpw > 1 && smem_for(rpw) > 200 * 1024) rpw >>= 1;
    const size_t smem = smem_for(rpw);
    // chunks per block: enough blocks to fill the GPU (~8 per SM), at most 8 chunks
    const long long gy = (R + 8 * rpw - 1) / (8 * rpw), chunks = (N + QK_ENT - 1) / QK_ENT;
    long long gx_target = (148LL * 8 + gy - 1) / gy;
    long long nch = (chunks + gx_target - 1) / gx_target;
    nch = nch < 1 ? 1 : (nch > 8 ? 8 : nch);
    dim3 grid((unsigned)((chunks + nch - 1) / nch), (unsigned)gy);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, 256, smem, s>>>(E, Rel, N, R, d, (int)nch, rpw, pivot, kq, minmax, nonfinite);
    };
    if (norm == 1) {
        if (pivot) go(query_keys_kernel<1, true>); else go(query_keys_kernel<1, false>);
    } else {
        if (pivot) go(query_keys_kernel<2, true>); else go(query_keys_kernel<2, false>);
    }
}

// ============================================================== scans
constexpr int SCAN_T = 256, SCAN_I = 8, SCAN_B = SCAN_T * SCAN_I;

template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
    __shared__ T warp_tot[SCAN_T / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += n;
    }
    if (lane == 31) warp_tot[w] = inc;
    __syncthreads();
    if (w == 0) {
        T x = lane < SCAN_T / 32 ? warp_tot[lane] : T(0);
        T xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T n = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += n;
        }
        if (lane < SCAN_T / 32) warp_tot[lane] = xi - x;
        if (lane == SCAN_T / 32 - 1) *total = xi;
    }
    __syncthreads();
    T r = warp_tot[w] + inc - v;
    __syncthreads();
    return r;
}

template <typename T>
__global__ void scan_reduce_kernel(const T* __restrict__ in, size_t n, T* partial) {
    size_t base = (size_t)blockIdx.x * SCAN_B + (size_t)threadIdx.x * SCAN_I;
    T s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_I; ++i)
        if (base + i < n) s += in[base + i];
    __shared__ T tot;
    block_excl_scan<T>(s, &tot);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

template <typename T>
__global__ void scan_partials_kernel(T* partial, size_t nb, T* grand_total) {
    __shared__ T carry;
    __shared__ T tot;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (size_t base = 0; base < nb; base += SCAN_T) {
        size_t i = base + threadIdx.x;
        T v = i < nb ? partial[i] : T(0);
        T ex = block_excl_scan<T>(v, &tot);
        if (i < nb) partial[i] = ex + carry;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && grand_total) *grand_total = carry;
}

template <typename T>
__global__ void scan_final_kernel(const T* __restrict__ in, T* __restrict__ out, size_t n, const T* partial) {
    size_t base = (size_t)blockIdx.x * SCAN_B + (size_t)threadIdx.x * SCAN_I;
    T v[SCAN_I];
    T s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_I; ++i) {
        v[i] = base + i < n ? in[base + i] : T(0);
        s += v[i];
    }
    __shared__ T tot;
    T ex = block_excl_scan<T>(s, &tot) + partial[blockIdx.x];
#pragma unroll
    for (int i = 0; i < SCAN_I; ++i) {
        if (base + i < n) out[base + i] = ex;
        ex += v[i];
    }
}

size_t scan_tmp_bytes(size_t n) { return ((n + SCAN_B - 1) / SCAN_B + 2) * sizeof(long long) + 256; }

template <typename T>
static void scan_exclusive(const T* in, T* out, size_t n, T* total, void* tmp, cudaStream_t s, int* launches) {
    size_t nb = (n + SCAN_B - 1) / SCAN_B;
    if (nb == 0) nb = 1;
    T* partial = reinterpret_cast<T*>(tmp);
    scan_reduce_kernel<T><<<(unsigned)nb, SCAN_T, 0, s>>>(in, n, partial);
    scan_partials_kernel<T><<<1, SCAN_T, 0, s>>>(partial, nb, total);
    scan_final_kernel<T><<<(unsigned)nb, SCAN_T, 0, s>>>(in, out, n, partial);
    if (launches) *launches += 3;
}

void scan_exclusive_i32(const int* in, int* out, size_t n, void* tmp, cudaStream_t s, int* launches) {
    scan_exclusive<int>(in, out, n, nullptr, tmp, s, launches);
}
void scan_exclusive_i64(const long long* in, long long* out, size_t n, long long* total, void* tmp,
                        cudaStream_t s, int* launches) {
    scan_exclusive<long long>(in, out, n, total, tmp, s, launches);
}

// ============================================================== K2: sort
// Segmented, stable LSD radix sort of S segments of L keys on a 16-bit
// quantisation of the float key inside its segment's [min, max] (two 8-bit
// passes).  Ties keep ascending original index, so the order is
// deterministic (identical on every rank).  Order only affects how tight the
// tile bounds are, never correctness: K3 uses the actual key min/max of every
// tile.
__global__ void radix_prep_kernel(const float* __restrict__ keys, const unsigned int* __restrict__ minmax,
                                  long long S, long long L, unsigned int* k0, unsigned int* v0) {
    long long n = S * L;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        long long s = idx / L, i = idx - s * L;
        float kmin = __uint_as_float(minmax[2 * s]), kmax = __uint_as_float(minmax[2 * s + 1]);
        float range = kmax - kmin;
        unsigned q = 0;
        if (range > 0.f) {
            float x = (keys[idx] - kmin) * (65536.0f / range);
            x = fminf(fmaxf(x, 0.f), 65535.f);
            q = (unsigned)x;
        }
        k0[idx] = q;
        v0[idx] = (unsigned)i;
    }
}

template <typename KeyT>
__global__ void radix_hist_kernel(const KeyT* __restrict__ kin, long long L, int B, int shift, int* counts) {
    __shared__ int h[256];
    const long long s = blockIdx.y;
    const int b = blockIdx.x;
    h[threadIdx.x] = 0;
    __syncthreads();
    long long base = (long long)b * SORT_IPB;
#pragma unroll
    for (int k = 0; k < SORT_IPB / 256; ++k) {
        long long i = base + k * 256 + threadIdx.x;
        if (i < L) atomicAdd(&h[(unsigned)(kin[s * L + i] >> shift) & 255u], 1);
    }
    __syncthreads();
    counts[(s * 256 + threadIdx.x) * B + b] = h[threadIdx.x];
}

template <typename KeyT>
__global__ void __launch_bounds__(256) radix_scatter_kernel(const KeyT* __restrict__ kin,
                                                            const unsigned int* __restrict__ vin,
                                                            KeyT* __restrict__ kout,
                                                            unsigned int* __restrict__ vout,
                                                            const int* __restrict__ offs, long long L, int B,
                                                            int shift) {
    __shared__ int run[256];
    __shared__ int wcnt[8][257];
    const long long s = blockIdx.y;
    const int b = blockIdx.x;
    const int w = threadIdx.x >> 5;
    run[threadIdx.x] = 0;
    const long long base = (long long)b * SORT_IPB;
    const int boff = offs[(s * 256 + threadIdx.x) * B + b];
    __shared__ int blk_off[256];
    blk_off[threadIdx.x] = boff;
    for (int round = 0; round < SORT_IPB / 256; ++round) {
        long long i = base + round * 256 + threadIdx.x;
        bool valid = i < L;
        KeyT key = valid ? kin[s * L + i] : KeyT(0);
        int dg = valid ? (int)((unsigned)(key >> shift) & 255u) : 256;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) wcnt[ww][threadIdx.x] = 0;
        __syncthreads();
        unsigned peers = __match_any_sync(0xffffffffu, dg);
        int lrank = __popc(peers & lanemask_lt());
        if (valid && lrank == 0) wcnt[w][dg] = __popc(peers);
        __syncthreads();
        {
            int sum = run[threadIdx.x];
#pragma unroll
            for (int ww = 0; ww < 8; ++ww) {
                int c = wcnt[ww][threadIdx.x];
                wcnt[ww][threadIdx.x] = sum;
                sum += c;
            }
            run[threadIdx.x] = sum;
        }
        __syncthreads();
        if (valid) {
            long long dst = (long long)blk_off[dg] + wcnt[w][dg] + lrank;
            kout[dst] = key;
            vout[dst] = vin[s * L + i];
        }
        __syncthreads();
    }
}

__global__ void radix_final_kernel(const unsigned int* __restrict__ v, const float* __restrict__ keys, long long S,
                                   long long L, int* perm, float* skeys) {
    long long n = S * L;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        long long s = idx / L;
        unsigned src = v[idx];
        perm[idx] = (int)src;
        skeys[idx] = keys[s * L + src];
    }
}

size_t radix_counts_len(long long S, long long L) {
    long long B = (L + SORT_IPB - 1) / SORT_IPB;
    return (size_t)(S * 256 * (B > 0 ? B : 1));
}

// Short segments (L <= RADIX_SMALL_L): the whole stable sort of a segment in one CTA's shared
// memory -- quantise, two 8-bit counting passes over packed (key16 << 16 | index) words,
// permutation out -- instead of ~12 launches that each round-trip the keys through global
// memory.  Same order as the multi-kernel path (stable by quantised key, ties by index).
// Measured per-rank fixed cost it removes: c3 at W = 8, 0.22 ms of sorts (mostly launch- and
// latency-bound small kernels).
constexpr int RADIX_SMALL_L = 20000;  // 2 L words + counters fit in shared memory; index fits 16 bits
constexpr int RS_NT = 512;
__global__ void __launch_bounds__(RS_NT) radix_small_kernel(const float* __restrict__ keys,
                                                            const unsigned int* __restrict__ minmax, long long L,
                                                            int* __restrict__ perm, float* __restrict__ skeys) {
    extern __shared__ unsigned int rs_smem[];
    constexpr int NW = RS_NT / 32;
    unsigned int* a = rs_smem;                                   // [L]
    unsigned int* b = rs_smem + L;                               // [L]
    int* hist = reinterpret_cast<int*>(rs_smem + 2 * L);         // [256] running digit offsets
    int* wcnt = hist + 256;                                      // [NW][257]
    const long long s = blockIdx.x;
    const float* kk = keys + s * L;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const float kmin = __uint_as_float(minmax[2 * s]), kmax = __uint_as_float(minmax[2 * s + 1]);
    const float range = kmax - kmin;
    for (int i = tid; i < L; i += RS_NT) {
        unsigned q = 0;
        if (range > 0.f) {
            float x = (kk[i] - kmin) * (65536.0f / range);
            x = fminf(fmaxf(x, 0.f), 65535.f);
            q = (unsigned)x;
        }
        a[i] = (q << 16) | (unsigned)i;
    }
    for (int pass = 0; pass < 2; ++pass) {
        const unsigned int* src = pass == 0 ? a : b;
        unsigned int* dst = pass == 0 ? b : a;
        const int shift = 16 + 8 * pass;
        if (tid < 256) hist[tid] = 0;
        __syncthreads();
        for (int i = tid; i < L; i += RS_NT) atomicAdd(&hist[(src[i] >> shift) & 255u], 1);
        __syncthreads();
        if (w == 0) {  // exclusive scan of the 256 bins: 8 per lane, then across lanes
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
        for (int base = 0; base < L; base += RS_NT) {
            const int i = base + tid;
            const bool valid = i < L;
            const unsigned int x = valid ? src[i] : 0u;
            const int dg = valid ? (int)((x >> shift) & 255u) : 256;
            for (int z = tid; z < NW * 257; z += RS_NT) wcnt[z] = 0;
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
            if (valid) dst[wcnt[w * 257 + dg] + lrank] = x;
            __syncthreads();
        }
    }
    for (int i = tid; i < L; i += RS_NT) {
        const unsigned int src_i = a[i] & 0xFFFFu;
        perm[s * L + i] = (int)src_i;
        skeys[s * L + i] = kk[src_i];
    }
}

int radix_sort_segments(const float* keys, const unsigned int* minmax, long long S, long long L, unsigned int* k0,
                        unsigned int* v0, unsigned int* k1, unsigned int* v1, int* counts, int* perm_out,
                        float* skeys_out, void* scan_tmp, size_t /*scan_tmp_bytes*/, cudaStream_t s,
                        int* launches) {
    if (S <= 0 || L <= 0) return 0;
    if (L <= RADIX_SMALL_L) {
        const size_t smem = (size_t)(2 * L + 256 + (RS_NT / 32) * 257) * 4;
        cudaFuncSetAttribute(radix_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        radix_small_kernel<<<(unsigned)S, RS_NT, smem, s>>>(keys, minmax, L, perm_out, skeys_out);
        if (launches) *launches += 1;
        return 0;
    }
    const int B = (int)((L + SORT_IPB - 1) / SORT_IPB);
    const size_t nc = (size_t)S * 256 * B;
    radix_prep_kernel<<<grid_for(S * L, 256), 256, 0, s>>>(keys, minmax, S, L, k0, v0);
    dim3 g((unsigned)B, (unsigned)S);
    for (int pass = 0; pass < 2; ++pass) {
        const unsigned int* ki = pass == 0 ? k0 : k1;
        const unsigned int* vi = pass == 0 ? v0 : v1;
        unsigned int* ko = pass == 0 ? k1 : k0;
        unsigned int* vo = pass == 0 ? v1 : v0;
        radix_hist_kernel<unsigned int><<<g, 256, 0, s>>>(ki, L, B, pass * 8, counts);
        scan_exclusive_i32(counts, counts, nc, scan_tmp, s, launches);
        radix_scatter_kernel<unsigned int><<<g, 256, 0, s>>>(ki, vi, ko, vo, counts, L, B, pass * 8);
    }
    radix_final_kernel<<<grid_for(S * L, 256), 256, 0, s>>>(v0, keys, S, L, perm_out, skeys_out);
    if (launches) *launches += 6;
    return 0;
}

// Stable LSD sort of S segments of L keys (already in k0, values = in-segment indices in v0) on
// the low `bits` bits; sorted values end in v0.  32-bit keys for the K-pivot Hilbert codes (4 x 8
// bits: 8 bytes per item per scatter instead of 12 with 64-bit keys).
template <class KeyT>
static void radix_sort_code_segments(long long S, long long L, int bits, KeyT* k0, unsigned int* v0, KeyT* k1,
                                     unsigned int* v1, int* counts, void* scan_tmp, cudaStream_t s, int* launches) {
    if (S <= 0 || L <= 0) return;
    const int B = (int)((L + SORT_IPB - 1) / SORT_IPB);
    const size_t nc = (size_t)S * 256 * B;
    dim3 g((unsigned)B, (unsigned)S);
    int passes = (bits + 7) / 8;
    if (passes & 1) ++passes;  // even pass count: the result lands back in (k0, v0)
    for (int pass = 0; pass < passes; ++pass) {
        const KeyT* ki = (pass & 1) ? k1 : k0;
        const unsigned int* vi = (pass & 1) ? v1 : v0;
        KeyT* ko = (pass & 1) ? k0 : k1;
        unsigned int* vo = (pass & 1) ? v0 : v1;
        radix_hist_kernel<KeyT><<<g, 256, 0, s>>>(ki, L, B, pass * 8, counts);
        scan_exclusive_i32(counts, counts, nc, scan_tmp, s, launches);
        radix_scatter_kernel<KeyT><<<g, 256, 0, s>>>(ki, vi, ko, vo, counts, L, B, pass * 8);
        if (launches) *launches += 2;
    }
}
void radix_sort_u64_segments(long long S, long long L, int bits, unsigned long long* k0, unsigned int* v0,
                             unsigned long long* k1, unsigned int* v1, int* counts, void* scan_tmp, cudaStream_t s,
                             int* launches) {
    radix_sort_code_segments(S, L, bits, k0, v0, k1, v1, counts, scan_tmp, s, launches);
}
void radix_sort_u32_segments(long long S, long long L, int bits, unsigned int* k0, unsigned int* v0, unsigned int* k1,
                             unsigned int* v1, int* counts, void* scan_tmp, cudaStream_t s, int* launches) {
    radix_sort_code_segments(S, L, bits, k0, v0, k1, v1, counts, scan_tmp, s, launches);
}

// ============================================================== K3: ranges
// Per tail tile j: [tmin_j, tmax_j] of its sorted keys; cmax = running max of
// tmax, cmin = running min of tmin from the right.  Both are monotone, so the
// tiles that can hold a tail within theta of a query-tile key interval form a
// contiguous range found by binary search (Lemma 2's s_i <= s_{i+1},
// e_i <= e_{i+1}, at tile granularity).
__global__ void tail_tile_minmax_kernel(const float* __restrict__ tskey, long long N, int BN, int TT, float* tmin,
                                        float* tmax) {
    const int lane = threadIdx.x & 31;
    long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long j = warp; j < TT; j += nwarps) {
        float mn = FLT_MAX, mx = -FLT_MAX;
        long long b = j * BN, e = min((long long)N, b + BN);
        for (long long i = b + lane; i < e; i += 32) {
            float k = tskey[i];
            mn = fminf(mn, k);
            mx = fmaxf(mx, k);
        }
        mn = warp_min_f(mn);
        mx = warp_max_f(mx);
        if (lane == 0) {
            tmin[j] = mn;
            tmax[j] = mx;
        }
    }
}

__global__ void tail_tile_cum_kernel(const float* tmin, const float* tmax, int TT, float* cmax, float* cmin) {
    if (threadIdx.x == 0) {
        float m = -FLT_MAX;
        for (int j = 0; j < TT; ++j) {
            m = fmaxf(m, tmax[j]);
            cmax[j] = m;
        }
    } else if (threadIdx.x == 32) {
        float m = FLT_MAX;
        for (int j = TT - 1; j >= 0; --j) {
            m = fminf(m, tmin[j]);
            cmin[j] = m;
        }
    }
}

void launch_tail_tile_bounds(const float* tskey, long long N, int BN, int TT, float* tmin, float* tmax, float* cmax,
                             float* cmin, cudaStream_t s, int* launches) {
    tail_tile_minmax_kernel<<<grid_for((long long)TT * 32, 256), 256, 0, s>>>(tskey, N, BN, TT, tmin, tmax);
    tail_tile_cum_kernel<<<1, 64, 0, s>>>(tmin, tmax, TT, cmax, cmin);
    if (launches) *launches += 2;
}

// Pruning margin: keys are FP64 norms rounded to float (relative error
// <= 2^-24); theta is widened by 2^-14 relative and the key bounds by 2^-20
// relative so that no pair with dist3 <= theta is ever pruned (DESIGN.md
// "Floating-point rigor of pruning").
__global__ void query_ranges_kernel(const float* __restrict__ qskey, long long N, long long R, int QT, int TT,
                                    int bq, const float* __restrict__ cmax, const float* __restrict__ cmin,
                                    float theta, int prune, int2* ranges, long long* cost) {
    const int lane = threadIdx.x & 31;
    long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long nq = R * (long long)QT;
    for (long long tq = warp; tq < nq; tq += nwarps) {
        long long r = tq / QT, qt = tq - r * QT;
        long long b = qt * bq, e = min(N, b + bq);
        float mn = FLT_MAX, mx = -FLT_MAX;
        for (long long i = b + lane; i < e; i += 32) {
            float k = qskey[r * N + i];
            mn = fminf(mn, k);
            mx = fmaxf(mx, k);
        }
        mn = warp_min_f(mn);
        mx = warp_max_f(mx);
        if (lane == 0) {
            int sb = 0, eb = TT - 1;
            if (prune) {
                const float th = theta * (1.0f + 6.103515625e-05f);                // theta (1 + 2^-14)
                const float lo = mn - th - fabsf(mn) * 9.5367431640625e-07f;      // - |key| 2^-20
                const float hi = mx + th + fabsf(mx) * 9.5367431640625e-07f;
                int a = 0, z = TT;  // first j with cmax[j] >= lo
                while (a < z) {
                    int m = (a + z) >> 1;
                    if (cmax[m] >= lo) z = m; else a = m + 1;
                }
                sb = a;
                a = 0; z = TT;      // first j with cmin[j] > hi
                while (a < z) {
                    int m = (a + z) >> 1;
                    if (cmin[m] > hi) z = m; else a = m + 1;
                }
                eb = a - 1;
            }
            ranges[tq] = make_int2(sb, eb);
            cost[tq] = eb >= sb ? (long long)(eb - sb + 1) : 0LL;
        }
    }
}

void launch_query_ranges(const float* qskey, long long N, long long R, int QT, int TT, int bq, const float* cmax,
                         const float* cmin, float theta, int prune, int2* ranges, long long* cost, cudaStream_t s) {
    query_ranges_kernel<<<grid_for(R * QT * 32, 256), 256, 0, s>>>(qskey, N, R, QT, TT, bq, cmax, cmin, theta, prune,
                                                                    ranges, cost);
}

// Shard assignment: query tile q belongs to rank min(W-1, W*cum[q]/total)
// (cum = exclusive prefix of surviving-tile counts) -- identical to the host
// function kgc_shard_range().  Work items of at most `chunk` tail tiles.
__global__ void shard_count_kernel(const long long* __restrict__ cost, const long long* __restrict__ cum,
                                   long long nq, int rank, int world, int chunk, DevCounters* ctr, int* nitem,
                                   long long force_lo, long long force_hi) {
    const long long total = ctr->total_cost;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nq; q += (long long)gridDim.x * blockDim.x) {
        int owner = 0;
        if (force_lo >= 0) {
            owner = (q >= force_lo && q < force_hi) ? rank : rank + 1;  // rank-local split: a fixed range
        } else if (force_lo == -2) {
            owner = (int)(q % world);  // cyclic split: query tiles dealt round-robin
        } else if (total > 0) {
            long long o = (long long)world * cum[q] / total;
            owner = (int)(o < world - 1 ? o : world - 1);
        }
        int n = 0;
        if (owner == rank) {
            atomicMin(&ctr->tq_begin, (int)q);
            atomicMax(&ctr->tq_end, (int)q + 1);
            long long c = cost[q];
            atomicAdd((unsigned long long*)&ctr->my_cost, (unsigned long long)c);
            n = (int)((c + chunk - 1) / chunk);
        }
        nitem[q] = n;
    }
}

__global__ void shard_emit_kernel(const int2* __restrict__ ranges, const int* __restrict__ nitem,
                                  const int* __restrict__ off, long long nq, int chunk, DevCounters* ctr,
                                  int4* items, long long* item_tiles, const long long* __restrict__ cum, int list_mode) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nq; q += (long long)gridDim.x * blockDim.x) {
        int n = nitem[q];
        int o = off[q];
        if (q == nq - 1) ctr->n_items = (long long)o + n;
        int2 rg = ranges[q];
        const int loff = (list_mode && n > 0) ? (int)(cum[q] - cum[ctr->tq_begin]) : -1;
        for (int k = 0; k < n; ++k) {
            int j0 = rg.x + k * chunk;
            int j1 = min(rg.y, j0 + chunk - 1);
            items[o + k] = make_int4((int)q, j0, j1, loff);
            item_tiles[o + k] = j1 - j0 + 1;
        }
    }
}

void launch_shard_items(const int2* ranges, const long long* cost, const long long* cum, long long nq, int rank,
                        int world, int chunk, DevCounters* ctr, int* nitem, int* item_off, int4* items,
                        long long* item_tiles, void* tmp, cudaStream_t s, int* launches, int phase, int list_mode,
                        long long force_lo, long long force_hi) {
    if (phase == 0) {
        shard_count_kernel<<<grid_for(nq, 256), 256, 0, s>>>(cost, cum, nq, rank, world, chunk, ctr, nitem, force_lo,
                                                             force_hi);
        scan_exclusive_i32(nitem, item_off, (size_t)nq, tmp, s, launches);
        if (launches) *launches += 1;
    } else {
        shard_emit_kernel<<<grid_for(nq, 256), 256, 0, s>>>(ranges, nitem, item_off, nq, chunk, ctr, items,
                                                            item_tiles, cum, list_mode);
        if (launches) *launches += 1;
    }
}

// ============================================================== staging
// Operand tiles in HBM in exactly the shared-memory layout the engines read,
// so one bulk TMA copy moves a whole (chunk of a) tile:
//   tensor-core layout (UMMA K-major, no swizzle): element (i, k) of a ROWS-row
//     tile at float offset ((k/4) * (ROWS/8) + i/8) * 32 + (i%8) * 4 + k%4;
//   SIMT layout: element (i, k) at k * ROWS + i.
// Zero padding for rows >= N and k >= d.  Query values q = fl32(h + r).
// Row scalars (FP64 sums of the fp32 values): ||v||^2, ||v||, ||v - tf32(v)||
// (truncation residual, which bounds the round-to-nearest residual too), ||v||_1.
__device__ __forceinline__ float tf32_trunc(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

struct RowStat {
    double s2, sd2, s1;
};

template <bool TC>
__device__ __forceinline__ size_t stage_off(int i, int k, int ROWS) {
    if (TC) return ((size_t)(k >> 2) * (ROWS >> 3) + (i >> 3)) * 32 + (i & 7) * 4 + (k & 3);
    return (size_t)k * ROWS + i;
}

// grid: one block per tile; 256 threads.  `rel` == nullptr for tails.
template <bool TC>
__global__ void __launch_bounds__(1024) stage_kernel(const float* __restrict__ E, const float* __restrict__ Rel,
                                                    const int* __restrict__ perm, long long N, int d, int Kpad,
                                                    int ROWS, int QT, int tile0, int norm, float theta,
                                                    float* __restrict__ out, float4* __restrict__ qs,
                                                    float* __restrict__ T2, float2* __restrict__ tstile, int split,
                                                    int cyc_world = 0, int cyc_rank = 0) {
    const int tile = tile0 + blockIdx.x;
    if (cyc_world > 1 && tile % cyc_world != cyc_rank) return;  // cyclic split: another rank's query tile
    long long r = 0, t_in_rel = tile;
    if (Rel) {
        r = tile / QT;
        t_in_rel = tile - r * QT;
    }
    const int* pr = perm + (Rel ? r * N : 0);
    const float* rel = Rel ? Rel + r * d : nullptr;
    float* dst = out + (size_t)blockIdx.x * ROWS * Kpad;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
    __shared__ float sTn[32], sTd[32];
    float tn_max = 0.f, td_max = 0.f;

    // rows handled by warp w; TC: lanes over k (4 consecutive k per lane),
    // SIMT: lanes over rows.
    if (TC) {
        for (int i = w; i < ROWS; i += NW) {
            long long p = t_in_rel * ROWS + i;
            bool valid = p < N;
            long long h = valid ? pr[p] : 0;
            RowStat st{0, 0, 0};
            for (int kq = lane; kq < (Kpad >> 2); kq += 32) {
                float4 v;
                float* vv = reinterpret_cast<float*>(&v);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    int k = kq * 4 + c;
                    float x = 0.f;
                    if (valid && k < d) x = rel ? __fadd_rn(E[h * d + k], rel[k]) : E[h * d + k];
                    vv[c] = x;
                    double xd = x, rd = (double)(x - tf32_trunc(x));
                    st.s2 += xd * xd;
                    st.sd2 += rd * rd;
                    st.s1 += fabs(xd);
                }
                // UMMA layout per block of `split` rows (split = 128: one block per CTA of a pair)
                *reinterpret_cast<float4*>(dst + (size_t)(i / split) * split * Kpad + stage_off<true>(i % split, kq * 4, split)) = v;
            }
            st.s2 = warp_sum_d(st.s2);
            st.sd2 = warp_sum_d(st.sd2);
            st.s1 = warp_sum_d(st.s1);
            if (lane == 0) {
                float Qn = f2up(sqrt(st.s2)), Qd = f2up(sqrt(st.sd2));
                if (rel) {
                    float thr;
                    if (norm == 1) {
                        thr = f2up(((double)theta + st.s1 * 2.384185791015625e-07) * (1.0 + (d + 2) * 1.1920928955078125e-07) *
                                   (1.0 + 9.5367431640625e-07));
                    } else {
                        double thf = (double)theta * (1.0 + 2.44140625e-04) + 2.384185791015625e-07 * sqrt(st.s2);
                        thr = f2up(thf * thf * (1.0 + (d + 3) * 1.1920928955078125e-07) * (1.0 + 9.5367431640625e-07));
                    }
                    qs[(size_t)blockIdx.x * ROWS + i] =
                        valid ? make_float4(__double2float_rn(st.s2), Qn, Qd, thr) : make_float4(3e38f, 0.f, 0.f, -1.f);
                } else {
                    // ||t||^2 / 2: the tensor-core epilogues test acc - ||t||^2/2 >= c/2 (exact rescaling)
                    T2[(size_t)tile * ROWS + i] = valid ? __double2float_rn(0.5 * st.s2) : 3e38f;
                    if (valid) {
                        tn_max = fmaxf(tn_max, Qn);
                        td_max = fmaxf(td_max, Qd);
                    }
                }
            }
        }
    } else {
        for (int g = w; g < ROWS / 32; g += NW) {
            int i = g * 32 + lane;
            long long p = t_in_rel * ROWS + i;
            bool valid = p < N;
            long long h = valid ? pr[p] : 0;
            RowStat st{0, 0, 0};
            for (int k = 0; k < Kpad; ++k) {
                float x = 0.f;
                if (valid && k < d) x = rel ? __fadd_rn(E[h * d + k], rel[k]) : E[h * d + k];
                dst[stage_off<false>(i, k, ROWS)] = x;
                double xd = x;
                st.s2 += xd * xd;
                st.s1 += fabs(xd);
            }
            if (rel) {
                float thr;
                if (norm == 1) {
                    thr = f2up(((double)theta + st.s1 * 2.384185791015625e-07) * (1.0 + (d + 2) * 1.1920928955078125e-07) *
                               (1.0 + 9.5367431640625e-07));
                } else {
                    double thf = (double)theta * (1.0 + 2.44140625e-04) + 2.384185791015625e-07 * sqrt(st.s2);
                    thr = f2up(thf * thf * (1.0 + (d + 3) * 1.1920928955078125e-07) * (1.0 + 9.5367431640625e-07));
                }
                qs[(size_t)blockIdx.x * ROWS + i] =
                    valid ? make_float4(__double2float_rn(st.s2), f2up(sqrt(st.s2)), 0.f, thr)
                          : make_float4(3e38f, 0.f, 0.f, -1.f);
            }
        }
    }
    if (!Rel && TC) {
        tn_max = warp_max_f(tn_max);
        td_max = warp_max_f(td_max);
        if (lane == 0) {
            sTn[w] = tn_max;
            sTd[w] = td_max;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            float a = 0.f, b = 0.f;
            for (int x = 0; x < NW; ++x) {
                a = fmaxf(a, sTn[x]);
                b = fmaxf(b, sTd[x]);
            }
            tstile[tile] = make_float2(a, b);
        }
    }
}

// ------------------------------------------------------ split cost estimate
// For the rank-local multi-GPU split: estimated surviving work per relation
// from Lemma 1 at element level with the zero pivot -- a histogram of tail
// keys ||t||_p (ESTB bins) and S sampled queries per relation; cost_r =
// (N / S) * sum over samples of #tails with |key(q) - key(t)| <= theta (bin
// resolution).  Integer histogram + fixed-order per-relation sums: identical
// on every rank.  Only steers load balance; never what is computed.
constexpr int ESTB = 4096, EST_S = EST_SAMPLES;

// warp per tail row (lanes over k, coalesced)
__global__ void est_tail_keys_kernel(const float* __restrict__ E, long long N, int d, int norm, float* kt,
                                     unsigned int* mm) {
    const int lane = threadIdx.x & 31;
    const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    float mn = FLT_MAX, mx = 0.f;
    for (long long i = w0; i < N; i += nw) {
        float acc = 0.f;
        for (int k = lane; k < d; k += 32) {
            const float v = E[i * d + k];
            acc = norm == 1 ? acc + fabsf(v) : fmaf(v, v, acc);
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const float key = norm == 2 ? sqrtf(acc) : acc;
        if (lane == 0) kt[i] = key;
        mn = fminf(mn, key);
        mx = fmaxf(mx, key);
    }
    if (lane == 0) {
        atomicMin(&mm[0], __float_as_uint(mn));
        atomicMax(&mm[1], __float_as_uint(mx));
    }
}

__global__ void est_hist_kernel(const float* __restrict__ kt, long long N, const unsigned int* mm, unsigned int* hist) {
    const float lo = __uint_as_float(mm[0]), hi = __uint_as_float(mm[1]);
    const float sc = hi > lo ? (float)ESTB / (hi - lo) : 0.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
        int b = (int)((kt[i] - lo) * sc);
        b = b < 0 ? 0 : (b >= ESTB ? ESTB - 1 : b);
        atomicAdd(&hist[b], 1u);
    }
}

// exclusive-to-inclusive prefix of the histogram: cum[0] = 0, cum[b + 1] = sum of hist[0..b]
// (one block of 1024 threads, 4 bins per thread; integer sums, identical on every rank)
__global__ void __launch_bounds__(1024) est_cum_kernel(const unsigned int* __restrict__ hist, unsigned int* cum) {
    __shared__ unsigned int ws[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    unsigned int v[4], sum = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) { v[i] = hist[t * 4 + i]; sum += v[i]; }
    unsigned int inc = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int x = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += x;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
        unsigned int x = ws[lane], y = x;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        ws[lane] = y - x;  // exclusive warp offsets
    }
    __syncthreads();
    unsigned int run = ws[w] + inc - sum;
    if (t == 0) cum[0] = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) { run += v[i]; cum[t * 4 + i + 1] = run; }
}

// grid (R, EST_S / 32): block y of relation r takes samples y*32 .. y*32+31, 4 per warp with the
// loads of all 4 in flight; sample s is head h = s N / EST_S, q = h + r (lanes over k); the count
// of tails within theta comes from the cumulative histogram.  Integer atomics: the per-relation
// totals are exact and order-independent, so every rank derives the same split.
__global__ void __launch_bounds__(256) est_relation_cost_kernel(const float* __restrict__ E,
                                                                const float* __restrict__ Rel, long long N, int d,
                                                                int norm, float theta, const unsigned int* mm,
                                                                const unsigned int* __restrict__ cum,
                                                                unsigned long long* cnt) {
    const long long r = blockIdx.x;
    const float lo = __uint_as_float(mm[0]), hi = __uint_as_float(mm[1]);
    const float sc = hi > lo ? (float)ESTB / (hi - lo) : 0.f;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int s0 = blockIdx.y * 32 + w * 4;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k = lane; k < d; k += 32) {
        const float rk = Rel[r * d + k];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long h = (long long)(s0 + u) * N / EST_S;
            const float v = E[h * d + k] + rk;
            acc[u] = norm == 1 ? acc[u] + fabsf(v) : fmaf(v, v, acc[u]);
        }
    }
    unsigned long long c = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        float a = acc[u];
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        const float key = norm == 2 ? sqrtf(a) : a;
        int b0 = (int)floorf((key - theta - lo) * sc), b1 = (int)floorf((key + theta - lo) * sc);
        b0 = b0 < 0 ? 0 : (b0 > ESTB ? ESTB : b0);
        b1 = b1 < -1 ? -1 : (b1 >= ESTB ? ESTB - 1 : b1);
        c += b1 >= b0 ? (unsigned long long)(cum[b1 + 1] - cum[b0]) : 0ull;
    }
    if (lane == 0) atomicAdd(&cnt[r], c);
}

void launch_split_estimate(const float* E, const float* Rel, long long N, long long R, int d, int norm, float theta,
                           float* kt, unsigned int* mm, unsigned int* hist, unsigned long long* cnt, cudaStream_t s) {
    init_minmax_kernel<<<1, 32, 0, s>>>(mm, 1);
    cudaMemsetAsync(hist, 0, 2 * (ESTB + 1) * sizeof(unsigned int), s);
    cudaMemsetAsync(cnt, 0, (size_t)R * sizeof(unsigned long long), s);
    est_tail_keys_kernel<<<grid_for(N * 32, 256, 148 * 8), 256, 0, s>>>(E, N, d, norm, kt, mm);
    est_hist_kernel<<<grid_for(N, 256), 256, 0, s>>>(kt, N, mm, hist);
    unsigned int* cum = hist + (ESTB + 1);
    est_cum_kernel<<<1, 1024, 0, s>>>(hist, cum);
    est_relation_cost_kernel<<<dim3((unsigned)R, EST_S / 32), 256, 0, s>>>(E, Rel, N, d, norm, theta, mm, cum, cnt);
}

// ------------------------------------------------------------ FP16x2 staging
// L1 FP16x2 engine operands: half2 words (dims 2p, 2p + 1) at p * ROWS + i.
// Per row: R = sum_k |v_k - fp16(v_k)| (each difference exact in FP32, sum
// rounded up) -- the exact price of the FP16 rounding in the L1 bound
// (DESIGN.md "FP16x2 L1 engine").  Queries: qs.w = (theta + 2^-23 ||q||_1 + R) gam
// (rounded up); tails: rt = R gam (rounded up).  One thread per row.
__global__ void __launch_bounds__(128) stage_half_kernel(const float* __restrict__ E, const float* __restrict__ Rel,
                                                         const int* __restrict__ perm, long long N, int d, int Kpad,
                                                         int ROWS, int QT, int tile0, float theta, float gam,
                                                         __half2* __restrict__ out, float4* __restrict__ qs,
                                                         float* __restrict__ rt) {
    const int tile = tile0 + blockIdx.x;
    long long r = 0, t_in_rel = tile;
    if (Rel) {
        r = tile / QT;
        t_in_rel = tile - r * QT;
    }
    const int* pr = perm + (Rel ? r * N : 0);
    const float* rel = Rel ? Rel + r * d : nullptr;
    __half2* dst = out + (size_t)blockIdx.x * ROWS * (Kpad / 2);
    for (int i = threadIdx.x; i < ROWS; i += blockDim.x) {
        const long long p = t_in_rel * ROWS + i;
        const bool valid = p < N;
        const long long h = valid ? pr[p] : 0;
        float res = 0.f, l1 = 0.f;
        for (int kp = 0; kp < Kpad / 2; ++kp) {
            float v[2] = {0.f, 0.f};
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int k = 2 * kp + c;
                if (valid && k < d) v[c] = rel ? __fadd_rn(E[h * d + k], rel[k]) : E[h * d + k];
            }
            const __half2 hv = __floats2half2_rn(v[0], v[1]);
            const float2 back = __half22float2(hv);
            res = __fadd_ru(res, __fadd_ru(fabsf(v[0] - back.x), fabsf(v[1] - back.y)));
            l1 = __fadd_ru(l1, __fadd_ru(fabsf(v[0]), fabsf(v[1])));
            dst[(size_t)kp * ROWS + i] = hv;
        }
        if (rel) {
            const float thr = __fmul_ru(__fadd_ru(__fadd_ru(theta, __fmul_ru(l1, 1.1920928955078125e-07f)), res), gam);
            qs[(size_t)blockIdx.x * ROWS + i] = valid ? make_float4(0.f, 0.f, res, thr) : make_float4(0.f, 0.f, 0.f, -1.f);
        } else {
            rt[(size_t)tile * ROWS + i] = valid ? __fmul_ru(res, gam) : 0.f;
        }
    }
}

void launch_stage_half(const float* E, const float* Rel, const int* perm, long long N, int d, int Kpad, int ROWS,
                       int QT, int tile0, int ntiles, float theta, float gam, void* out, float4* qs, float* rt,
                       cudaStream_t s) {
    if (ntiles <= 0) return;
    stage_half_kernel<<<ntiles, 128, 0, s>>>(E, Rel, perm, N, d, Kpad, ROWS, QT, tile0, theta, gam,
                                             reinterpret_cast<__half2*>(out), qs, rt);
}

__global__ void absmax_kernel(const float* __restrict__ E, long long nE, const float* __restrict__ Rel, long long nR,
                              unsigned int* out) {
    float m = 0.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nE + nR; i += (long long)gridDim.x * blockDim.x)
        m = fmaxf(m, fabsf(i < nE ? E[i] : Rel[i - nE]));
    m = warp_max_f(m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

void launch_absmax(const float* E, long long nE, const float* Rel, long long nR, unsigned int* out, cudaStream_t s) {
    absmax_kernel<<<grid_for(nE + nR, 256, 148 * 4), 256, 0, s>>>(E, nE, Rel, nR, out);
}

// SIMT-layout staging of query tiles (and tail tiles for the contiguous SIMT engine),
// coalesced: one block per tile, warp per row with lanes over k (row reads of E are
// whole 128-byte lines), rows parked in shared memory (stride Kpad + 1: conflict-free
// column reads), then written out column by column ([k][ROWS], consecutive threads on
// consecutive rows).  Same staged values as stage_kernel<false>; the row sums are FP32 with
// rigorous upper bounds (>= the exact sums), so thresholds stay upper bounds.  The old kernel gave every lane a
// whole row and walked k: 32 rows per load instruction, two active warps per block
// (c2 L1 queries 0.44 ms).
template <int ROWS>
__global__ void __launch_bounds__(256) stage_simt_kernel(const float* __restrict__ E, const float* __restrict__ Rel,
                                                         const int* __restrict__ perm, long long N, int d, int Kpad,
                                                         int QT, int tile0, int norm, float theta,
                                                         float* __restrict__ out, float4* __restrict__ qs,
                                                         float* __restrict__ T2, int cyc_world, int cyc_rank) {
    extern __shared__ float ss_smem[];  // [ROWS][Kpad + 1]
    const int tile = tile0 + blockIdx.x;
    if (cyc_world > 1 && tile % cyc_world != cyc_rank) return;
    long long r = 0, t_in_rel = tile;
    if (Rel) {
        r = tile / QT;
        t_in_rel = tile - r * QT;
    }
    const int* pr = perm + (Rel ? r * N : 0);
    const float* rel = Rel ? Rel + r * d : nullptr;
    const int LDS = Kpad + 1;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
    for (int i = w; i < ROWS; i += NW) {
        const long long p = t_in_rel * ROWS + i;
        const bool valid = p < N;
        const long long h = valid ? pr[p] : 0;
        // FP32 sums (FP64 conversions issue at 1/8 of the FFMA rate), then rigorous upper bounds:
        // any-order sums of d nonnegative terms err by <= (d - 1) 2^-24 relative, the squares by 2^-24 more
        float f2 = 0.f, f1 = 0.f;
        for (int k = lane; k < Kpad; k += 32) {
            float x = 0.f;
            if (valid && k < d) x = rel ? __fadd_rn(__ldg(E + h * d + k), __ldg(rel + k)) : __ldg(E + h * d + k);
            ss_smem[i * LDS + k] = x;
            f2 = fmaf(x, x, f2);
            f1 += fabsf(x);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            f2 += __shfl_xor_sync(0xffffffffu, f2, o);
            f1 += __shfl_xor_sync(0xffffffffu, f1, o);
        }
        const double s2 = (double)f2 * (1.0 + (d + 2) * 5.9604644775390625e-08);
        const double s1 = (double)f1 * (1.0 + (d + 1) * 5.9604644775390625e-08);
        if (lane == 0) {
            if (rel) {
                float thr;
                if (norm == 1) {
                    thr = f2up((theta + s1 * 2.384185791015625e-07) * (1.0 + (d + 2) * 1.1920928955078125e-07) *
                               (1.0 + 9.5367431640625e-07));
                } else {
                    const double thf = (double)theta * (1.0 + 2.44140625e-04) + 2.384185791015625e-07 * sqrt(s2);
                    thr = f2up(thf * thf * (1.0 + (d + 3) * 1.1920928955078125e-07) * (1.0 + 9.5367431640625e-07));
                }
                qs[(size_t)blockIdx.x * ROWS + i] =
                    valid ? make_float4(__double2float_rn(s2), f2up(sqrt(s2)), 0.f, thr) : make_float4(3e38f, 0.f, 0.f, -1.f);
            }
        }
    }
    __syncthreads();
    float* dst = out + (size_t)blockIdx.x * ROWS * Kpad;
    static_assert(256 % ROWS == 0, "whole rows per pass");
    const int i = threadIdx.x % ROWS;
    for (int k = threadIdx.x / ROWS; k < Kpad; k += 256 / ROWS)
        dst[k * ROWS + i] = ss_smem[i * LDS + k];  // SIMT layout: element (i, k) at k * ROWS + i
}

// the coalesced SIMT staging parks a whole tile in shared memory (<= 100 KB)
static bool stage_simt_ok(int rows, int Kpad) {
    const size_t smem = (size_t)rows * (Kpad + 1) * 4;
    if (rows != SIMT_T || smem > 100 * 1024) return false;
    cudaFuncSetAttribute(stage_simt_kernel<SIMT_T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return true;
}

void launch_stage_tails(const float* E, const int* tperm, long long N, int d, int Kpad, int BN, int TT, int tc_layout,
                        float* Tp, float* T2, float2* tstile, cudaStream_t s) {
    if (TT <= 0) return;
    if (tc_layout)
        stage_kernel<true><<<TT, 1024, 0, s>>>(E, nullptr, tperm, N, d, Kpad, BN, 1, 0, 2, 0.f, Tp, nullptr, T2, tstile,
                                              tc_layout == 2 ? BN / 2 : BN);
    else if (stage_simt_ok(BN, Kpad))
        stage_simt_kernel<SIMT_T><<<TT, 256, (size_t)BN * (Kpad + 1) * 4, s>>>(E, nullptr, tperm, N, d, Kpad, 1, 0, 2,
                                                                              0.f, Tp, nullptr, T2, 0, 0);
    else
        stage_kernel<false><<<TT, 256, 0, s>>>(E, nullptr, tperm, N, d, Kpad, BN, 1, 0, 2, 0.f, Tp, nullptr, T2, tstile,
                                               BN);
}

void launch_stage_queries(const float* E, const float* Rel, const int* qperm, long long N, int d, int Kpad, int QT,
                          int bq, int tq0, int tq1, int tc_layout, int norm, float theta, float* Qp, float4* qs,
                          cudaStream_t s, int cyc_world, int cyc_rank) {
    if (tq1 <= tq0) return;
    if (tc_layout)
        stage_kernel<true><<<tq1 - tq0, 256, 0, s>>>(E, Rel, qperm, N, d, Kpad, bq, QT, tq0, norm, theta, Qp, qs,
                                                     nullptr, nullptr, bq, cyc_world, cyc_rank);
    else if (stage_simt_ok(bq, Kpad))
        stage_simt_kernel<SIMT_T><<<tq1 - tq0, 256, (size_t)bq * (Kpad + 1) * 4, s>>>(E, Rel, qperm, N, d, Kpad, QT,
                                                                                     tq0, norm, theta, Qp, qs, nullptr,
                                                                                     cyc_world, cyc_rank);
    else
        stage_kernel<false><<<tq1 - tq0, 256, 0, s>>>(E, Rel, qperm, N, d, Kpad, bq, QT, tq0, norm, theta, Qp, qs,
                                                      nullptr, nullptr, bq, cyc_world, cyc_rank);
}

// ------------------------------------------------ relation-factored L2 tables
// (tiles_tc.cu MODE 2).  One warp per (relation, row), lanes
// over k, FP64 sums of the fp32 inputs:
//   fz[r][h]  = (||E_h + Rel_r||^2 - theta^2) / 2, rounded down (h + r formed in FP64)
//   frt[r][j] = Rel_r . E_t for the sorted tail t = tperm[j], rounded to nearest (0 for j >= N)
//   frn[r]    = ||Rel_r||, rounded up
__global__ void factored_tables_kernel(const float* __restrict__ E, const float* __restrict__ Rel,
                                       const int* __restrict__ tperm, long long N, long long R, int d, double theta,
                                       long long ntpad, float* __restrict__ fz, float* __restrict__ frt,
                                       float* __restrict__ frn, unsigned int* __restrict__ nonfinite) {
    const int lane = threadIdx.x & 31;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long total = R * ntpad;
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < total; w += nw) {
        const long long r = w / ntpad, j = w - r * ntpad;
        const float* rel = Rel + r * d;
        double z = 0.0, rt = 0.0, rr = 0.0;
        if (j < N) {
            const float* eh = E + j * d;                    // fz: natural head order
            const float* et = E + (long long)tperm[j] * d;  // frt: sorted tail order
            for (int k = lane; k < d; k += 32) {
                const double a = (double)eh[k] + (double)rel[k];
                z += a * a;
                rt += (double)rel[k] * (double)et[k];
                if (j == 0) rr += (double)rel[k] * (double)rel[k];
            }
        }
        z = warp_sum_d(z);
        rt = warp_sum_d(rt);
        rr = warp_sum_d(rr);
        if (lane == 0) {
            if (j < N && !(isfinite(z) && isfinite(rt))) atomicOr(nonfinite, 1u);  // any non-finite E or Rel
            if (j < N) fz[r * N + j] = __double2float_rd(0.5 * (z - theta * theta));
            frt[r * ntpad + j] = j < N ? __double2float_rn(rt) : 0.f;
            if (j == 0) frn[r] = __double2float_ru(sqrt(rr));
        }
    }
}

__global__ void iota_kernel(int* out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = (int)i;
}

void launch_factored_tables(const float* E, const float* Rel, const int* tperm, long long N, long long R, int d,
                            float theta, long long ntpad, float* fz, float* frt, float* frn, unsigned int* nonfinite,
                            cudaStream_t s) {
    factored_tables_kernel<<<grid_for(R * ntpad * 32, 256), 256, 0, s>>>(E, Rel, tperm, N, R, d, (double)theta, ntpad,
                                                                       fz, frt, frn, nonfinite);
}

void launch_iota(int* out, long long n, cudaStream_t s) { iota_kernel<<<grid_for(n, 256), 256, 0, s>>>(out, n); }

}  // namespace kgc
