// topk.cu -- the k smallest dist3 over all N*R*N triplets (SURVEY §8(f) row 4,
// "top-k / top-1 min-join"; the paper's minimum-distance statistic
// "min_{i,j,k} ||h_i + r_j - t_k||", with or without self edges).
//
// Built on the epsilon-join (kgc_api.cu::kgc_topk):
//   1. sample_dist: FP64 dist3 of S sampled query rows against EVERY tail,
//      rounded up to float (with a 2^-40 relative margin over the FP64 value, so
//      each stored value is >= the distance K6 will compute for that triplet).
//   2. theta = the k-th smallest sampled value (bisection on the float bit
//      pattern with count_le): k actual triplets lie within theta, so the join at
//      theta returns at least k triplets -- no iteration, no guessing.
//   3. the join at theta (all of K1-K7), then the k-th smallest returned distance
//      by the same bisection, compaction of the records within it, final order
//      (dist, h, r, t) on the host.
#include <cfloat>

#include "common.cuh"

namespace kgc {

// grid (ceil(N / 64), ceil(S / 32)); block 256: a tile of 64 tails against 32 sampled query
// rows, dims in chunks of TK_K staged in shared memory (E_h and Rel_r kept separately so
// q = h + r is formed in FP64 like K6); thread = one tail x 8 query rows
constexpr int TK_T = 64, TK_Q = 32, TK_K = 64;
__global__ void __launch_bounds__(256) sample_dist_kernel(const float* __restrict__ E, const float* __restrict__ Rel,
                                                          long long N, long long R, int d, int norm, int S,
                                                          int exclude_self, float* __restrict__ out) {
    __shared__ float Ts[TK_T][TK_K + 1];
    __shared__ float Hs[TK_Q][TK_K + 1];
    __shared__ float Rs[TK_Q][TK_K + 1];
    __shared__ long long hrow[TK_Q];
    const long long t0 = (long long)blockIdx.x * TK_T;
    const int s0 = blockIdx.y * TK_Q;
    const long long NR = N * R;
    if (threadIdx.x < TK_Q) {
        const int s = s0 + threadIdx.x;
        hrow[threadIdx.x] = s < S ? ((long long)s * NR / S) : -1;  // sampled row id = h * R + r
    }
    const int ti = threadIdx.x & (TK_T - 1), qg = threadIdx.x >> 6;  // 4 groups of 8 query rows
    double acc[TK_Q / 4];
#pragma unroll
    for (int u = 0; u < TK_Q / 4; ++u) acc[u] = 0.0;
    for (int k0 = 0; k0 < d; k0 += TK_K) {
        const int kl = d - k0 < TK_K ? d - k0 : TK_K;
        __syncthreads();
        for (int x = threadIdx.x; x < TK_T * kl; x += blockDim.x) {
            const int i = x / kl, k = x % kl;
            Ts[i][k] = t0 + i < N ? E[(t0 + i) * d + k0 + k] : 0.f;
        }
        for (int x = threadIdx.x; x < TK_Q * kl; x += blockDim.x) {
            const int i = x / kl, k = x % kl;
            const long long row = hrow[i];
            Hs[i][k] = row >= 0 ? E[(row / R) * d + k0 + k] : 0.f;
            Rs[i][k] = row >= 0 ? Rel[(row % R) * d + k0 + k] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < TK_Q / 4; ++u) {
            const int qi = qg * (TK_Q / 4) + u;
            double a = acc[u];
            for (int k = 0; k < kl; ++k) {
                const double x = ((double)Hs[qi][k] + (double)Rs[qi][k]) - (double)Ts[ti][k];
                a += norm == 1 ? fabs(x) : x * x;
            }
            acc[u] = a;
        }
    }
    const long long t = t0 + ti;
    if (t >= N) return;
#pragma unroll
    for (int u = 0; u < TK_Q / 4; ++u) {
        const int qi = qg * (TK_Q / 4) + u;
        const long long row = hrow[qi];
        if (row < 0) continue;
        const double dist = norm == 2 ? sqrt(acc[u]) : acc[u];
        const bool self = exclude_self && (row / R) == t;
        out[(size_t)(s0 + qi) * N + t] = self ? FLT_MAX : f2up(dist * (1.0 + 9.094947017729282e-13));
    }
}

// number of values <= theta (values >= FLT_MAX never counted)
__global__ void count_le_kernel(const float* __restrict__ a, long long n, float theta, unsigned long long* cnt) {
    unsigned long long c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        c += (a[i] <= theta && a[i] < FLT_MAX);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

// the same over result records (optionally skipping self edges)
__global__ void count_res_le_kernel(const KgcTripletDev* __restrict__ res, long long n, float theta, int exclude_self,
                                    unsigned long long* cnt) {
    unsigned long long c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const KgcTripletDev o = res[i];
        c += (o.dist <= theta && !(exclude_self && o.h == o.t));
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

__global__ void compact_res_le_kernel(const KgcTripletDev* __restrict__ res, long long n, float theta,
                                      int exclude_self, KgcTripletDev* __restrict__ out, unsigned long long* cnt,
                                      long long cap) {
    for (long long i0 = blockIdx.x * (long long)blockDim.x; i0 < n; i0 += (long long)gridDim.x * blockDim.x) {
        const long long i = i0 + threadIdx.x;
        bool keep = false;
        KgcTripletDev o{};
        if (i < n) {
            o = res[i];
            keep = o.dist <= theta && !(exclude_self && o.h == o.t);
        }
        const unsigned long long slot = warp_append(keep, cnt);
        if (keep && slot < (unsigned long long)cap) out[slot] = o;
    }
}

static unsigned grid_tk(long long n) {
    long long g = (n + 255) / 256;
    return (unsigned)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

void launch_sample_dist(const float* E, const float* Rel, long long N, long long R, int d, int norm, int S,
                        int exclude_self, float* out, cudaStream_t s) {
    dim3 grid((unsigned)((N + TK_T - 1) / TK_T), (unsigned)((S + TK_Q - 1) / TK_Q));
    sample_dist_kernel<<<grid, 256, 0, s>>>(E, Rel, N, R, d, norm, S, exclude_self, out);
}

void launch_count_le(const float* a, long long n, float theta, unsigned long long* cnt, cudaStream_t s) {
    cudaMemsetAsync(cnt, 0, 8, s);
    count_le_kernel<<<grid_tk(n), 256, 0, s>>>(a, n, theta, cnt);
}

void launch_count_res_le(const KgcTripletDev* res, long long n, float theta, int exclude_self,
                         unsigned long long* cnt, cudaStream_t s) {
    cudaMemsetAsync(cnt, 0, 8, s);
    count_res_le_kernel<<<grid_tk(n), 256, 0, s>>>(res, n, theta, exclude_self, cnt);
}

void launch_compact_res_le(const KgcTripletDev* res, long long n, float theta, int exclude_self, KgcTripletDev* out,
                           unsigned long long* cnt, long long cap, cudaStream_t s) {
    cudaMemsetAsync(cnt, 0, 8, s);
    compact_res_le_kernel<<<grid_tk(n), 256, 0, s>>>(res, n, theta, exclude_self, out, cnt, cap);
}

}  // namespace kgc
