// se.cu -- Structured Embedding (SE) on the same join (the
// paper's second model): dist3(h, r, t) = ||W_r^lhs h - W_r^rhs t||_1
// with connector_1(h, r) = W_r^lhs h, connector_2(t, r) = W_r^rhs t and
// dist = L1, so "SE is also transformable to a metric space" and the join applies
// per relation with a relation-specific TAIL side (unlike TransE).
//
// Per relation (kgc_api.cu::kgc_join_se):
//   se_connector_kernel  A = E W_lhs^T and B = E W_rhs^T in FP64 (index-order
//                        sums), kept in FP64 for the exact re-check and rounded
//                        once to fp32 for the filters; max_h ||fl(a_h)||_1 per side
//   the L1 join of fl(A) (queries) against fl(B) (tails): keys, sorts, tile
//                        pruning, FP32 SIMT tiles -- with theta widened by the
//                        rounding of both sides (2^-24 (max||a||_1 + max||b||_1))
//   verify_se_kernel     FP64 sum |A_h - B_t| from the FP64 connectors; keep iff
//                        <= theta, emit {h, r, t, dist}
#include "common.cuh"

namespace kgc {

// grid (ceil(N / 32), ceil(d / 32)), block 32 x 32: thread (ty, tx) computes row h0 + ty,
// output dim k0 + tx of both connectors; inputs staged in 96-wide chunks of j
constexpr int SE_T = 32, SE_J = 96;
__global__ void __launch_bounds__(1024) se_connector_kernel(const float* __restrict__ E, const float* __restrict__ Wl,
                                                            const float* __restrict__ Wr, long long N, int d,
                                                            double* __restrict__ A64, double* __restrict__ B64,
                                                            float* __restrict__ Af, float* __restrict__ Bf) {
    __shared__ float Es[SE_T][SE_J + 1];
    __shared__ float Ls[SE_T][SE_J + 1];
    __shared__ float Rs[SE_T][SE_J + 1];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const long long h0 = (long long)blockIdx.x * SE_T;
    const int k0 = blockIdx.y * SE_T;
    double a = 0.0, b = 0.0;
    for (int j0 = 0; j0 < d; j0 += SE_J) {
        const int jl = d - j0 < SE_J ? d - j0 : SE_J;
        __syncthreads();
        for (int j = tx; j < jl; j += SE_T) {
            Es[ty][j] = h0 + ty < N ? E[(h0 + ty) * d + j0 + j] : 0.f;
            Ls[ty][j] = k0 + ty < d ? Wl[(long long)(k0 + ty) * d + j0 + j] : 0.f;
            Rs[ty][j] = k0 + ty < d ? Wr[(long long)(k0 + ty) * d + j0 + j] : 0.f;
        }
        __syncthreads();
        for (int j = 0; j < jl; ++j) {  // index order, as the oracle
            const double e = Es[ty][j];
            a = fma((double)Ls[tx][j], e, a);
            b = fma((double)Rs[tx][j], e, b);
        }
    }
    const long long h = h0 + ty;
    const int k = k0 + tx;
    if (h < N && k < d) {
        A64[h * d + k] = a;
        B64[h * d + k] = b;
        Af[h * d + k] = __double2float_rn(a);
        Bf[h * d + k] = __double2float_rn(b);
    }
}

// max over rows of ||x_h||_1 (FP64 sums, rounded up), as float bits (values >= 0); a
// non-finite connector (NaN or inf in E, W_lhs or W_rhs) gives +inf, which the host
// reports as KGC_EDATA
__global__ void row_l1_max_kernel(const double* __restrict__ X, long long N, int d, unsigned int* out) {
    const int lane = threadIdx.x & 31;
    float m = 0.f;
    for (long long h = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; h < N;
         h += ((long long)gridDim.x * blockDim.x) >> 5) {
        double s = 0.0;
        for (int k = lane; k < d; k += 32) s += fabs(X[h * d + k]);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        m = isfinite(s) ? fmaxf(m, f2up(s)) : __int_as_float(0x7f800000);  // NaN / inf -> +inf: KGC_EDATA
    }
    if (lane == 0) atomicMax(out, __float_as_uint(m));
}

// as verify_kernel (verify.cu), distances from the FP64 connectors
__global__ void __launch_bounds__(256) verify_se_kernel(const int2* __restrict__ cand,
                                                        const unsigned long long* __restrict__ cand_count,
                                                        long long cand_cap, const int* __restrict__ qperm,
                                                        const int* __restrict__ tperm, const double* __restrict__ A64,
                                                        const double* __restrict__ B64, long long N, long long rows,
                                                        int d, double theta, KgcTripletDev* __restrict__ out,
                                                        unsigned long long* res_count, long long res_cap, int r) {
    long long nc = (long long)*cand_count;
    if (nc > cand_cap) nc = cand_cap;
    const int lane = threadIdx.x & 31, g = lane >> 3, s = lane & 7;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long base = warp * 32; base < nc; base += nwarps * 32) {
        const long long idx = base + lane;
        bool valid = idx < nc;
        int h = 0, t = 0;
        if (valid) {
            const int2 cv = cand[idx];
            valid = cv.x < rows && cv.x < N && cv.y < N;
            if (valid) {
                h = qperm[cv.x];
                t = tperm[cv.y];
            }
        }
        double mine = 0.0;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            const int src = g * 8 + it;
            const int hh = __shfl_sync(0xffffffffu, h, src);
            const int tt = __shfl_sync(0xffffffffu, t, src);
            const double* a = A64 + (long long)hh * d;
            const double* b = B64 + (long long)tt * d;
            double acc = 0.0;
            for (int k = s; k < d; k += 8) acc += fabs(a[k] - b[k]);
            acc += __shfl_xor_sync(0xffffffffu, acc, 4);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            if (s == it) mine = acc;
        }
        const bool keep = valid && mine <= theta;
        const unsigned long long slot = warp_append(keep, res_count);
        if (keep && slot < (unsigned long long)res_cap) {
            KgcTripletDev o;
            o.h = h;
            o.r = r;
            o.t = t;
            o.dist = (float)mine;
            out[slot] = o;
        }
    }
}

void launch_se_connectors(const float* E, const float* Wl, const float* Wr, long long N, int d, double* A64,
                          double* B64, float* Af, float* Bf, unsigned int* maxa, unsigned int* maxb, cudaStream_t s) {
    dim3 grid((unsigned)((N + SE_T - 1) / SE_T), (unsigned)((d + SE_T - 1) / SE_T));
    se_connector_kernel<<<grid, dim3(SE_T, SE_T), 0, s>>>(E, Wl, Wr, N, d, A64, B64, Af, Bf);
    cudaMemsetAsync(maxa, 0, 4, s);
    cudaMemsetAsync(maxb, 0, 4, s);
    long long g = (N * 32 + 255) / 256;
    g = g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g);
    row_l1_max_kernel<<<(unsigned)g, 256, 0, s>>>(A64, N, d, maxa);
    row_l1_max_kernel<<<(unsigned)g, 256, 0, s>>>(B64, N, d, maxb);
}

void launch_verify_se(const int2* cand, const unsigned long long* cand_count, long long cand_cap, const int* qperm,
                      const int* tperm, const double* A64, const double* B64, long long N, long long rows, int d,
                      float theta, KgcTripletDev* out, unsigned long long* res_count, long long res_cap, int num_sms,
                      cudaStream_t s, int r) {
    verify_se_kernel<<<num_sms * 8, 256, 0, s>>>(cand, cand_count, cand_cap, qperm, tperm, A64, B64, N, rows, d,
                                                 (double)theta, out, res_count, res_cap, r);
}

}  // namespace kgc
