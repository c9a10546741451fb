// verify.cu -- K6 + K7: exact re-check of every candidate and compaction of
// the results.
//
// "Finally, we compute the similarity values ... verify if the results are
// valid and return the valid results" (Fig. algo1 line 17,
// PAPER.md:369).  Each candidate (sorted query row, sorted tail) is mapped
// back through the permutations (h = pi_r[i], t = pi_T[j]) and its distance
// dist3(h, r, t) = ||h + r - t||_p is recomputed from the
// ORIGINAL fp32 embeddings in FP64 (one warp per candidate, lanes over k,
// warp-shuffle tree).  Kept iff dist <= theta (inclusive);
// emitted as {h, r, t, (float)dist} with one atomic per warp.
#include "common.cuh"

namespace kgc {

__device__ __forceinline__ double warp_sum_dd(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(256) verify_kernel(const int2* __restrict__ cand,
                                                     const unsigned long long* __restrict__ cand_count,
                                                     long long cand_cap, const int* __restrict__ qperm,
                                                     const int* __restrict__ tperm, const float* __restrict__ E,
                                                     const float* __restrict__ Rel, long long N, int QT, int d,
                                                     int norm, double theta, KgcTripletDev* __restrict__ out,
                                                     unsigned long long* res_count, long long res_cap) {
    long long nc = (long long)*cand_count;
    if (nc > cand_cap) nc = cand_cap;
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long rows_per_rel = (long long)QT * BM;
    for (long long g = warp; g * 32 < nc; g += nwarps) {
        const long long idx = g * 32 + lane;
        bool valid = idx < nc;
        int h = 0, r = 0, t = 0;
        if (valid) {
            const int2 cv = cand[idx];
            const long long rr = cv.x / rows_per_rel;
            const long long pos = cv.x - rr * rows_per_rel;
            valid = pos < N && cv.y < N;
            if (valid) {
                r = (int)rr;
                h = qperm[rr * N + pos];
                t = tperm[cv.y];
            }
        }
        const int n_here = (int)min(32LL, nc - g * 32);
        double mine = 0.0;
        for (int c = 0; c < n_here; ++c) {
            const int hc = __shfl_sync(0xffffffffu, h, c);
            const int rc = __shfl_sync(0xffffffffu, r, c);
            const int tc = __shfl_sync(0xffffffffu, t, c);
            const float* eh = E + (long long)hc * d;
            const float* er = Rel + (long long)rc * d;
            const float* et = E + (long long)tc * d;
            double s = 0.0;
            for (int k = lane; k < d; k += 32) {
                const double q = (double)eh[k] + (double)er[k];   // connector_1(h, r) = h + r
                const double x = q - (double)et[k];              // - connector_2(t, r) = t
                s += norm == 1 ? fabs(x) : x * x;
            }
            s = warp_sum_dd(s);
            if (lane == c) mine = s;
        }
        const double dist = norm == 2 ? sqrt(mine) : mine;
        const bool keep = valid && dist <= theta;
        const unsigned long long slot = warp_append(keep, res_count);
        if (keep && slot < (unsigned long long)res_cap) {
            KgcTripletDev o;
            o.h = h;
            o.r = r;
            o.t = t;
            o.dist = (float)dist;
            out[slot] = o;
        }
    }
}

void launch_verify(const int2* cand, const unsigned long long* cand_count, long long cand_cap, const int* qperm,
                   const int* tperm, const float* E, const float* Rel, long long N, int QT, int d, int norm,
                   float theta, KgcTripletDev* out, unsigned long long* res_count, long long res_cap, int num_sms,
                   cudaStream_t s) {
    verify_kernel<<<num_sms * 8, 256, 0, s>>>(cand, cand_count, cand_cap, qperm, tperm, E, Rel, N, QT, d, norm,
                                              (double)theta, out, res_count, res_cap);
}

}  // namespace kgc
