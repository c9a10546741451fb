// verify.cu -- K6 + K7: exact re-check of every candidate and compaction of
// the results.
//
// "Finally, we compute the similarity values ... verify if the results are
// valid and return the valid results" (Fig. algo1 line 17,
// PAPER.md:369).  Each candidate (sorted query row, sorted tail) is mapped
// back through the permutations (h = pi_r[i], t = pi_T[j]) and its distance
// dist3(h, r, t) = ||h + r - t||_p is recomputed from the
// ORIGINAL fp32 embeddings in FP64 (VERIFY_LPC lanes per candidate, lanes over
// k, shuffle tree; 1 by default: one lane per candidate, k in order).  Kept iff dist <= theta (inclusive); emitted as
// {h, r, t, (float)dist} with one atomic per warp per 32 candidates.
#include "common.cuh"

#ifndef VERIFY_LPC
#define VERIFY_LPC 1
#endif

namespace kgc {

// One warp verifies 32 candidates per round.  Stage 1: lane l loads
// candidate base + l and maps it through the permutations (one independent
// load chain per lane, all 32 in flight together).  Stage 2: the LPC lanes of
// group g compute the distances of candidates g*LPC .. g*LPC+LPC-1 (lanes over
// k, FP64 partial sums, log2(LPC)-step shuffle tree); the sum of candidate c
// lands back in lane c.  Stage 3: warp-aggregated append of the kept
// candidates in candidate order.  No data-dependent branches in stage 2, so
// the loads of consecutive k overlap; E_h and Rel_r repeat across consecutive
// candidates of one query row and hit L1.  Measured on c2 (L2 / L1 verify ms):
// LPC 8 0.71 / 0.48 (the shuffles saturated the MIO queue), 4 0.51 / 0.35,
// 2 0.48 / 0.33, 1 0.47 / 0.33.
template <int NORM, bool VEC4>
__global__ void __launch_bounds__(256, 3) verify_kernel(const int2* __restrict__ cand,
                                                        const unsigned long long* __restrict__ cand_count,
                                                        long long cand_cap, const int* __restrict__ qperm,
                                                        const int* __restrict__ tperm, const float* __restrict__ E,
                                                        const float* __restrict__ Rel, const float* __restrict__ Et,
                                                        long long N, int QT, int bq,
                                                        int d, double theta, KgcTripletDev* __restrict__ out,
                                                        unsigned long long* res_count, long long res_cap, int r_off,
                                                        long long Nt, long long t_off, long long h_off) {
    long long nc = (long long)*cand_count;
    if (nc > cand_cap) nc = cand_cap;
    constexpr int LPC = VERIFY_LPC;  // lanes per candidate
    const int lane = threadIdx.x & 31, g = lane / LPC, s = lane % LPC;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long rows_per_rel = (long long)QT * bq;
    for (long long base = warp * 32; base < nc; base += nwarps * 32) {
        // ---- stage 1: this lane's candidate
        const long long idx = base + lane;
        bool valid = idx < nc;
        int h = 0, r = 0, t = 0;  // h: row of E, t: row of Et
        if (valid) {
            const int2 cv = cand[idx];
            const long long rr = cv.x / rows_per_rel;
            const long long pos = cv.x - rr * rows_per_rel;
            valid = pos < N && cv.y < Nt;
            if (valid) {
                r = (int)rr;
                h = qperm ? qperm[rr * N + pos] : (int)pos;  // null: natural order
                t = tperm ? tperm[cv.y] : cv.y;
            }
        }
        // ---- stage 2: distances, LPC lanes per candidate
        double mine = 0.0;
#pragma unroll
        for (int it = 0; it < LPC; ++it) {
            const int src = g * LPC + it;
            const int hh = __shfl_sync(0xffffffffu, h, src);
            const int rq = __shfl_sync(0xffffffffu, r, src);
            const int tt = __shfl_sync(0xffffffffu, t, src);
            const float* eh = E + (long long)hh * d;
            const float* er = Rel + (long long)rq * d;
            const float* et = Et + (long long)tt * d;
            double acc = 0.0;
            if (VEC4) {
#pragma unroll 2
                for (int k = s * 4; k < d; k += 4 * LPC) {
                    const float4 a = __ldg(reinterpret_cast<const float4*>(eh + k));
                    const float4 b = __ldg(reinterpret_cast<const float4*>(er + k));
                    const float4 c = __ldg(reinterpret_cast<const float4*>(et + k));
                    const double x0 = ((double)a.x + (double)b.x) - (double)c.x;  // (h + r) - t, FP64
                    const double x1 = ((double)a.y + (double)b.y) - (double)c.y;
                    const double x2 = ((double)a.z + (double)b.z) - (double)c.z;
                    const double x3 = ((double)a.w + (double)b.w) - (double)c.w;
                    if (NORM == 1) acc += fabs(x0) + fabs(x1) + fabs(x2) + fabs(x3);
                    else acc += x0 * x0 + x1 * x1 + x2 * x2 + x3 * x3;
                }
            } else {
                for (int k = s; k < d; k += LPC) {
                    const double x = ((double)__ldg(eh + k) + (double)__ldg(er + k)) - (double)__ldg(et + k);
                    acc += NORM == 1 ? fabs(x) : x * x;
                }
            }
#pragma unroll
            for (int o = LPC / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (s == it) mine = acc;  // lane g*LPC + it owns candidate g*LPC + it
        }
        // ---- stage 3: keep iff dist <= theta (inclusive); append in candidate order
        const double dist = NORM == 2 ? sqrt(mine) : mine;
        const bool keep = valid && dist <= theta;
        const unsigned long long slot = warp_append(keep, res_count);
        if (keep && slot < (unsigned long long)res_cap) {
            KgcTripletDev o;
            o.h = (int)(h + h_off);  // global ids: head block / tail partition offsets,
            o.r = r + r_off;         // relation index in the caller's Rel
            o.t = (int)(t + t_off);
            o.dist = (float)dist;
            out[slot] = o;
        }
    }
}

void launch_verify(const int2* cand, const unsigned long long* cand_count, long long cand_cap, const int* qperm,
                   const int* tperm, const float* E, const float* Rel, const float* Et, long long N, int QT, int bq,
                   int d, int norm, float theta, KgcTripletDev* out, unsigned long long* res_count, long long res_cap,
                   int num_sms, cudaStream_t s, int r_off, long long Nt, long long t_off, long long h_off) {
    const bool vec4 = (d % 4 == 0) && ((reinterpret_cast<uintptr_t>(E) | reinterpret_cast<uintptr_t>(Rel) |
                                        reinterpret_cast<uintptr_t>(Et)) % 16 == 0);
    auto kern = norm == 1 ? (vec4 ? verify_kernel<1, true> : verify_kernel<1, false>)
                          : (vec4 ? verify_kernel<2, true> : verify_kernel<2, false>);
    kern<<<num_sms * 8, 256, 0, s>>>(cand, cand_count, cand_cap, qperm, tperm, E, Rel, Et, N, QT, bq, d,
                                     (double)theta, out, res_count, res_cap, r_off, Nt < 0 ? N : Nt, t_off, h_off);
}

}  // namespace kgc
