// verify.cu -- K6 + K7: exact re-check of every candidate and compaction of
// the results.
//
// "Finally, we compute the similarity values ... verify if the results are
// valid and return the valid results" (Fig. algo1 line 17,
// PAPER.md:369).  Each candidate (sorted query row, sorted tail) is mapped
// back through the permutations (h = pi_r[i], t = pi_T[j]) and its distance
// dist3(h, r, t) = ||h + r - t||_p is recomputed from the
// ORIGINAL fp32 embeddings: in FP32 with a rigorous error bound, and in FP64
// (index-order sum, as the oracle) wherever the bound cannot decide.  Kept iff
// dist <= theta (inclusive); emitted as {h, r, t, dist} with one
// atomic per warp per 32 candidates.
#include "common.cuh"

namespace kgc {

// FP64 dist3 of one candidate (index-order sum, as the oracle): the exact decision.
template <int NORM>
__device__ __forceinline__ double dist_f64(const float* __restrict__ eh, const float* __restrict__ er,
                                           const float* __restrict__ et, int d) {
    double acc = 0.0;
    for (int k = 0; k < d; ++k) {
        const double x = ((double)__ldg(eh + k) + (double)__ldg(er + k)) - (double)__ldg(et + k);  // (h + r) - t
        acc += NORM == 1 ? fabs(x) : x * x;
    }
    return NORM == 2 ? sqrt(acc) : acc;
}

// One lane per candidate, 32 candidates per warp round.  Stage 1: the candidate and its
// permutation lookups (one independent load chain per lane).  Stage 2 (rows 16-byte aligned,
// d % 4 == 0): FP32 first -- y = fl(fl(h - t) + r) per dimension (two packed FP32 ops per two
// dims: FFMA2 with -1 for h - t, FADD2 for + r) and the sums of y^2 (or |y|) and a^2 (or |a|),
// a = fl(h - t).  With u = 2^-24, |y_k - x_k| <= u/(1-u) (|y_k| + |a_k|) for the exact
// x = h + r - t, so (triangle inequality, FP32 sums of n = d/2 + 2 terms per partial)
//   |dist32 - dist| <= B = u ((d/4 + 8) dist32 + 2 ||a||_2)        (L2)
//   |dist32 - dist| <= B = u ((d/2 + 8) dist32 + 2 ||a||_1)        (L1)
// (rounded up by 1 + 2^-10).  The decision is taken in FP32 when |dist32 - theta| > B and the
// reported distance is dist32 when B <= 8e-6 max(dist32, theta) (within the 1e-5 bar);
// every other candidate -- near theta, or operands whose ||a|| is huge against dist -- goes
// through the FP64 index-order sum.
//
// Data movement.  The 32 tail rows of a round are 32 different rows of E; read lane by lane
// they made every load instruction touch 32 cache lines and the L1 data stage saturated (ncu,
// c4: l1tex data-pipe wavefronts 88% of peak, 2.6 ms for 1.5e7 candidates).  So the warp stages
// them in shared memory per 32-float K-chunk with cp.async (8 lanes per 128-byte row chunk: 4
// lines per instruction), double-buffered, and each lane reads its row there (row stride 36
// floats: conflict-free float4 reads).  E_h and Rel_r stay direct loads (consecutive
// candidates mostly share the query row).  Kept records of VB rounds are staged per warp and
// appended with one atomic.
constexpr int VB = 4;   // 32-candidate rounds per warp between result appends
constexpr int VKC = 32; // floats per staged K-chunk of a tail row
constexpr int VST = 36; // staged row stride (floats)
template <int NORM, bool VEC4>
__global__ void __launch_bounds__(256, 2) verify_kernel(const int2* __restrict__ cand,
                                                        const unsigned long long* __restrict__ cand_count,
                                                        long long cand_cap, const int* __restrict__ qperm,
                                                        const int* __restrict__ tperm, const float* __restrict__ E,
                                                        const float* __restrict__ Rel, const float* __restrict__ Et,
                                                        long long N, int QT, int bq,
                                                        int d, double theta, KgcTripletDev* __restrict__ out,
                                                        unsigned long long* res_count, long long res_cap, int r_off,
                                                        long long Nt, long long t_off, long long h_off,
                                                        const int* __restrict__ hmap) {
    long long nc = (long long)*cand_count;
    if (nc > cand_cap) nc = cand_cap;
    const int lane = threadIdx.x & 31, wib = (threadIdx.x >> 5) & 7;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long rows_per_rel = (long long)QT * bq;
    const float thf = (float)theta;  // theta is a float value
    const float cf = 5.9604644775390625e-08f * 1.0009765625f;  // u (1 + 2^-10)
    const float dterm = NORM == 2 ? (float)d * 0.25f + 8.0f : (float)d * 0.5f + 8.0f;
    // dynamic shared memory (91 KB per block): per warp the result stage, two tail-row buffers
    // and the 32 row indices
    extern __shared__ __align__(16) uint8_t vsm[];
    KgcTripletDev* st = reinterpret_cast<KgcTripletDev*>(vsm) + wib * (VB * 32);
    float* tbw = reinterpret_cast<float*>(vsm + 8 * VB * 32 * sizeof(KgcTripletDev)) + wib * (2 * 32 * VST);
    int* trw = reinterpret_cast<int*>(vsm + 8 * VB * 32 * sizeof(KgcTripletDev) + 8 * 2 * 32 * VST * 4) + wib * 32;
    const int nck = (d + VKC - 1) / VKC;
    for (long long base0 = warp * 32 * VB; base0 < nc; base0 += nwarps * 32 * VB) {
        int cnt = 0;
        for (int rr = 0; rr < VB; ++rr) {
            const long long base = base0 + rr * 32;
            if (base >= nc) break;
            // ---- stage 1: this lane's candidate
            const long long idx = base + lane;
            bool valid = idx < nc;
            int h = 0, r = 0, t = 0;  // h: row of E, t: row of Et
            if (valid) {
                const int2 cv = cand[idx];
                const long long rq = cv.x / rows_per_rel;
                const long long pos = cv.x - rq * rows_per_rel;
                valid = pos < N && cv.y < Nt;
                if (valid) {
                    r = (int)rq;
                    h = qperm ? qperm[rq * N + pos] : (int)pos;  // null: natural order
                    t = tperm ? tperm[cv.y] : cv.y;
                }
            }
            const float* eh = E + (long long)h * d;
            const float* er = Rel + (long long)r * d;
            const float* et = Et + (long long)t * d;
            // ---- stage 2: FP32 distance + error bound, FP64 only where it cannot decide
            float dist = 0.f;
            bool keep = false;
            bool exact = !VEC4;
            if (VEC4) {
                __syncwarp();
                trw[lane] = t;  // invalid lanes stage row 0 (in range, unused)
                __syncwarp();
                // chunk c of the 32 tail rows into tbuf[wib][c & 1]: piece p = 32 j + lane is row
                // p / 8 (= 4 j + lane / 8), 16-byte piece lane % 8 of the chunk
                auto issue = [&](int c) {
                    const int klen = d - c * VKC < VKC ? d - c * VKC : VKC;
                    const int pq = lane & 7;
                    float* dst = tbw + (c & 1) * 32 * VST;
                    if (4 * pq < klen) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int row = 4 * j + (lane >> 3);
                            const float* src = Et + (long long)trw[row] * d + c * VKC + 4 * pq;
                            cp_async16(smem_u32(dst + row * VST + 4 * pq), src);
                        }
                    }
                    cp_async_commit();
                };
                float2 sy = make_float2(0.f, 0.f), sa = make_float2(0.f, 0.f);
                const float2 m1 = make_float2(-1.f, -1.f);
                issue(0);
                for (int c = 0; c < nck; ++c) {
                    if (c + 1 < nck) {
                        issue(c + 1);
                        cp_async_wait_n(1);
                    } else {
                        cp_async_wait_n(0);
                    }
                    __syncwarp();  // every lane's pieces of chunk c have landed
                    const int klen = d - c * VKC < VKC ? d - c * VKC : VKC;
                    const float* tz = tbw + (c & 1) * 32 * VST + lane * VST;
                    for (int q = 0; q < klen; q += 4) {
                        const int k = c * VKC + q;
                        const float4 x = __ldg(reinterpret_cast<const float4*>(eh + k));
                        const float4 y = __ldg(reinterpret_cast<const float4*>(er + k));
                        const float4 z = *reinterpret_cast<const float4*>(tz + q);
                        const float2 a0 = __ffma2_rn(make_float2(z.x, z.y), m1, make_float2(x.x, x.y));  // fl(h - t)
                        const float2 a1 = __ffma2_rn(make_float2(z.z, z.w), m1, make_float2(x.z, x.w));
                        const float2 y0 = __fadd2_rn(a0, make_float2(y.x, y.y));                        // fl(a + r)
                        const float2 y1 = __fadd2_rn(a1, make_float2(y.z, y.w));
                        if (NORM == 2) {
                            sy = __ffma2_rn(y0, y0, sy);
                            sy = __ffma2_rn(y1, y1, sy);
                            sa = __ffma2_rn(a0, a0, sa);
                            sa = __ffma2_rn(a1, a1, sa);
                        } else {
                            sy.x += fabsf(y0.x) + fabsf(y1.x);
                            sy.y += fabsf(y0.y) + fabsf(y1.y);
                            sa.x += fabsf(a0.x) + fabsf(a1.x);
                            sa.y += fabsf(a0.y) + fabsf(a1.y);
                        }
                    }
                    __syncwarp();  // buffer c & 1 is refilled by chunk c + 2
                }
                const float s2 = sy.x + sy.y;
                const float an = NORM == 2 ? sqrtf(sa.x + sa.y) : sa.x + sa.y;
                const float d32 = NORM == 2 ? sqrtf(s2) : s2;
                const float B = cf * (dterm * d32 + 2.0f * an);
                if (d32 - B > thf) {
                    keep = false;                                   // certainly farther than theta
                } else if (d32 + B <= thf && B <= 8e-6f * fmaxf(d32, thf)) {
                    keep = true;                                    // certainly within, distance accurate
                    dist = d32;
                } else {
                    exact = true;                                   // undecided: FP64
                }
            }
            if (valid && exact) {
                const double dd = dist_f64<NORM>(eh, er, et, d);
                keep = dd <= theta;
                dist = (float)dd;
            }
            // ---- stage 3: keep iff dist <= theta (inclusive); stage in candidate order
            keep = keep && valid;
            const uint32_t m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                KgcTripletDev o;
                o.h = hmap ? hmap[h] : (int)(h + h_off);  // global ids: head map / block / partition offsets,
                o.r = r + r_off;         // relation index in the caller's Rel
                o.t = (int)(t + t_off);
                o.dist = dist;
                st[cnt + __popc(m & lanemask_lt())] = o;
            }
            cnt += __popc(m);
        }
        __syncwarp();
        unsigned long long slot = 0;
        if (lane == 0 && cnt) slot = atomicAdd(res_count, (unsigned long long)cnt);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        for (int i = lane; i < cnt; i += 32)
            if (slot + i < (unsigned long long)res_cap) out[slot + i] = st[i];
        __syncwarp();
    }
}

// Pull a buffer into L2 (prefetch.global.L2::evict_last, one per 128-byte line).  Before
// the re-check of a large join: the tile kernel has just streamed the staged tails through
// L2, evicting E, and the re-check then gathers two rows of E per candidate (c4: 98.5 MB
// of E, ~6e6 candidates x 2 x 800 B) -- from DRAM at random unless E is L2-resident again.
// Reading E once in order costs ~15 us of HBM time.
__global__ void l2_prefetch_kernel(const char* __restrict__ p, size_t bytes) {
    for (size_t o = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 128; o < bytes;
         o += (size_t)gridDim.x * blockDim.x * 128)
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p + o));
}

void launch_l2_prefetch(const void* p, size_t bytes, int num_sms, cudaStream_t s) {
    if (!p || bytes == 0) return;
    l2_prefetch_kernel<<<num_sms * 4, 256, 0, s>>>(reinterpret_cast<const char*>(p), bytes);
}

void launch_verify(const int2* cand, const unsigned long long* cand_count, long long cand_cap, const int* qperm,
                   const int* tperm, const float* E, const float* Rel, const float* Et, long long N, int QT, int bq,
                   int d, int norm, float theta, KgcTripletDev* out, unsigned long long* res_count, long long res_cap,
                   int num_sms, cudaStream_t s, int r_off, long long Nt, long long t_off, long long h_off,
                   const int* hmap) {
    const bool vec4 = (d % 4 == 0) && ((reinterpret_cast<uintptr_t>(E) | reinterpret_cast<uintptr_t>(Rel) |
                                        reinterpret_cast<uintptr_t>(Et)) % 16 == 0);
    auto kern = norm == 1 ? (vec4 ? verify_kernel<1, true> : verify_kernel<1, false>)
                          : (vec4 ? verify_kernel<2, true> : verify_kernel<2, false>);
    const int smem = 8 * VB * 32 * (int)sizeof(KgcTripletDev) + 8 * 2 * 32 * VST * 4 + 8 * 32 * 4;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<num_sms * 4, 256, smem, s>>>(cand, cand_count, cand_cap, qperm, tperm, E, Rel, Et, N, QT, bq, d,
                                        (double)theta, out, res_count, res_cap, r_off, Nt < 0 ? N : Nt, t_off, h_off,
                                        hmap);
}

}  // namespace kgc
