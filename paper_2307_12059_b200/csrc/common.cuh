// common.cuh -- device helpers for the sm_100a kernels of libkgc.
//
// Thin inline-PTX wrappers: mbarrier, 1-D bulk TMA copies (cp.async.bulk,
// SASS UBLKCP), and the tcgen05 instructions (alloc / mma kind::tf32 /
// commit / ld) used by the tensor-core filter.  No method arithmetic here.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kgc_internal.h"

namespace kgc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// One lane of a converged warp (PTX elect.sync).
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// Blocks until the phase with parity `parity` of the barrier has completed.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
        "r"(parity)
        : "memory");
}

// ------------------------------------------------------ clusters (pairs)
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// Arrive on the barrier at the same shared-memory offset in CTA `rank` of the
// cluster (default .release.cta semantics, as CUTLASS's ClusterBarrier: the
// operands these barriers guard are read by the tensor cores through the
// async proxy, published by fence.proxy.async or by TMA completion).
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\t"
        "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
        "r"(rank)
        : "memory");
}
// mbar_wait with cluster-scope acquire (for phases completed by remote arrivals).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n\t}" ::"r"(addr),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ------------------------------------------------------- bulk TMA (1-D)
// Global -> shared copy of `bytes` (multiple of 16, both addresses 16-B
// aligned) completing as transaction bytes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// L2 eviction-priority policies (createpolicy) for the cache-hinted copies below.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// bulk_g2s with an L2 cache hint (e.g. keep the staged tail tiles, re-read per query tile)
__device__ __forceinline__ void bulk_g2s_hint(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(smem_dst)), "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// ------------------------------------------------ cp.async (16-byte pieces)
// Global -> shared 16-byte copy (LDGSTS, L1 bypass); completion is tracked by
// cp_async_mbar_arrive_noinc: the barrier receives one arrival (not counted in
// advance by the instruction) once all of this thread's prior cp.async are done.
__device__ __forceinline__ void cp_async16(uint32_t smem_dst, const void* gmem_src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_dst), "l"(gmem_src) : "memory");
}
// cp_async16 with an L2 cache hint (e.g. evict-first for rows read once per item)
__device__ __forceinline__ void cp_async16_hint(uint32_t smem_dst, const void* gmem_src, uint64_t policy) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_dst), "l"(gmem_src),
                 "l"(policy) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// wait until at most n of this thread's committed cp.async groups are pending (n <= 7)
__device__ __forceinline__ void cp_async_wait_n(int n) {
    switch (n) {
        case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
        case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
        case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
        case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
        case 5: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
        case 6: asm volatile("cp.async.wait_group 6;" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 7;" ::: "memory"); break;
    }
}

// ------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_slot, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor, K-major, no swizzle ("interleaved"):
// core matrices of 8 rows x 16 B stored as 128 contiguous bytes; LBO = byte
// distance between the two core matrices adjacent in K, SBO = byte distance
// between core matrices adjacent in M/N; bits 46-47 = 1 (sm_100 version).
__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
}

// K-major, 128-byte swizzle: rows of 128 bytes (32 fp32 of K) in 8-row atoms of
// 1024 bytes, 16-byte chunks XOR-permuted by row % 8 (the layout TMA writes with
// CU_TENSOR_MAP_SWIZZLE_128B); SBO = 1024 between 8-row groups, LBO unused (1),
// layout type 2 (SWIZZLE_128B) in bits 61-63.  The atom must be 1024-B aligned;
// a K step of 8 fp32 advances the start address by 32 bytes.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// TMA row gather (sm_100): rows r0..r3 of a 2-D tensor map (box = {cols, 1}),
// columns [c0, c0 + cols), written as 4 consecutive box rows at smem_dst with the
// map's swizzle; completes as transaction bytes on `bar`.
__device__ __forceinline__ void tma_gather4(uint32_t smem_dst, const void* tmap, int c0, int r0, int r1, int r2,
                                            int r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_dst),
        "l"(tmap), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}

// Instruction descriptor for kind::tf32: D = F32, A = B = TF32, both K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4)                          // D format F32
           | (2u << 7)                        // A format TF32
           | (2u << 10)                       // B format TF32
           | ((uint32_t)(N >> 3) << 17)       // N / 8
           | ((uint32_t)(M >> 4) << 24);      // M / 16
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// Arrive on `bar` when every previously issued tcgen05 op of this thread is done.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// CTA-pair forms (cta_group::2): TMEM allocation by the same warp of both
// CTAs; the MMA is issued by the even CTA and reads A / B rows from both
// CTAs' shared memory at the same offsets (M = 256: 128 rows per CTA; the
// B tile of N rows: N / 2 per CTA); each CTA's TMEM receives its 128 rows.
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_slot, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// Arrive on the barrier at this offset in every CTA of `mask` when the
// pair's previously issued tcgen05 ops are done.
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: lane l gets row (lane base + l).
// Issue a 32-column TMEM load without waiting (pair with tmem_wait_ld()).
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Warp-aggregated append: every lane with `pred` gets a unique slot in a
// global list whose length counter is `*counter` (one atomic per warp).
__device__ __forceinline__ unsigned long long warp_append(bool pred, unsigned long long* counter) {
    uint32_t m = __ballot_sync(0xffffffffu, pred);
    unsigned long long base = 0;
    if (m) {
        int leader = __ffs(m) - 1;
        if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(counter, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, leader);
    }
    return base + __popc(m & lanemask_lt());
}

// Warp-aggregated reservation of n (per lane) consecutive slots: returns the
// first slot of this lane's block.  One atomic per warp.
__device__ __forceinline__ unsigned long long warp_reserve(uint32_t n, unsigned long long* counter) {
    const int lane = threadIdx.x & 31;
    uint32_t incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && total) base = atomicAdd(counter, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    return base + (incl - n);
}

// Contiguous, cost-balanced block of work items for CTA b of G: the first item
// whose exclusive tile prefix reaches floor(total * b / G) (b == G gives n).
__device__ __forceinline__ long long balanced_begin(const long long* __restrict__ cum, long long n, long long total,
                                                    long long b, long long G) {
    if (b >= G) return n;
    const long long target = total * b / G;
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long m = (lo + hi) >> 1;
        if (cum[m] >= target) hi = m; else lo = m + 1;
    }
    return lo;
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Tensor-core epilogue: max over 32 accumulator columns of (acc_j - th_j), th = ||t||^2 / 2 --
// packed subtraction (FADD2) and 3-input max (FMNMX3), both sm_100 forms: half the instructions
// of FFMA + FMNMX per column.  fl(acc - t/2) = fl(2 acc - t) / 2 exactly, so the test
// max >= c / 2 is the same decision as max(2 acc - t) >= c.
__device__ __forceinline__ void sub2_f32(uint32_t a0, uint32_t a1, float t0, float t1, float& d0, float& d1) {
    unsigned long long A, T, D;
    asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "r"(a0), "r"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(T) : "f"(t0), "f"(t1));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(T));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(D));
}
__device__ __forceinline__ float max3_f32(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float epi_max32(const uint32_t (&r)[32], const float4* __restrict__ th) {
    float m[4] = {-3.0e38f, -3.0e38f, -3.0e38f, -3.0e38f};
#pragma unroll
    for (int u4 = 0; u4 < 8; ++u4) {
        const float4 tt = __ldg(th + u4);
        float a0, a1, a2, a3;
        sub2_f32(r[4 * u4 + 0], r[4 * u4 + 1], tt.x, tt.y, a0, a1);
        sub2_f32(r[4 * u4 + 2], r[4 * u4 + 3], tt.z, tt.w, a2, a3);
        const int c = (u4 & 1) * 2;
        m[c] = max3_f32(m[c], a0, a1);
        m[c + 1] = max3_f32(m[c + 1], a2, a3);
    }
    return fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
}
// the same with the thresholds in shared memory (plain loads)
__device__ __forceinline__ float epi_max32_s(const uint32_t (&r)[32], const float4* th) {
    float m[4] = {-3.0e38f, -3.0e38f, -3.0e38f, -3.0e38f};
#pragma unroll
    for (int u4 = 0; u4 < 8; ++u4) {
        const float4 tt = th[u4];
        float a0, a1, a2, a3;
        sub2_f32(r[4 * u4 + 0], r[4 * u4 + 1], tt.x, tt.y, a0, a1);
        sub2_f32(r[4 * u4 + 2], r[4 * u4 + 3], tt.z, tt.w, a2, a3);
        const int c = (u4 & 1) * 2;
        m[c] = max3_f32(m[c], a0, a1);
        m[c + 1] = max3_f32(m[c + 1], a2, a3);
    }
    return fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
}
__device__ __forceinline__ uint32_t epi_hits32_s(const uint32_t (&r)[32], const float4* th, float ch) {
    uint32_t hit = 0;
#pragma unroll
    for (int u4 = 0; u4 < 8; ++u4) {
        const float4 tt = th[u4];
        hit |= (uint32_t)(__fsub_rn(__uint_as_float(r[4 * u4 + 0]), tt.x) >= ch) << (4 * u4 + 0);
        hit |= (uint32_t)(__fsub_rn(__uint_as_float(r[4 * u4 + 1]), tt.y) >= ch) << (4 * u4 + 1);
        hit |= (uint32_t)(__fsub_rn(__uint_as_float(r[4 * u4 + 2]), tt.z) >= ch) << (4 * u4 + 2);
        hit |= (uint32_t)(__fsub_rn(__uint_as_float(r[4 * u4 + 3]), tt.w) >= ch) << (4 * u4 + 3);
    }
    return hit;
}
// bit j set iff acc_j - th_j >= ch (the rare path after epi_max32 found a candidate)
__device__ __forceinline__ uint32_t epi_hits32(const uint32_t (&r)[32], const float4* __restrict__ th, float ch) {
    uint32_t hit = 0;
#pragma unroll
    for (int u4 = 0; u4 < 8; ++u4) {
        const float4 tt = __ldg(th + u4);
        hit |= (uint32_t)(__fsub_rn(__uint_as_float(r[4 * u4 + 0]), tt.x) >= ch) << (4 * u4 + 0);
        hit |= (uint32_t)(__fsub_rn(__uint_as_float(r[4 * u4 + 1]), tt.y) >= ch) << (4 * u4 + 1);
        hit |= (uint32_t)(__fsub_rn(__uint_as_float(r[4 * u4 + 2]), tt.z) >= ch) << (4 * u4 + 2);
        hit |= (uint32_t)(__fsub_rn(__uint_as_float(r[4 * u4 + 3]), tt.w) >= ch) << (4 * u4 + 3);
    }
    return hit;
}

// float -> float rounded towards +inf from a double
__device__ __forceinline__ float f2up(double x) { return __double2float_ru(x); }

}  // namespace kgc
