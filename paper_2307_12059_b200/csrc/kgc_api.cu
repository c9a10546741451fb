// kgc_api.cu -- host runtime and C ABI of libkgc (include/kgc.h).
//
// One kgc_join runs the whole hot path on the context's stream:
//   a1 stage inputs (H2D when the caller passes host pointers)
//   a2 K1 pivot distances (tails once; queries per relation)
//   a3 K2 sorts
//   a4 K3 tile ranges (Lemma 1 + 2), shard split, work items   -> sync #1
//   stage operand tiles
//   a5/a6 K4 (L2, tcgen05) or K5 (L1 / L2 SIMT) over the work items
//   a7/a8 K6+K7 FP64 re-check and compaction                    -> sync #2
// Device buffers grow monotonically and are reused across joins.
#include <cfloat>
#include <chrono>
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled (driver entry point through cudart)

#include "../../include/kgc.h"
#include "kgc_internal.h"

using namespace kgc;

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
};

enum Phase { EV_START, EV_H2D, EV_KEYS, EV_SORT, EV_RANGES, EV_STAGE, EV_TILES, EV_VERIFY, EV_COUNT };

}  // namespace

// Every device buffer of a context, in one list: the context declares them and
// kgc_destroy frees them from the same list, so no buffer can be left out.
#define KGC_DEVBUFS(X) X(E) X(Rel) X(pivot) X(kt) X(kq) X(mm_t) X(mm_q) X(sk0) X(sv0) X(sk1) X(sv1) X(counts) \
    X(scan_tmp) X(qperm) X(qskey) X(tperm) X(tskey) X(tmin) X(tmax) X(cmax) X(cmin) X(ranges) X(cost) X(cum) \
    X(nitem) X(item_off) X(items) X(item_tiles) X(item_cum) X(Qp) X(qs) X(Tp) X(T2) X(tstile) X(cand) X(res) X(ctr) \
    X(est_hist) X(est_cost) X(mpP) X(mpkt) X(mpkq) X(mpmm_t) X(mpmm_q) X(mpc0) X(mpc1) X(tbmin) X(tbmax) X(qbmin) \
    X(qbmax) X(tile_list) X(tk_sample) X(tk_sel) X(tk_cnt) X(Ts) X(tks) X(gblk) X(granges) X(glist) X(tsc) X(gT2) \
    X(gtst) X(tmapbuf) X(fz) X(frt) X(frn) X(fzero) X(se_w) X(se_a64) X(se_b64) X(se_af) X(se_bf) X(se_zero) \
    X(acc) X(Eb) X(mpbits) X(se_max) X(mpqn) X(mpA) X(mphx) X(mpB) X(mpC) X(mpk4) X(mpmm4) X(mpHP) \
    X(sp_P) X(sp_keys) X(sp_mm) X(sp_c0) X(sp_v0) X(sp_c1) X(sp_v1) X(sp_hidx) X(sp_Eh)

struct kgc_ctx {
    kgc_options opt{};
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    std::string err;
#define KGC_DECLARE_BUF(n) DevBuf n;
    KGC_DEVBUFS(KGC_DECLARE_BUF)
#undef KGC_DECLARE_BUF
    long long cand_cap = 0, res_cap = 0;
    long long n_results = -1;
    kgc_stats_t st{};
    cudaEvent_t ev[EV_COUNT] = {};
    cudaEvent_t ev_split[2] = {};
    cudaStream_t aux = nullptr;     // fork / join stream for pivot-independent work (the h.r GEMM)
    cudaEvent_t ev_fork[2] = {};
    cudaEvent_t ev_sp[2] = {};    // split 3: the head order on the aux stream beside the pivot choice
    bool pivots_ready = false;    // split 3: mpP already holds this join's pivots (launched on stream)
    int launches = 0;
    // geometry of the last join (for kgc_inspect)
    long long N = 0, R = 0;
    int QT = 0, TT = 0, BN = 0;
    int K = 1;                  // pivots used by the last join
    int d = 0;                  // embedding dimension of the last join
    bool l2f = false;           // the last join's K-pivot L2 keys came from the factorisation (not materialised)
    long long list_len = 0;     // multi-pivot tile-list length of this shard
    long long glist_len = 0;    // gathered-tail list length of this shard (entries)
    CUtensorMap tmap_host;      // tensor map over the sorted tails (gathered tensor-core engine)
    std::vector<int4> fitems;   // relation-factored engine: work items built on the host
    bool have_join = false;
    unsigned int* mp_bits = nullptr;  // this join's K-pivot survival masks (or nullptr)
};

static std::string g_create_err;

static void set_err(kgc_ctx* c, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            set_err(ctx, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
            return e_ == cudaErrorMemoryAllocation ? KGC_ENOMEM : KGC_ECUDA;                       \
        }                                                                                          \
    } while (0)

#define LAUNCHED(n)                                                                                \
    do {                                                                                           \
        ctx->launches += (n);                                                                      \
        cudaError_t e_ = cudaGetLastError();                                                       \
        if (e_ != cudaSuccess) {                                                                   \
            set_err(ctx, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return KGC_ECUDA;                                                                      \
        }                                                                                          \
    } while (0)

static cudaError_t ensure(DevBuf& b, size_t bytes) {
    if (bytes <= b.n && b.p) return cudaSuccess;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.n = 0;
    size_t nb = bytes + bytes / 8 + 256;
    cudaError_t e = cudaMalloc(&b.p, nb);
    if (e == cudaSuccess) b.n = nb;
    return e;
}

template <typename T>
static T* P(DevBuf& b) {
    return reinterpret_cast<T*>(b.p);
}

// Engine choice and the plan's query-tile height (tensor cores / FP16x2: 128, FP32 SIMT: 64).
static bool use_tc(const kgc_ctx* ctx, int norm, int d) {
    return norm == 2 && ctx->opt.l2_engine != 2 && ((d + 7) / 8) * 8 <= TC_MAX_KPAD;
}
// Tensor cores on CTA pairs (cta_group::2, 256-row query tiles): l2_engine 3,
// or automatically once the staged tails outgrow a fraction of L2 (48 MiB),
// where the 1-CTA kernel waits on tail bytes (measured: c4 +9%, c5 +11%
// tile-kernel throughput; on c2 the coarser query tiles prune less and the
// pair kernel is 8% slower).
static bool use_tc2(const kgc_ctx* ctx, int norm, int d, long long N) {
    if (!use_tc(ctx, norm, d)) return false;
    if (ctx->opt.l2_engine == 3 || ctx->opt.l2_engine == 6) return true;  // 6: gathered when K > 1
    if (ctx->opt.l2_engine != 0) return false;
    const char* e = kgc_knob("KGC_TC2");  // experiment knob: force the automatic choice
    if (e) return atoi(e) != 0;
    return (double)N * (double)(((d + 7) / 8) * 8) * 4.0 > 48.0 * 1048576.0;
}
// FP32 SIMT tile edge (experiment knob KGC_SIMT_T = 32 | 64)
static int simt_t() {
    const char* e = kgc_knob("KGC_SIMT_T");
    return (e && atoi(e) == 32) ? 32 : SIMT_T;
}
// Gathered-tail SIMT engine (l1_engine 3; auto for L1 with multi-pivot pruning):
// element-level tail pruning inside surviving tiles (pivots.cu, tiles_simt.cu).
// Tensor-core engine on gathered tail blocks (l2_engine 4): the same per-tail test,
// blocks of 256 gathered rows (tiles_tc.cu, GATHER); needs K pivots and the 1-CTA geometry.
// l2_engine 6: the same on CTA pairs (256-row query tiles, each CTA gathers half of every
// block with cp.async pieces; tiles_tc2.cu, GATHER).
static bool use_gather_tc(const kgc_ctx* ctx) {
    const char* e = kgc_knob("KGC_GATHER_TC");  // experiment knob
    if (e) return atoi(e) != 0;
    return ctx->opt.l2_engine == 4 || ctx->opt.l2_engine == 6;
}
// 2-D tensor map over the sorted row-major tails Ts[N + 1][Kpad] (fp32): box = 32 columns x 1
// row, 128-byte swizzle -- the operand of the TMA row gathers (tiles_tc.cu, GATHER).
static int make_tails_tmap(CUtensorMap* m, const float* Ts, long long rows, int Kpad) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return -1;
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t gdim[2] = {(cuuint64_t)Kpad, (cuuint64_t)rows};
    const cuuint64_t gstride[1] = {(cuuint64_t)Kpad * 4};
    const cuuint32_t box[2] = {32, 1};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(Ts), gdim, gstride, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -1;
}

// Device memory the gathered tensor-core lists may take (glist + ||t||^2/2 per entry)
// before the join falls back to contiguous tiles.
constexpr size_t GATHER_TC_BUDGET = 8ull << 30;
static bool use_gather(const kgc_ctx* ctx, int norm) {
    const char* e = kgc_knob("KGC_GATHER");  // experiment knob: 0 = off, 1 = on for both norms
    if (e) return atoi(e) != 0;
    if (ctx->opt.l1_engine == 3) return true;
    return norm == 1 && ctx->opt.l1_engine == 0;
}
static int plan_bq(const kgc_ctx* ctx, int norm, int d, long long N) {
    if (use_tc2(ctx, norm, d, N)) return 2 * BM;
    if (use_tc(ctx, norm, d)) return BM;
    return (norm == 1 && ctx->opt.l1_engine == 1) ? BN_HALF : simt_t();
}

// Relative margin covering the FP32 pivot keys.
static float mp_relm(int d) { return (float)(d + 8) * 1.1920928955078125e-07f; }

static float __uint_as_float_host(unsigned int u) {
    float f;
    memcpy(&f, &u, 4);
    return f;
}

static bool is_device_ptr(const void* p, int device) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) && (a.device == device);
}

extern "C" {

int kgc_abi_version(void) { return KGC_ABI_VERSION; }

void kgc_default_options(kgc_options* o) {
    if (!o) return;
    memset(o, 0, sizeof *o);
    o->device = -1;
    o->rank = 0;
    o->world = 1;
    o->prune = 1;
    o->pivot = 0;
    o->l2_engine = 0;
    o->chunk_tiles = 0;
    o->pivots = 1;
    o->l1_engine = 0;
    o->split = 0;
    o->tail_shard = 0;
    o->relation_batch = 0;
    o->result_capacity = 0;
    o->stream = nullptr;
}

int kgc_create(kgc_ctx** out, const kgc_options* opt) {
    if (!out) return KGC_EINVAL;
    *out = nullptr;
    kgc_options o;
    if (opt) o = *opt; else kgc_default_options(&o);
    if (o.world < 1 || o.rank < 0 || o.rank >= o.world || (o.pivot != 0 && o.pivot != 1) || o.l2_engine < 0 ||
        o.l2_engine > 6 || o.chunk_tiles < 0 || o.result_capacity < 0 || o.pivots < 0 || o.pivots > MP_MAX || !mp_pivots_ok(o.pivots) || o.l1_engine < 0 || o.l1_engine > 3 || o.split < 0 || o.split > 3 || o.tail_shard < 0 || o.tail_shard > 1 || o.relation_batch < 0) {
        g_create_err = "kgc_create: invalid options";
        return KGC_EINVAL;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        g_create_err = "kgc_create: no CUDA device";
        return KGC_ENODEV;
    }
    int dev = o.device;
    if (dev < 0) cudaGetDevice(&dev);
    if (dev >= ndev) {
        g_create_err = "kgc_create: device ordinal out of range";
        return KGC_EINVAL;
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.major != 10 || prop.minor != 0) {
        cudaGetLastError();
        g_create_err = "kgc_create: libkgc is built for sm_100a (B200); device " + std::to_string(dev) + " is sm_" +
                       std::to_string(prop.major) + std::to_string(prop.minor);
        return KGC_ENODEV;
    }
    kgc_ctx* ctx = new kgc_ctx();
    ctx->opt = o;
    ctx->device = dev;
    ctx->num_sms = prop.multiProcessorCount;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
    if (o.stream) {
        ctx->stream = reinterpret_cast<cudaStream_t>(o.stream);
    } else {
        if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
            g_create_err = "kgc_create: cudaStreamCreate failed";
            delete ctx;
            return KGC_ECUDA;
        }
        ctx->stream = ctx->own_stream;
    }
    for (auto& e : ctx->ev) cudaEventCreate(&e);
    for (auto& e : ctx->ev_split) cudaEventCreate(&e);
    cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking);
    for (auto& e : ctx->ev_fork) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    for (auto& e : ctx->ev_sp) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaSetDevice(prev);
    *out = ctx;
    return KGC_OK;
}

void kgc_destroy(kgc_ctx* ctx) {
    if (!ctx) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
#define KGC_FREE_BUF(n) if (ctx->n.p) cudaFree(ctx->n.p);
    KGC_DEVBUFS(KGC_FREE_BUF)
#undef KGC_FREE_BUF
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto e : ctx->ev_split)
        if (e) cudaEventDestroy(e);
    for (auto e : ctx->ev_sp)
        if (e) cudaEventDestroy(e);
    for (auto e : ctx->ev_fork)
        if (e) cudaEventDestroy(e);
    if (ctx->aux) {
        cudaStreamSynchronize(ctx->aux);
        cudaStreamDestroy(ctx->aux);
    }
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    cudaSetDevice(prev);
    delete ctx;
}

const char* kgc_last_error(const kgc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

int kgc_set_stream(kgc_ctx* ctx, void* stream) {
    if (!ctx) return KGC_EINVAL;
    ctx->stream = stream ? reinterpret_cast<cudaStream_t>(stream) : ctx->own_stream;
    if (!ctx->stream) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(ctx->device);
        cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
        cudaSetDevice(prev);
        ctx->stream = ctx->own_stream;
    }
    return KGC_OK;
}

}  // extern "C"
// split = 3: the curve order is cut into nch = W m equal chunks, m = max(2, round(N / (W chunk)))
static int64_t sp_nchunks(int64_t N, int64_t world, int64_t chunk) {
    int64_t m = (int64_t)std::llround((double)N / ((double)world * (double)chunk));
    if (m < 2) m = 2;
    return std::min<int64_t>(N, world * m);
}
extern "C" {

int64_t kgc_spatial_chunks(int64_t N, int32_t world, int32_t rank, int64_t chunk, int64_t* begin, int64_t* len,
                           int64_t cap) {
    if (N < 0 || world < 1 || rank < 0 || rank >= world || chunk < 1 || cap < 0 || (cap > 0 && (!begin || !len)))
        return KGC_EINVAL;
    if (N == 0) return 0;
    const int64_t nch = sp_nchunks(N, world, chunk);
    int64_t owned = 0;
    for (int64_t c = rank; c < nch; c += world, ++owned) {
        if (owned < cap) {
            begin[owned] = c * N / nch;
            len[owned] = (c + 1) * N / nch - c * N / nch;
        }
    }
    return owned;
}

int64_t kgc_shard_range(const int64_t* cum, int64_t n, int64_t total, int32_t rank, int32_t world, int64_t* begin,
                        int64_t* end) {
    if (!cum || !begin || !end || n < 0 || total < 0 || world < 1 || rank < 0 || rank >= world) return KGC_EINVAL;
    int64_t b = n, e = 0, cost = 0;
    for (int64_t q = 0; q < n; ++q) {
        int64_t owner = 0;
        if (total > 0) {
            int64_t o = (int64_t)world * cum[q] / total;
            owner = o < world - 1 ? o : world - 1;
        }
        if (owner == rank) {
            if (q < b) b = q;
            e = q + 1;
            int64_t next = q + 1 < n ? cum[q + 1] : total;
            cost += next - cum[q];
        }
    }
    if (b > e) b = e = 0;
    *begin = b;
    *end = e;
    return cost;
}

}  // extern "C"

// ------------------------------------------------------------------ join
// R, Rel_in: the relations this context preprocesses (rank-local split: a
// sub-range starting at global relation r_off); [force_lo, force_hi): the
// query tiles (in local numbering) this rank joins, or -1 for the
// cost-balanced rule over all of them.
// Optional parts of a join beyond TransE (SE, se.cu): a separate tail matrix, a wider
// filter threshold (operands rounded on both sides), and FP64 connectors for the re-check.
struct JoinExtra {
    const float* Et = nullptr;    // tails (default: E, or rows [t_off, t_off + Nt) of the device copy of E)
    long long Nt = -1;            // tail rows (default: N); tail partitions (kgc_options.tail_shard)
    long long t_off = 0;          // first tail row of the partition (added to emitted t)
    long long h_off = 0;          // first head row of a head block (added to emitted h; kgc_join_block)
    const int* hmap = nullptr;    // device head ids: emitted h = hmap[local head row] (split = 3)
    float filt_eps = -1.f;        // threshold of every filter and pruning test (default: eps)
    const double* A64 = nullptr;  // exact connectors for verify_se (default: TransE verify)
    const double* B64 = nullptr;
};

static int join_impl(kgc_ctx* ctx, const float* E_in, const float* Rel_in, long long N, long long R, int d, int norm,
                     float eps, int r_off, long long force_lo, long long force_hi, long long R_global,
                     const JoinExtra& ex = JoinExtra()) {
    cudaStream_t s = ctx->stream;
    ctx->launches = 0;
    kgc_stats_t& st = ctx->st;
    memset(&st, 0, sizeof st);
    st.N = N;
    st.R = R_global;
    st.d = d;
    st.norm = norm;
    st.eps = eps;
    st.rank = ctx->opt.rank;
    st.world = ctx->opt.world;
    st.triplets = (double)N * (double)N * (double)R_global;

    const bool tc = use_tc(ctx, norm, d);
    const int K_plan = (ctx->opt.pivots >= 2 && ctx->opt.prune && d <= MP_MAX_DIM) ? ctx->opt.pivots : 1;
    const bool gtc_req = tc && K_plan > 1 && use_gather_tc(ctx);  // gathered tensor-core blocks requested
    const long long NT = ex.Nt >= 0 ? ex.Nt : N;  // tail rows (a tail partition, or all N)
    const bool tc2 = !gtc_req && use_tc2(ctx, norm, d, NT);
    if (norm == 2 && (ctx->opt.l2_engine == 1 || ctx->opt.l2_engine == 3 || ctx->opt.l2_engine >= 4) && !tc) {
        set_err(ctx, "l2_engine=%d (tcgen05) supports d <= %d", ctx->opt.l2_engine, TC_MAX_KPAD);
        return KGC_EINVAL;
    }
    const int Kpad = ((d + 7) / 8) * 8;
    // tile geometry of the plan: tensor cores 128 x 256; FP16x2 L1 128 x 128; FP32 SIMT 64 x 64
    const bool half_req = norm == 1 && ctx->opt.l1_engine == 1;
    // query-tile rows: the engine's (the pair engine's choice follows the tail rows, so a tail
    // partition may use the 1-CTA engine where the whole tail set would not)
    const bool gtc_pair = gtc_req && ctx->opt.l2_engine == 6;       // gathered blocks on CTA pairs
    const int bq = gtc_req ? (gtc_pair ? 2 * BM : BM) : (tc2 ? 2 * BM : (tc ? BM : (half_req ? BN_HALF : simt_t())));
    // tail tile rows: the contiguous pair engine uses 128-row tail tiles (UMMA N = 128; finer tail
    // tiles prune better at the same B bytes per MAC: c4 5.70% -> 4.76% of pairs, c3 9.18 -> 6.30%)
    // (the same pairing in the 1-CTA engine needs 16 bulk copies of 2 KB per chunk to interleave two
    // 128-row tiles into one N = 256 operand and measured 1.55x slower on c3: it keeps 256-row tiles)
    const int BN = tc ? ((tc2 && !gtc_req) ? BN_PAIR : BN_TC) : (half_req ? BN_HALF : simt_t());
    const int QT = (int)((N + bq - 1) / bq);
    const int TT = (int)((NT + BN - 1) / BN);
    const long long nq = R * (long long)QT;
    int chunk = ctx->opt.chunk_tiles > 0 ? ctx->opt.chunk_tiles : (tc ? 16 : 8);
    if (tc && ctx->opt.chunk_tiles == 0) {
        int as = 0, bs = 0, kc = 0;
        const int sb = (tc2 || gtc_pair) ? tc2_smem_bytes(Kpad, &as, &bs, &kc, BN) : tc_smem_bytes(Kpad, &as, &bs, &kc);
        if (sb > 0 && as == 1) chunk = 64;  // amortise A rebuilds
    }
    ctx->N = N;
    ctx->R = R;
    ctx->QT = QT;
    ctx->TT = TT;
    ctx->BN = BN;
    st.query_tile_rows = bq;
    st.tail_tile_rows = BN;
    st.query_tiles = QT;
    st.tail_tiles = TT;
    st.tile_pairs_total = nq * TT;

    CK(cudaEventRecord(ctx->ev[EV_START], s));
    // ---- a1: inputs on the device
    const float* E = E_in;
    const float* Rel = Rel_in;
    if (!is_device_ptr(E_in, ctx->device)) {
        CK(ensure(ctx->E, (size_t)N * d * 4));
        CK(cudaMemcpyAsync(ctx->E.p, E_in, (size_t)N * d * 4, cudaMemcpyDefault, s));
        E = P<float>(ctx->E);
        st.h2d_bytes += (int64_t)N * d * 4;
    }
    if (!is_device_ptr(Rel_in, ctx->device)) {
        CK(ensure(ctx->Rel, (size_t)R * d * 4));
        CK(cudaMemcpyAsync(ctx->Rel.p, Rel_in, (size_t)R * d * 4, cudaMemcpyDefault, s));
        Rel = P<float>(ctx->Rel);
        st.h2d_bytes += (int64_t)R * d * 4;
    }
    CK(cudaEventRecord(ctx->ev[EV_H2D], s));
    const float* Et = ex.Et ? ex.Et : E + ex.t_off * d;   // tails (device)
    const float feps = ex.filt_eps >= 0.f ? ex.filt_eps : eps;  // filters and pruning

    // ---- allocations for the preprocessing
    const size_t NR = (size_t)N * R;
    const size_t nsort = std::max(NR, (size_t)NT);
    CK(ensure(ctx->ctr, sizeof(DevCounters)));
    CK(ensure(ctx->kt, (size_t)NT * 4));
    CK(ensure(ctx->kq, NR * 4));
    CK(ensure(ctx->mm_t, 2 * 4));
    CK(ensure(ctx->mm_q, (size_t)R * 2 * 4));
    CK(ensure(ctx->sk0, nsort * 4));
    CK(ensure(ctx->sv0, nsort * 4));
    CK(ensure(ctx->sk1, nsort * 4));
    CK(ensure(ctx->sv1, nsort * 4));
    CK(ensure(ctx->counts, std::max(radix_counts_len(R, N), radix_counts_len(1, NT)) * 4));
    const size_t scan_n = std::max({radix_counts_len(R, N), (size_t)nq, (size_t)1});
    CK(ensure(ctx->scan_tmp, scan_tmp_bytes(scan_n)));
    CK(ensure(ctx->qperm, NR * 4));
    CK(ensure(ctx->qskey, NR * 4));
    CK(ensure(ctx->tperm, (size_t)NT * 4 + 4));
    CK(ensure(ctx->tskey, (size_t)NT * 4 + 4));
    CK(ensure(ctx->tmin, (size_t)TT * 4));
    CK(ensure(ctx->tmax, (size_t)TT * 4));
    CK(ensure(ctx->cmax, (size_t)TT * 4));
    CK(ensure(ctx->cmin, (size_t)TT * 4));
    CK(ensure(ctx->ranges, (size_t)nq * 8));
    CK(ensure(ctx->cost, (size_t)nq * 8));
    CK(ensure(ctx->cum, (size_t)nq * 8));
    CK(ensure(ctx->nitem, (size_t)nq * 4));
    CK(ensure(ctx->item_off, (size_t)nq * 4));
    DevCounters hc{};
    hc.tq_begin = INT_MAX;
    hc.tq_end = 0;
    CK(cudaMemcpyAsync(ctx->ctr.p, &hc, sizeof hc, cudaMemcpyHostToDevice, s));
    DevCounters* dctr = P<DevCounters>(ctx->ctr);

    // ---- relation-factored L2 (l2_engine 5): one G = H T^T tile serves every
    // relation; no pivots, sorts or pruning (it is the engine for data where tiles do not prune)
    if (norm == 2 && ctx->opt.l2_engine == 5 && tc && ex.Nt < 0 && !ex.A64 && !ex.Et) {
        const long long ntpad = (long long)TT * BN_TC;
        CK(ensure(ctx->tperm, (size_t)ntpad * 4));
        CK(ensure(ctx->qperm, (size_t)N * 4));
        launch_iota(P<int>(ctx->tperm), N, s);  // natural order on both sides
        launch_iota(P<int>(ctx->qperm), N, s);
        CK(ensure(ctx->fz, (size_t)R * N * 4));
        CK(ensure(ctx->frt, (size_t)R * ntpad * 4));
        CK(ensure(ctx->frn, (size_t)R * 4));
        CK(ensure(ctx->fzero, (size_t)d * 4));
        CK(cudaMemsetAsync(ctx->fzero.p, 0, (size_t)d * 4, s));
        launch_factored_tables(E, Rel, P<int>(ctx->tperm), N, R, d, feps, ntpad, P<float>(ctx->fz),
                               P<float>(ctx->frt), P<float>(ctx->frn), &dctr->nonfinite, s);
        LAUNCHED(3);
        CK(cudaEventRecord(ctx->ev[EV_KEYS], s));
        CK(cudaEventRecord(ctx->ev[EV_SORT], s));
        // this rank's head tiles (uniform dense work: a contiguous split), every tail tile
        const long long ha = (long long)QT * ctx->opt.rank / ctx->opt.world;
        const long long hb = (long long)QT * (ctx->opt.rank + 1) / ctx->opt.world;
        ctx->fitems.clear();
        for (long long q = ha; q < hb; ++q)
            for (int j0 = 0; j0 < TT; j0 += chunk)
                ctx->fitems.push_back(make_int4((int)q, j0, std::min(TT - 1, j0 + chunk - 1), -1));
        const long long n_items = (long long)ctx->fitems.size();
        st.tile_pairs_total = (long long)QT * TT;
        st.tile_pairs_surviving = st.tile_pairs_total;
        st.tile_pairs_mine = (hb - ha) * TT;
        st.work_items_mine = n_items;
        st.engine = 7;
        if (n_items > 0) {
            CK(ensure(ctx->items, (size_t)n_items * 16));
            CK(cudaMemcpyAsync(ctx->items.p, ctx->fitems.data(), (size_t)n_items * 16, cudaMemcpyHostToDevice, s));
        }
        CK(cudaEventRecord(ctx->ev[EV_RANGES], s));
        CK(ensure(ctx->Tp, (size_t)TT * BN * Kpad * 4));
        CK(ensure(ctx->T2, (size_t)TT * BN * 4));
        CK(ensure(ctx->tstile, (size_t)TT * 8));
        launch_stage_tails(E, P<int>(ctx->tperm), N, d, Kpad, BN, TT, 1, P<float>(ctx->Tp), P<float>(ctx->T2),
                           P<float2>(ctx->tstile), s);
        LAUNCHED(1);
        CK(cudaEventRecord(ctx->ev[EV_STAGE], s));
        if (ctx->cand_cap == 0) ctx->cand_cap = 1 << 20;
        if (ctx->res_cap == 0) ctx->res_cap = ctx->opt.result_capacity > 0 ? ctx->opt.result_capacity : (1 << 20);
        long long cand_n = 0, res_n = 0;
        for (;;) {
            CK(ensure(ctx->cand, (size_t)ctx->cand_cap * 8));
            CK(ensure(ctx->res, (size_t)ctx->res_cap * 16));
            CK(cudaMemsetAsync(&dctr->cand, 0, 16, s));
            TileParams tp{};
            tp.Tp = P<float>(ctx->Tp);
            tp.T2 = P<float>(ctx->T2);
            tp.tstile = P<float2>(ctx->tstile);
            tp.items = P<int4>(ctx->items);
            tp.n_items = n_items;
            tp.total_tiles = st.tile_pairs_mine;
            tp.Kpad = Kpad;
            tp.bq = bq;
            tp.bn = BN;
            tp.N = (int)N;
            tp.Nt = (int)N;
            tp.theta = feps;
            tp.eta = (float)((Kpad / 8) * 3.814697265625e-06);
            tp.cand = P<int2>(ctx->cand);
            tp.cand_count = &dctr->cand;
            tp.cand_cap = ctx->cand_cap;
            tp.E = E;
            tp.Rel = P<float>(ctx->fzero);  // builders form fl32(h + 0) = h
            tp.qperm = P<int>(ctx->qperm);
            tp.d = d;
            tp.QT = QT;
            tp.fz = P<float>(ctx->fz);
            tp.frt = P<float>(ctx->frt);
            tp.frn = P<float>(ctx->frn);
            tp.R = (int)R;
            tp.ntpad = ntpad;
            if (n_items > 0) {
                launch_tiles_tc_factored(tp, ctx->num_sms, s);
                LAUNCHED(1);
            }
            CK(cudaEventRecord(ctx->ev[EV_TILES], s));
            if (n_items > 0) {
                launch_verify(P<int2>(ctx->cand), &dctr->cand, ctx->cand_cap, nullptr, nullptr, E, Rel, E, N, QT, bq, d,
                              norm, eps, reinterpret_cast<KgcTripletDev*>(ctx->res.p), &dctr->res, ctx->res_cap,
                              ctx->num_sms, s, r_off);
                LAUNCHED(1);
            }
            CK(cudaEventRecord(ctx->ev[EV_VERIFY], s));
            unsigned long long hcnt[2];
            unsigned int nf = 0;
            CK(cudaMemcpyAsync(hcnt, &dctr->cand, 16, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(&nf, &dctr->nonfinite, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (nf) {
                set_err(ctx, "non-finite value in E or Rel");
                return KGC_EDATA;
            }
            cand_n = (long long)hcnt[0];
            res_n = (long long)hcnt[1];
            if (cand_n > ctx->cand_cap) {
                ctx->cand_cap = cand_n + cand_n / 4 + 1024;
                st.reruns++;
                continue;
            }
            if (res_n > ctx->res_cap) {
                ctx->res_cap = res_n + res_n / 4 + 1024;
                st.reruns++;
                continue;
            }
            break;
        }
        st.candidates = cand_n;
        st.results = res_n;
        st.launches = ctx->launches;
        float ms[EV_COUNT] = {};
        for (int k = 1; k < EV_COUNT; ++k) cudaEventElapsedTime(&ms[k], ctx->ev[k - 1], ctx->ev[k]);
        st.ms_h2d = ms[EV_H2D];
        st.ms_keys = ms[EV_KEYS];
        st.ms_ranges = ms[EV_RANGES];
        st.ms_stage = ms[EV_STAGE];
        st.ms_tiles = ms[EV_TILES];
        st.ms_recheck = ms[EV_VERIFY];
        cudaEventElapsedTime(&st.ms_total, ctx->ev[EV_START], ctx->ev[EV_VERIFY]);
        ctx->n_results = res_n;
        ctx->have_join = true;
        return KGC_OK;
    }

    const double* pivot = nullptr;
    if (ctx->opt.pivot == 1) {
        CK(ensure(ctx->pivot, (size_t)d * 8));
        launch_pivot_mean(Et, NT, d, P<double>(ctx->pivot), s);
        LAUNCHED(1);
        pivot = P<double>(ctx->pivot);
    }
    if (norm == 1 && ctx->opt.l1_engine == 1) {
        launch_absmax(E, N * d, Rel, R * d, &dctr->absmax_bits, s);
        LAUNCHED(1);
    }
    const int K = (ctx->opt.pivots >= 2 && ctx->opt.prune && d <= MP_MAX_DIM) ? ctx->opt.pivots : 1;
    ctx->K = K;
    ctx->d = d;
    st.pivots_used = K;
    if (K == 1) {
        // ---- a2: K1 keys (one pivot, FP64 -> float)
        launch_tail_keys(Et, NT, d, norm, pivot, P<float>(ctx->kt), P<unsigned>(ctx->mm_t), &dctr->nonfinite, s);
        LAUNCHED(2);
        launch_query_keys(E, Rel, N, R, d, norm, pivot, P<float>(ctx->kq), P<unsigned>(ctx->mm_q), &dctr->nonfinite,
                          s);
        LAUNCHED(2);
        CK(cudaEventRecord(ctx->ev[EV_KEYS], s));
        // ---- a3: K2 sorts (tails once, queries per relation)
        radix_sort_segments(P<float>(ctx->kt), P<unsigned>(ctx->mm_t), 1, NT, P<unsigned>(ctx->sk0),
                            P<unsigned>(ctx->sv0), P<unsigned>(ctx->sk1), P<unsigned>(ctx->sv1), P<int>(ctx->counts),
                            P<int>(ctx->tperm), P<float>(ctx->tskey), ctx->scan_tmp.p, ctx->scan_tmp.n, s,
                            &ctx->launches);
        LAUNCHED(0);
        radix_sort_segments(P<float>(ctx->kq), P<unsigned>(ctx->mm_q), R, N, P<unsigned>(ctx->sk0),
                            P<unsigned>(ctx->sv0), P<unsigned>(ctx->sk1), P<unsigned>(ctx->sv1), P<int>(ctx->counts),
                            P<int>(ctx->qperm), P<float>(ctx->qskey), ctx->scan_tmp.p, ctx->scan_tmp.n, s,
                            &ctx->launches);
        LAUNCHED(0);
        CK(cudaEventRecord(ctx->ev[EV_SORT], s));
        // ---- a4: K3 tile ranges (Lemma 1 + 2 at tile granularity)
        launch_tail_tile_bounds(P<float>(ctx->tskey), NT, BN, TT, P<float>(ctx->tmin), P<float>(ctx->tmax),
                                P<float>(ctx->cmax), P<float>(ctx->cmin), s, &ctx->launches);
        LAUNCHED(0);
        launch_query_ranges(P<float>(ctx->qskey), N, R, QT, TT, bq, P<float>(ctx->cmax), P<float>(ctx->cmin), feps,
                            ctx->opt.prune, P<int2>(ctx->ranges), P<long long>(ctx->cost), s);
        LAUNCHED(1);
    } else {
        // ---- a2: K pivot distances per row (FP32)
        CK(ensure(ctx->mpP, (size_t)K * d * 4));
        CK(ensure(ctx->mpkt, (size_t)NT * K * 4 + 4));
        if (norm == 1) CK(ensure(ctx->mpkq, NR * K * 4));  // L1: materialised FP32 keys; L2: on the fly
        if (norm == 1 && K > MP_MAX_L1) {
            set_err(ctx, "pivots > %d need norm 2 (the L1 keys support at most %d pivots)", MP_MAX_L1, MP_MAX_L1);
            return KGC_EINVAL;
        }
        ctx->l2f = norm == 2;
        CK(ensure(ctx->mpmm_t, (size_t)K * 8));
        CK(ensure(ctx->mpmm_q, (size_t)R * K * 8));
        CK(ensure(ctx->mpqn, (size_t)R * 4));
        CK(ensure(ctx->mpc0, nsort * 8));
        CK(ensure(ctx->mpc1, nsort * 8));
        CK(ensure(ctx->tbmin, (size_t)TT * K * 4));
        CK(ensure(ctx->tbmax, (size_t)TT * K * 4));
        CK(ensure(ctx->qbmin, (size_t)nq * K * 4));
        CK(ensure(ctx->qbmax, (size_t)nq * K * 4));
        if (norm == 2) {  // the h.r GEMM needs no pivots: it runs on the aux stream beside the pivot choice
            CK(ensure(ctx->mpB, (size_t)N * R * 8));
            CK(cudaEventRecord(ctx->ev_fork[0], s));
            CK(cudaStreamWaitEvent(ctx->aux, ctx->ev_fork[0], 0));
            launch_mp_hr(E, Rel, N, R, d, P<double>(ctx->mpB), ctx->aux);
            CK(cudaEventRecord(ctx->ev_fork[1], ctx->aux));
            LAUNCHED(1);
        }
        if (!ctx->pivots_ready) {  // split 3 launched it already, beside the head order
            launch_pick_pivots(Et, NT, d, norm, K, pivot, P<float>(ctx->mpP), s);
            LAUNCHED(1);
        }
        if (norm == 2) {  // FP64 factorisation: one h.r dot product per query row instead of K distances
            const int KO = K < MP_SORT_PIVOTS ? K : MP_SORT_PIVOTS;
            CK(ensure(ctx->mpA, (size_t)N * K * 8));
            CK(ensure(ctx->mpC, (size_t)R * (K + 1) * 8));
            CK(ensure(ctx->mpk4, NR * KO * 4));
            CK(ensure(ctx->mpmm4, (size_t)R * KO * 8));
            CK(ensure(ctx->mphx, 16));
            CK(ensure(ctx->mpHP, (size_t)std::max<long long>(N, NT) * K * 8));
            launch_mp_keys_l2f(E, Rel, N, R, Et, NT, d, K, P<float>(ctx->mpP), P<float>(ctx->mpkt),
                               P<unsigned>(ctx->mpmm_t), P<float>(ctx->mpk4), P<unsigned>(ctx->mpmm4),
                               P<unsigned>(ctx->mpqn), P<double>(ctx->mpA), P<double>(ctx->mpB), P<double>(ctx->mpC),
                               P<double>(ctx->mpHP), P<unsigned>(ctx->mphx), &dctr->nonfinite, &dctr->twid, s,
                               ctx->ev_fork[1]);
            LAUNCHED((Et == E && NT == N) ? 5 : 6);
        } else {
            launch_mp_keys(Et, nullptr, NT, 1, d, norm, K, P<float>(ctx->mpP), P<float>(ctx->mpkt),
                           P<unsigned>(ctx->mpmm_t), nullptr, &dctr->nonfinite, s);
            LAUNCHED(2);
            launch_mp_keys(E, Rel, N, R, d, norm, K, P<float>(ctx->mpP), P<float>(ctx->mpkq), P<unsigned>(ctx->mpmm_q),
                           P<unsigned>(ctx->mpqn), &dctr->nonfinite, s);
            LAUNCHED(2);
        }
        CK(cudaEventRecord(ctx->ev[EV_KEYS], s));
        // ---- a3: Morton-order sorts (tiles compact in pivot space)
        const int bits = 8;  // per pivot, over the first min(K, MP_SORT_PIVOTS) pivots
        launch_mp_morton(P<float>(ctx->mpkt), P<unsigned>(ctx->mpmm_t), 1, NT, K, bits,
                         P<unsigned>(ctx->mpc0), P<unsigned>(ctx->sv0), s);
        LAUNCHED(1);
        const int code_bits = bits * (K < MP_SORT_PIVOTS ? K : MP_SORT_PIVOTS);  // <= 32: 32-bit codes
        radix_sort_u32_segments(1, NT, code_bits, P<unsigned>(ctx->mpc0), P<unsigned>(ctx->sv0),
                                P<unsigned>(ctx->mpc1), P<unsigned>(ctx->sv1), P<int>(ctx->counts),
                                ctx->scan_tmp.p, s, &ctx->launches);
        LAUNCHED(0);
        CK(cudaMemcpyAsync(ctx->tperm.p, ctx->sv0.p, (size_t)NT * 4, cudaMemcpyDeviceToDevice, s));
        const char* kde = kgc_knob("KGC_KD");  // local kd refinement of both orders (experiment knob)
        const bool kd = kde ? atoi(kde) != 0 : false;
        if (kd) launch_kd_refine(P<float>(ctx->mpkt), P<int>(ctx->tperm), 1, NT, K, s);
        // the Hilbert pivots' keys (L2: the first 4 from the factorisation; the rest are computed
        // on the fly by the boxes; L1: the materialised keys)
        const float* qk4 = norm == 2 ? P<float>(ctx->mpk4) : P<float>(ctx->mpkq);
        const unsigned* qmm4 = norm == 2 ? P<unsigned>(ctx->mpmm4) : P<unsigned>(ctx->mpmm_q);
        const int qks = norm == 2 ? (K < MP_SORT_PIVOTS ? K : MP_SORT_PIVOTS) : K;
        if (launch_mp_sort_small(qk4, qmm4, R, N, qks, bits, P<int>(ctx->qperm), s)) {  // short segments (c3)
            LAUNCHED(1);
        } else {
            launch_mp_morton(qk4, qmm4, R, N, qks, bits, P<unsigned>(ctx->mpc0), P<unsigned>(ctx->sv0), s);
            LAUNCHED(1);
            radix_sort_u32_segments(R, N, code_bits, P<unsigned>(ctx->mpc0), P<unsigned>(ctx->sv0),
                                    P<unsigned>(ctx->mpc1), P<unsigned>(ctx->sv1), P<int>(ctx->counts),
                                    ctx->scan_tmp.p, s, &ctx->launches);
            LAUNCHED(0);
            CK(cudaMemcpyAsync(ctx->qperm.p, ctx->sv0.p, NR * 4, cudaMemcpyDeviceToDevice, s));
        }
        if (kd && norm == 1) launch_kd_refine(P<float>(ctx->mpkq), P<int>(ctx->qperm), R, N, K, s);
        CK(cudaEventRecord(ctx->ev[EV_SORT], s));
        // ---- a4: K-dim tile boxes and the L_inf test of every tile pair
        // tail boxes [k][TT]; L2: widened by the GEMM-form tail-key bound delta_t (DevCounters::twid)
        launch_mp_boxes(P<float>(ctx->mpkt), P<unsigned>(ctx->tperm), 1, NT, BN, TT, K, P<float>(ctx->tbmin),
                        P<float>(ctx->tbmax), norm == 2 ? &dctr->twid : nullptr, s, 1);
        if (norm == 2)
            launch_mp_qboxes_fact(P<unsigned>(ctx->qperm), P<double>(ctx->mpB), P<double>(ctx->mpA), P<double>(ctx->mpC),
                                  N, R, K, bq, QT, P<unsigned>(ctx->mpqn), P<float>(ctx->qbmin), P<float>(ctx->qbmax), s);
        else
            launch_mp_boxes(P<float>(ctx->mpkq), P<unsigned>(ctx->qperm), R, N, bq, QT, K, P<float>(ctx->qbmin),
                            P<float>(ctx->qbmax), P<unsigned>(ctx->mpqn), s);
        LAUNCHED(2);
        // survival masks kept for mp_emit when they fit (c4: 2.2 MB; c5: 380 MB; beyond 2 GiB: recompute)
        const size_t bits_bytes = (size_t)nq * ((TT + 31) / 32) * 4;
        unsigned int* sbits = nullptr;
        if (bits_bytes <= (2ull << 30)) {
            CK(ensure(ctx->mpbits, bits_bytes + 4));
            sbits = P<unsigned int>(ctx->mpbits);
        }
        ctx->mp_bits = sbits;
        launch_mp_count(P<float>(ctx->qbmin), P<float>(ctx->qbmax), P<float>(ctx->tbmin), P<float>(ctx->tbmax), nq, TT,
                        K, feps, mp_relm(d), 1, P<int2>(ctx->ranges), P<long long>(ctx->cost), sbits, s);
        LAUNCHED(1);
    }
    scan_exclusive_i64(P<long long>(ctx->cost), P<long long>(ctx->cum), (size_t)nq, &dctr->total_cost,
                       ctx->scan_tmp.p, s, &ctx->launches);
    LAUNCHED(0);
    launch_shard_items(P<int2>(ctx->ranges), P<long long>(ctx->cost), P<long long>(ctx->cum), nq, ctx->opt.rank,
                       ctx->opt.world, chunk, dctr, P<int>(ctx->nitem), P<int>(ctx->item_off), nullptr, nullptr,
                       ctx->scan_tmp.p, s, &ctx->launches, 0, 0, force_lo, force_hi);
    LAUNCHED(0);
    // sync #1: plan totals
    struct {
        DevCounters c;
        int last_n, last_off;
    } h1{};
    CK(cudaMemcpyAsync(&h1.c, ctx->ctr.p, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&h1.last_n, P<int>(ctx->nitem) + (nq - 1), 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&h1.last_off, P<int>(ctx->item_off) + (nq - 1), 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h1.c.nonfinite) {
        set_err(ctx, "non-finite value in E or Rel");
        return KGC_EDATA;
    }
    const long long n_items = (long long)h1.last_off + h1.last_n;
    st.tile_pairs_surviving = h1.c.total_cost;
    st.tile_pairs_mine = h1.c.my_cost;
    st.work_items_mine = n_items;
    const int tq0 = h1.c.tq_begin == INT_MAX ? 0 : h1.c.tq_begin;
    const int tq1 = h1.c.tq_begin == INT_MAX ? 0 : h1.c.tq_end;
    ctx->list_len = 0;
    ctx->glist_len = 0;
    // Lists are laid out by the surviving-tile prefix over this shard's query-tile range; with the
    // cyclic split (force_lo == -2) that range interleaves other ranks' tiles: size by the total.
    const bool cyc = force_lo == -2;
    const long long list_span = cyc ? h1.c.total_cost : h1.c.my_cost;
    if (n_items > 0 && K > 1) {
        ctx->list_len = list_span;
        CK(ensure(ctx->tile_list, (size_t)list_span * 4 + 4));
        launch_mp_emit(P<float>(ctx->qbmin), P<float>(ctx->qbmax), P<float>(ctx->tbmin), P<float>(ctx->tbmax),
                       P<long long>(ctx->cum), dctr, nq, TT, K, feps, mp_relm(d), 1, P<int>(ctx->tile_list), ctx->mp_bits,
                       s);
        LAUNCHED(1);
    }
    // Gathered tails: per query tile, the tails of its surviving tiles that pass the K-pivot
    // test on their own keys, in blocks of GT_ROWS; work items reference blocks.
    const bool gather = n_items > 0 && K > 1 && !tc && !half_req && simt_t() == GT_ROWS && use_gather(ctx, norm);
    const bool gather_tc = n_items > 0 && gtc_req && K > 1 && (gtc_pair ? tc2_gather_ok(Kpad) : tc_gather_ok(Kpad)) &&
                           (size_t)list_span * BN_TC * 8 <= GATHER_TC_BUDGET;
    // rows per gathered block: tensor cores 256 (= tail tile rows); SIMT 64 or 32 (KGC_GT_TB experiment knob)
    const char* gtb = kgc_knob("KGC_GT_TB");
    const int GB = gather_tc ? BN_TC : ((gtb && atoi(gtb) == 32) ? 32 : GT_ROWS);
    long long g_max_items = 0;
    if (gather || gather_tc) {
        g_max_items = h1.c.my_cost * (BN / GB > 1 ? BN / GB : 1);  // blocks (and items) <= tiles x rows per block
        CK(ensure(ctx->Ts, (size_t)(NT + 1) * Kpad * 4));
        CK(ensure(ctx->tks, (size_t)NT * MP_G * 4 + 4));
        CK(ensure(ctx->gblk, (size_t)nq * 8));
        CK(ensure(ctx->granges, (size_t)nq * 8));
        CK(ensure(ctx->glist, (size_t)list_span * BN * 4 + 4));  // laid out at BN x the tile-list offsets
        CK(ensure(ctx->items, (size_t)g_max_items * 16));
        CK(ensure(ctx->item_tiles, (size_t)g_max_items * 8));
        CK(ensure(ctx->item_cum, (size_t)g_max_items * 8));
        CK(ensure(ctx->scan_tmp, scan_tmp_bytes((size_t)std::max<long long>(g_max_items, nq))));
        if (gather_tc) {
            CK(ensure(ctx->tsc, (size_t)NT * 16 + 16));
            CK(ensure(ctx->gT2, (size_t)list_span * GB * 4 + 4));
            CK(ensure(ctx->gtst, (size_t)list_span * 8));
        }
        launch_stage_rows(Et, P<int>(ctx->tperm), P<float>(ctx->mpkt), NT, d, Kpad, K, P<float>(ctx->Ts),
                          P<float>(ctx->tks), gather_tc ? P<float4>(ctx->tsc) : nullptr, s);
        if (gather_tc && !gtc_pair) {  // the 1-CTA engine gathers with TMA row gathers
            CK(ensure(ctx->tmapbuf, sizeof(CUtensorMap)));
            if (make_tails_tmap(&ctx->tmap_host, P<float>(ctx->Ts), NT + 1, Kpad)) {
                set_err(ctx, "cuTensorMapEncodeTiled failed for the gathered tails");
                return KGC_ECUDA;
            }
            CK(cudaMemcpyAsync(ctx->tmapbuf.p, &ctx->tmap_host, sizeof(CUtensorMap), cudaMemcpyHostToDevice, s));
        }
        CK(cudaMemsetAsync(ctx->gblk.p, 0, (size_t)nq * 8, s));
        CK(cudaMemsetAsync(ctx->nitem.p, 0, (size_t)nq * 4, s));
        CK(cudaMemsetAsync(ctx->item_tiles.p, 0, (size_t)g_max_items * 8, s));
        // the per-tail test reads single tail keys: with the L2 GEMM-form keys widen theta by delta_t
        const float gtheta = norm == 2 ? std::nextafter(feps + ldexpf(__uint_as_float_host(h1.c.twid), -23), INFINITY)
                                       : feps;
        launch_gather_tails(P<float>(ctx->qbmin), P<float>(ctx->qbmax), P<float>(ctx->tks), P<int>(ctx->tile_list),
                            P<long long>(ctx->cum), P<int2>(ctx->ranges), dctr, NT, BN, K, gtheta, mp_relm(d), chunk, nq,
                            P<long long>(ctx->gblk), P<int2>(ctx->granges), P<int>(ctx->nitem), P<int>(ctx->glist),
                            gather_tc ? P<float4>(ctx->tsc) : nullptr, gather_tc ? P<float>(ctx->gT2) : nullptr,
                            gather_tc ? P<float2>(ctx->gtst) : nullptr, cyc ? ctx->opt.world : 0, ctx->opt.rank,
                            s, GB);
        LAUNCHED(2);
        scan_exclusive_i32(P<int>(ctx->nitem), P<int>(ctx->item_off), (size_t)nq, ctx->scan_tmp.p, s,
                           &ctx->launches);
        LAUNCHED(0);
        // items {q, b0, b1, tile-list offset of q}: block b of q is glist[GT_ROWS * (offset + b) ...]
        launch_shard_items(P<int2>(ctx->granges), nullptr, P<long long>(ctx->cum), nq, ctx->opt.rank,
                           ctx->opt.world, chunk, dctr, P<int>(ctx->nitem), P<int>(ctx->item_off),
                           P<int4>(ctx->items), P<long long>(ctx->item_tiles), ctx->scan_tmp.p, s, &ctx->launches, 1,
                           1, force_lo, force_hi);
        LAUNCHED(0);
        scan_exclusive_i64(P<long long>(ctx->item_tiles), P<long long>(ctx->item_cum), (size_t)g_max_items, nullptr,
                           ctx->scan_tmp.p, s, &ctx->launches);
        LAUNCHED(0);
    } else if (n_items > 0) {
        CK(ensure(ctx->items, (size_t)n_items * 16));
        CK(ensure(ctx->item_tiles, (size_t)n_items * 8));
        CK(ensure(ctx->item_cum, (size_t)n_items * 8));
        CK(ensure(ctx->scan_tmp, scan_tmp_bytes((size_t)n_items)));
        launch_shard_items(P<int2>(ctx->ranges), P<long long>(ctx->cost), P<long long>(ctx->cum), nq, ctx->opt.rank,
                           ctx->opt.world, chunk, dctr, P<int>(ctx->nitem), P<int>(ctx->item_off),
                           P<int4>(ctx->items), P<long long>(ctx->item_tiles), ctx->scan_tmp.p, s, &ctx->launches, 1,
                           K > 1 ? 1 : 0, force_lo, force_hi);
        LAUNCHED(0);
        scan_exclusive_i64(P<long long>(ctx->item_tiles), P<long long>(ctx->item_cum), (size_t)n_items, nullptr,
                           ctx->scan_tmp.p, s, &ctx->launches);
        LAUNCHED(0);
    }
    CK(cudaEventRecord(ctx->ev[EV_RANGES], s));

    // ---- stage operand tiles (tails: all; queries: this shard's range)
    // FP16x2 L1 engine only on request (l1_engine = 1) and when every |value| <= 1000 (FP16 range and
    // partial sums safe).  Measured on B200 it is no faster than FP32: HADD2 issues at half the FADD rate,
    // so two elements per instruction buy nothing (scripts/micro/l1_inner.cu).
    const bool half = half_req && __uint_as_float_host(h1.c.absmax_bits) <= 1000.0f;
    if (half_req && !half) {
        set_err(ctx, "l1_engine=1 (FP16x2) needs every |E|, |Rel| value <= 1000; use l1_engine 0 or 2");
        return KGC_EINVAL;
    }
    st.engine = gather_tc ? (gtc_pair ? 8 : 6) : ((tc2 || gtc_pair) ? 4 : (tc ? 1 : (half ? 3 : (gather ? 5 : 2))));
    const float gam = 1.0f + 10.0f * 4.8828125e-04f + (float)(d / 8 + 4) * 1.1920928955078125e-07f;
    if (n_items > 0) {
        CK(ensure(ctx->Tp, (size_t)TT * BN * Kpad * 4));
        CK(ensure(ctx->T2, (size_t)TT * BN * 4));
        CK(ensure(ctx->tstile, (size_t)TT * 8));
        if (half) {
            CK(ensure(ctx->Qp, (size_t)(tq1 - tq0) * bq * Kpad * 2));
            CK(ensure(ctx->qs, (size_t)(tq1 - tq0) * bq * 16));
            launch_stage_half(Et, nullptr, P<int>(ctx->tperm), NT, d, Kpad, BN, 1, 0, TT, feps, gam, ctx->Tp.p, nullptr,
                              P<float>(ctx->T2), s);
            launch_stage_half(E, Rel, P<int>(ctx->qperm), N, d, Kpad, bq, QT, tq0, tq1 - tq0, feps, gam, ctx->Qp.p,
                              P<float4>(ctx->qs), nullptr, s);
            LAUNCHED(2);
        } else if (gather_tc) {
            // nothing to stage: builder warps form the query tiles, the producer gathers the tails
        } else if (gather) {
            CK(ensure(ctx->Qp, (size_t)(tq1 - tq0) * bq * Kpad * 4));
            CK(ensure(ctx->qs, (size_t)(tq1 - tq0) * bq * 16));
            launch_stage_queries(E, Rel, P<int>(ctx->qperm), N, d, Kpad, QT, bq, tq0, tq1, 0, norm, feps,
                                 P<float>(ctx->Qp), P<float4>(ctx->qs), s, cyc ? ctx->opt.world : 0, ctx->opt.rank);
            LAUNCHED(1);
        } else {
            // pair engine: 256-row tiles as two 128-row UMMA blocks (layout 2); 128-row tiles whole (layout 1)
            launch_stage_tails(Et, P<int>(ctx->tperm), NT, d, Kpad, BN, TT, ((tc2 || gtc_pair) && BN == BN_TC) ? 2 : (tc ? 1 : 0), P<float>(ctx->Tp),
                               P<float>(ctx->T2), P<float2>(ctx->tstile), s);
            LAUNCHED(1);
            if (!tc) {  // the tensor-core engine forms its query tiles on the fly
                CK(ensure(ctx->Qp, (size_t)(tq1 - tq0) * bq * Kpad * 4));
                CK(ensure(ctx->qs, (size_t)(tq1 - tq0) * bq * 16));
                launch_stage_queries(E, Rel, P<int>(ctx->qperm), N, d, Kpad, QT, bq, tq0, tq1, 0, norm, feps,
                                     P<float>(ctx->Qp), P<float4>(ctx->qs), s, cyc ? ctx->opt.world : 0,
                                     ctx->opt.rank);
                LAUNCHED(1);
            }
        }
    }
    CK(cudaEventRecord(ctx->ev[EV_STAGE], s));

    // ---- a5/a6 tiles, a7/a8 verify (rerun on capacity overflow)
    if (ctx->cand_cap == 0) ctx->cand_cap = 1 << 20;
    if (ctx->res_cap == 0) ctx->res_cap = ctx->opt.result_capacity > 0 ? ctx->opt.result_capacity : (1 << 20);
    long long cand_n = 0, res_n = 0;
    for (int attempt = 0;; ++attempt) {
        CK(ensure(ctx->cand, (size_t)ctx->cand_cap * 8));
        CK(ensure(ctx->res, (size_t)ctx->res_cap * 16));
        CK(cudaMemsetAsync(&dctr->cand, 0, 16, s));  // cand + res counters
        if (attempt > 0) CK(cudaEventRecord(ctx->ev[EV_STAGE], s));
        TileParams tp{};
        tp.Qp = P<float>(ctx->Qp);
        tp.qs = P<float4>(ctx->qs);
        tp.Tp = P<float>(ctx->Tp);
        tp.T2 = P<float>(ctx->T2);
        tp.tstile = P<float2>(ctx->tstile);
        tp.items = P<int4>(ctx->items);
        tp.tile_list = P<int>(ctx->tile_list);
        tp.n_items = n_items;
        tp.item_cum = P<long long>(ctx->item_cum);
        tp.total_tiles = h1.c.my_cost;
        {   // tuning knob for experiments: KGC_SCHED_TC / KGC_SCHED_SIMT = 0 (round-robin) | 1 (balanced blocks)
            const char* e = kgc_knob(tc ? "KGC_SCHED_TC" : "KGC_SCHED_SIMT");
            tp.sched = e ? atoi(e) : (tc ? 0 : 1);
        }
        {
            const char* e = kgc_knob("KGC_T2_PREFETCH");
            tp.t2pf = e ? atoi(e) : ((tc2 || gtc_pair) ? 1 : 0);  // measured: helps the pair kernel, not the 1-CTA one
        }
        {
            const char* e = kgc_knob("KGC_L2HINT");
            tp.l2hint = e ? atoi(e) : 1;
        }
        tp.Kpad = Kpad;
        tp.bq = bq;
        tp.bn = BN;
        tp.tq0 = tq0;
        tp.N = (int)N;
        tp.Nt = (int)NT;
        tp.theta = feps;
        tp.gam = gam;
        tp.Rt = P<float>(ctx->T2);
        tp.eta = (float)((Kpad / 8) * 3.814697265625e-06);  // Ksteps * 2^-18
        tp.cand = P<int2>(ctx->cand);
        tp.cand_count = &dctr->cand;
        tp.cand_cap = ctx->cand_cap;
        tp.E = E;
        tp.Rel = Rel;
        tp.qperm = P<int>(ctx->qperm);
        tp.d = d;
        tp.QT = QT;
        tp.Ts = P<float>(ctx->Ts);
        tp.glist = P<int>(ctx->glist);
        tp.dn_items = &dctr->n_items;
        tp.dtotal = &dctr->gblocks;
        tp.gT2 = P<float>(ctx->gT2);
        tp.gtst = P<float2>(ctx->gtst);
        tp.tmap = ctx->tmapbuf.p;
        tp.gb = GB;
        if (n_items > 0) {
            if (gather) {
                const char* pe = kgc_knob("KGC_GT_PROF");  // experiment: wait-cycle instrumentation
                unsigned long long* prof = nullptr;
                if (pe && atoi(pe)) {
                    CK(cudaMalloc(&prof, 16 * 8));
                    CK(cudaMemsetAsync(prof, 0, 128, s));
                }
                tp.prof = prof;
                launch_tiles_gather(tp, norm, ctx->num_sms, g_max_items, s);
                if (prof) {
                    unsigned long long h[16];
                    CK(cudaMemcpyAsync(h, prof, 128, cudaMemcpyDeviceToHost, s));
                    CK(cudaStreamSynchronize(s));
                    cudaFree(prof);
                    fprintf(stderr, "gt_prof warps %llu avg cycles %.0f | wait/warp: item-start %.0f (%llu) "
                            "block-start %.0f (%llu) other %.0f (%llu) | waited: issue->ready %.0f cycles (%llu)\n", h[7],
                            (double)h[6] / h[7], (double)h[0] / h[7], h[1], (double)h[2] / h[7], h[3],
                            (double)h[4] / h[7], h[5], h[9] ? (double)h[8] / h[9] : 0.0, h[9]);
                }
            }
            else if (gather_tc) {
                TileParams tg = tp;
                tg.n_items = g_max_items;  // grid bound; the kernel reads the item count on the device
                if (gtc_pair) launch_tiles_tc2_gather(tg, ctx->num_sms, s);
                else launch_tiles_tc_gather(tg, ctx->num_sms, s);
            } else if (tc2 || gtc_pair) launch_tiles_tc2(tp, ctx->num_sms, s);  // gtc_pair: list fallback
            else if (tc) launch_tiles_tc(tp, ctx->num_sms, s);
            else if (half) launch_tiles_half_l1(tp, ctx->num_sms, s);
            else launch_tiles_simt(tp, norm, ctx->num_sms, s);
            LAUNCHED(1);
        }
        CK(cudaEventRecord(ctx->ev[EV_TILES], s));
        if (n_items > 0) {
            if (ex.A64)
                launch_verify_se(P<int2>(ctx->cand), &dctr->cand, ctx->cand_cap, P<int>(ctx->qperm),
                                 P<int>(ctx->tperm), ex.A64, ex.B64, N, (long long)QT * bq, d, eps,
                                 reinterpret_cast<KgcTripletDev*>(ctx->res.p), &dctr->res, ctx->res_cap,
                                 ctx->num_sms, s, r_off);
            else {
                // E back into L2 for the row gathers (the tile kernel streamed the staged tails through it)
                if ((size_t)N * d * 4 > (32u << 20)) {
                    launch_l2_prefetch(E, (size_t)N * d * 4, ctx->num_sms, s);
                    if (Et != E) launch_l2_prefetch(Et, (size_t)NT * d * 4, ctx->num_sms, s);
                    LAUNCHED(Et != E ? 2 : 1);
                }
                launch_verify(P<int2>(ctx->cand), &dctr->cand, ctx->cand_cap, P<int>(ctx->qperm), P<int>(ctx->tperm),
                              E, Rel, Et, N, QT, bq, d, norm, eps, reinterpret_cast<KgcTripletDev*>(ctx->res.p),
                              &dctr->res, ctx->res_cap, ctx->num_sms, s, r_off, NT, ex.t_off, ex.h_off, ex.hmap);
            }
            LAUNCHED(1);
        }
        CK(cudaEventRecord(ctx->ev[EV_VERIFY], s));
        unsigned long long hcnt[2], hg[2] = {0, 0};  // cand, res; gathered blocks, pairs
        CK(cudaMemcpyAsync(hcnt, &dctr->cand, 16, cudaMemcpyDeviceToHost, s));
        if (gather || gather_tc) CK(cudaMemcpyAsync(hg, &dctr->gblocks, 16, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        cand_n = (long long)hcnt[0];
        res_n = (long long)hcnt[1];
        st.gathered_pairs = (int64_t)hg[1] * bq;
        ctx->glist_len = (gather || gather_tc) ? ctx->list_len * BN : 0;
        if (cand_n > ctx->cand_cap) {
            ctx->cand_cap = cand_n + cand_n / 4 + 1024;
            st.reruns++;
            continue;
        }
        if (res_n > ctx->res_cap) {
            ctx->res_cap = res_n + res_n / 4 + 1024;
            st.reruns++;
            continue;
        }
        break;
    }
    st.candidates = cand_n;
    st.results = res_n;
    st.launches = ctx->launches;
    float ms[EV_COUNT] = {};
    for (int i = 1; i < EV_COUNT; ++i) cudaEventElapsedTime(&ms[i], ctx->ev[i - 1], ctx->ev[i]);
    st.ms_h2d = ms[EV_H2D];
    st.ms_keys = ms[EV_KEYS];
    st.ms_sort = ms[EV_SORT];
    st.ms_ranges = ms[EV_RANGES];
    st.ms_stage = ms[EV_STAGE];
    st.ms_tiles = ms[EV_TILES];
    st.ms_recheck = ms[EV_VERIFY];
    cudaEventElapsedTime(&st.ms_total, ctx->ev[EV_START], ctx->ev[EV_VERIFY]);
    ctx->n_results = res_n;
    ctx->have_join = true;
    return KGC_OK;
}

// Query-tile range [a, b) of this rank: cumulative estimated cost, each
// relation's estimate spread evenly over its QT query tiles.
static int split_range(kgc_ctx* ctx, const float* E_in, const float* Rel_in, long long N, long long R, int d, int norm,
                       float eps, long long QT, long long* a, long long* b, const float** E_dev, const float** Rel_dev,
                       long long* h2d) {
    cudaStream_t s = ctx->stream;
    const float* E = E_in;
    const float* Rel = Rel_in;
    *h2d = 0;
    if (!is_device_ptr(E_in, ctx->device)) {
        CK(ensure(ctx->E, (size_t)N * d * 4));
        CK(cudaMemcpyAsync(ctx->E.p, E_in, (size_t)N * d * 4, cudaMemcpyDefault, s));
        E = P<float>(ctx->E);
        *h2d += (long long)N * d * 4;
    }
    if (!is_device_ptr(Rel_in, ctx->device)) {
        CK(ensure(ctx->Rel, (size_t)R * d * 4));
        CK(cudaMemcpyAsync(ctx->Rel.p, Rel_in, (size_t)R * d * 4, cudaMemcpyDefault, s));
        Rel = P<float>(ctx->Rel);
        *h2d += (long long)R * d * 4;
    }
    *E_dev = E;
    *Rel_dev = Rel;
    CK(ensure(ctx->kt, (size_t)N * 4));
    CK(ensure(ctx->mm_t, 2 * 4));
    CK(ensure(ctx->est_hist, 2 * 4097 * 4));  // histogram + its cumulative form
    CK(ensure(ctx->est_cost, (size_t)R * 8));
    CK(cudaEventRecord(ctx->ev_split[0], s));
    launch_split_estimate(E, Rel, N, R, d, norm, eps, P<float>(ctx->kt), P<unsigned>(ctx->mm_t),
                          P<unsigned>(ctx->est_hist), P<unsigned long long>(ctx->est_cost), s);
    LAUNCHED(5);
    std::vector<unsigned long long> cnt((size_t)R);
    CK(cudaMemcpyAsync(cnt.data(), ctx->est_cost.p, (size_t)R * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(ctx->ev_split[1], s));
    CK(cudaStreamSynchronize(s));
    // estimated surviving work per relation: sampled in-range tail counts scaled to N queries
    // (+1: never a zero-cost relation); integer inputs, so identical on every rank
    std::vector<double> cost((size_t)R);
    for (long long r = 0; r < R; ++r) cost[(size_t)r] = (double)cnt[(size_t)r] * (double)N / EST_SAMPLES + 1.0;
    double total = 0.0;
    for (double c : cost) total += c;
    const int W = ctx->opt.world, k = ctx->opt.rank;
    // first query tile whose cumulative cost before it reaches t: relation-granular scan,
    // then uniform within the relation
    auto first_at = [&](double t) -> long long {
        double acc = 0.0;
        for (long long r = 0; r < R; ++r) {
            const double c = cost[(size_t)r];
            if (acc + c > t) {
                long long qt = (long long)std::ceil((t - acc) / c * (double)QT);
                if (qt < 0) qt = 0;
                if (qt > QT) qt = QT;
                return r * QT + qt;
            }
            acc += c;
        }
        return R * QT;
    };
    *a = k == 0 ? 0 : first_at(total * k / W);
    *b = k == W - 1 ? R * QT : first_at(total * (k + 1) / W);
    return KGC_OK;
}

// ------------------------------------------------------------ relation batches
// Results of several join_impl calls (relation batches, SE relations) are appended to
// ctx->acc; acc_finish makes the accumulated list the context's results.
static int acc_append(kgc_ctx* ctx, long long* total) {
    const long long n = ctx->n_results;
    if (n <= 0) return KGC_OK;
    cudaStream_t s = ctx->stream;
    const size_t need = (size_t)(*total + n) * 16;
    if (need > ctx->acc.n) {
        DevBuf nb;
        CK(ensure(nb, std::max<size_t>(need + need / 2, (size_t)1 << 20)));
        if (*total) CK(cudaMemcpyAsync(nb.p, ctx->acc.p, (size_t)*total * 16, cudaMemcpyDeviceToDevice, s));
        CK(cudaStreamSynchronize(s));
        if (ctx->acc.p) cudaFree(ctx->acc.p);
        ctx->acc = nb;
    }
    CK(cudaMemcpyAsync(P<char>(ctx->acc) + (size_t)*total * 16, ctx->res.p, (size_t)n * 16, cudaMemcpyDeviceToDevice,
                       s));
    *total += n;
    return KGC_OK;
}
static int acc_finish(kgc_ctx* ctx, long long total) {
    CK(cudaStreamSynchronize(ctx->stream));
    std::swap(ctx->res, ctx->acc);  // the accumulated results become the context's results
    ctx->res_cap = (long long)(ctx->res.n / 16);
    ctx->n_results = total;
    return KGC_OK;
}
// Sum of the per-call statistics of a multi-call join (geometry from the last call).
static void acc_stats(kgc_stats_t& a, const kgc_stats_t& st) {
    a.tile_pairs_total += st.tile_pairs_total;
    a.tile_pairs_surviving += st.tile_pairs_surviving;
    a.tile_pairs_mine += st.tile_pairs_mine;
    a.work_items_mine += st.work_items_mine;
    a.candidates += st.candidates;
    a.results += st.results;
    a.h2d_bytes += st.h2d_bytes;
    a.launches += st.launches;
    a.reruns += st.reruns;
    a.gathered_pairs += st.gathered_pairs;
    a.ms_h2d += st.ms_h2d;
    a.ms_keys += st.ms_keys;
    a.ms_sort += st.ms_sort;
    a.ms_ranges += st.ms_ranges;
    a.ms_stage += st.ms_stage;
    a.ms_tiles += st.ms_tiles;
    a.ms_recheck += st.ms_recheck;
    a.ms_total += st.ms_total;
    a.query_tile_rows = st.query_tile_rows;
    a.tail_tile_rows = st.tail_tile_rows;
    a.query_tiles = st.query_tiles;
    a.tail_tiles = st.tail_tiles;
    a.pivots_used = st.pivots_used;
    a.engine = st.engine;
}

// Relations per join_impl call.  Row ids (relation x sorted query position) are 32-bit in
// the candidate records and several kernels, and the per-call buffers grow with N x R
// (keys, sort scratch, permutations), so a join over more than 2^28 query rows (the
// paper's motivating 10^6 entities x 1000 relations, is 10^9) runs as
// consecutive relation batches of at most 2^28 rows each; results are appended.  Every
// batch is a complete join of its relations (Definition 1 is per triplet), so the union is
// the join.  kgc_options.relation_batch overrides the size (tests).
static long long relation_batch(const kgc_ctx* ctx, long long N) {
    if (ctx->opt.relation_batch > 0) return ctx->opt.relation_batch;
    const long long rb = (1LL << 28) / std::max<long long>(N, 1);
    return std::max<long long>(rb, 1);
}

// The join of relations [r_lo, r_hi).  Query tiles [a, b) in the global numbering r * QT + q
// (a >= 0), or the modes of join_impl: a = b = -1 (cost-balanced shard of everything), -2
// (cyclic), or a = 0, b = LLONG_MAX (every query tile: tail partitions).
static int join_relations(kgc_ctx* ctx, const float* E, const float* Rel, long long N, long long R, int d, int norm,
                          float eps, long long r_lo, long long r_hi, long long a, long long b, long long QT,
                          const JoinExtra& ex) {
    const long long rb = relation_batch(ctx, N);
    auto local = [&](long long r1, long long r2, long long* la, long long* lb) {
        if (a < 0 || b == LLONG_MAX) {
            *la = a;
            *lb = b;
            return true;
        }
        *la = std::max(a, r1 * QT) - r1 * QT;
        *lb = std::min(b, r2 * QT) - r1 * QT;
        return *la < *lb;
    };
    if (r_hi - r_lo <= rb) {
        long long la = 0, lb = 0;
        local(r_lo, r_hi, &la, &lb);
        return join_impl(ctx, E, Rel + r_lo * d, N, r_hi - r_lo, d, norm, eps, (int)r_lo, la, lb, R, ex);
    }
    cudaStream_t s = ctx->stream;
    // stage host inputs once (join_impl would copy them per batch)
    const float* Ed = E;
    const float* Rd = Rel;
    int64_t h2d = 0;
    if (!is_device_ptr(E, ctx->device)) {
        CK(ensure(ctx->E, (size_t)N * d * 4));
        CK(cudaMemcpyAsync(ctx->E.p, E, (size_t)N * d * 4, cudaMemcpyDefault, s));
        Ed = P<float>(ctx->E);
        h2d += (int64_t)N * d * 4;
    }
    if (!is_device_ptr(Rel, ctx->device)) {
        CK(ensure(ctx->Rel, (size_t)R * d * 4));
        CK(cudaMemcpyAsync(ctx->Rel.p, Rel, (size_t)R * d * 4, cudaMemcpyDefault, s));
        Rd = P<float>(ctx->Rel);
        h2d += (int64_t)R * d * 4;
    }
    kgc_stats_t acc{};
    long long total = 0;
    for (long long r1 = r_lo; r1 < r_hi; r1 += rb) {
        const long long r2 = std::min(r_hi, r1 + rb);
        long long la = 0, lb = 0;
        if (!local(r1, r2, &la, &lb)) continue;
        const int rc = join_impl(ctx, Ed, Rd + r1 * d, N, r2 - r1, d, norm, eps, (int)r1, la, lb, R, ex);
        if (rc != KGC_OK) return rc;
        acc_stats(acc, ctx->st);
        const int rc2 = acc_append(ctx, &total);
        if (rc2 != KGC_OK) return rc2;
    }
    const int rc = acc_finish(ctx, total);
    if (rc != KGC_OK) return rc;
    acc.N = N;
    acc.R = R;
    acc.d = d;
    acc.norm = norm;
    acc.eps = eps;
    acc.rank = ctx->opt.rank;
    acc.world = ctx->opt.world;
    acc.triplets = (double)N * (double)N * (double)R;
    acc.h2d_bytes += h2d;
    acc.results = total;
    ctx->st = acc;
    ctx->have_join = true;
    return KGC_OK;
}

// Spatial block-cyclic head split (split = 3, split.cu): every rank orders the heads along the
// same space-filling curve, cuts the order into W * m chunks and keeps chunks k, k + W, ...;
// their rows are gathered into sp_Eh and their global ids into sp_hidx (the records' h).
constexpr long long SP_CHUNK = 4096;  // target heads per chunk (c5 emulated W = 8: 1024 -> 0.79,
                                      // 4096 -> 0.84-0.87, 8192 -> 0.87-0.88 but c4 2.90 -> 2.98 ms,
                                      // 16384 -> 0.80 of linear)
static int spatial_heads(kgc_ctx* ctx, const float* E, long long N, int d, long long* nh_out, cudaStream_t s) {
    const long long W = ctx->opt.world, k = ctx->opt.rank;
    *nh_out = 0;
    CK(ensure(ctx->pivot, (size_t)d * 8));  // first curve pivot: the row farthest from the origin
    CK(cudaMemsetAsync(ctx->pivot.p, 0, (size_t)d * 8, s));
    CK(ensure(ctx->sp_P, (size_t)4 * d * 4));
    launch_pick_pivots(E, N, d, 2, 4, P<double>(ctx->pivot), P<float>(ctx->sp_P), s);
    CK(ensure(ctx->sp_keys, (size_t)N * 16));
    CK(ensure(ctx->sp_mm, 32));
    CK(ensure(ctx->sp_c0, (size_t)N * 4));
    CK(ensure(ctx->sp_v0, (size_t)N * 4));
    CK(ensure(ctx->sp_c1, (size_t)N * 4));
    CK(ensure(ctx->sp_v1, (size_t)N * 4));
    launch_sp_order(E, N, d, P<float>(ctx->sp_P), P<float>(ctx->sp_keys), P<unsigned>(ctx->sp_mm),
                    P<unsigned>(ctx->sp_c0), P<unsigned>(ctx->sp_v0), s);
    const size_t nc = std::max<size_t>(radix_counts_len(1, N), 1);
    CK(ensure(ctx->counts, nc * 4));
    CK(ensure(ctx->scan_tmp, scan_tmp_bytes(nc)));
    radix_sort_u32_segments(1, N, 32, P<unsigned>(ctx->sp_c0), P<unsigned>(ctx->sp_v0), P<unsigned>(ctx->sp_c1),
                            P<unsigned>(ctx->sp_v1), P<int>(ctx->counts), ctx->scan_tmp.p, s, &ctx->launches);
    LAUNCHED(5);
    // the chunks of this rank (kgc_spatial_chunks: the same rule on the host, tested on the CPU)
    const long long owned = kgc_spatial_chunks(N, (int32_t)W, (int32_t)k, SP_CHUNK, nullptr, nullptr, 0);
    std::vector<int64_t> cb((size_t)std::max(owned, 1LL)), cl((size_t)std::max(owned, 1LL));
    kgc_spatial_chunks(N, (int32_t)W, (int32_t)k, SP_CHUNK, cb.data(), cl.data(), owned);
    long long dst = 0, max_len = 0;
    for (long long i = 0; i < owned; ++i) {
        dst += cl[(size_t)i];
        max_len = std::max<long long>(max_len, cl[(size_t)i]);
    }
    const long long nch = sp_nchunks(N, W, SP_CHUNK);
    *nh_out = dst;
    if (dst == 0) return KGC_OK;
    CK(ensure(ctx->sp_hidx, (size_t)dst * 4));
    CK(ensure(ctx->sp_Eh, (size_t)dst * d * 4));
    launch_sp_gather(E, d, P<unsigned>(ctx->sp_v0), N, nch, W, k, owned, max_len, P<int>(ctx->sp_hidx),
                     P<float>(ctx->sp_Eh), s);
    LAUNCHED(1);
    return KGC_OK;
}

// split = 3: this rank's heads (chunks of a space-filling curve) against all N tails; records
// carry the global head ids.
static int join_spatial(kgc_ctx* ctx, const float* E, const float* Rel, long long N, long long R, int d, int norm,
                        float eps) {
    cudaStream_t s = ctx->stream;
    CK(cudaEventRecord(ctx->ev_split[0], s));
    const float* Ed = E;
    long long h2d = 0;
    if (!is_device_ptr(E, ctx->device)) {
        CK(ensure(ctx->E, (size_t)N * d * 4));
        CK(cudaMemcpyAsync(ctx->E.p, E, (size_t)N * d * 4, cudaMemcpyDefault, s));
        Ed = P<float>(ctx->E);
        h2d = N * d * 4;
    }
    // The join's own pivot choice (one CTA, tails only) on the stream, the head order (every other
    // SM) on the aux stream beside it; the join waits for both.
    const int K = (ctx->opt.pivots >= 2 && ctx->opt.prune && d <= MP_MAX_DIM) ? ctx->opt.pivots : 1;
    const bool pre = K > 1 && ctx->opt.pivot == 0 && !(norm == 1 && K > MP_MAX_L1);
    CK(cudaEventRecord(ctx->ev_sp[0], s));  // inputs ready (before the pivot choice: the two overlap)
    CK(cudaStreamWaitEvent(ctx->aux, ctx->ev_sp[0], 0));
    if (pre) {
        CK(ensure(ctx->mpP, (size_t)K * d * 4));
        launch_pick_pivots(Ed, N, d, norm, K, nullptr, P<float>(ctx->mpP), s);
        LAUNCHED(1);
    }
    long long nh = 0;
    int rc = spatial_heads(ctx, Ed, N, d, &nh, ctx->aux);
    if (rc != KGC_OK) return rc;
    CK(cudaEventRecord(ctx->ev_split[1], ctx->aux));
    CK(cudaEventRecord(ctx->ev_sp[1], ctx->aux));
    CK(cudaStreamWaitEvent(s, ctx->ev_sp[1], 0));
    ctx->pivots_ready = pre;
    if (nh == 0) {
        ctx->pivots_ready = false;
        memset(&ctx->st, 0, sizeof ctx->st);
        ctx->st.R = R; ctx->st.d = d; ctx->st.norm = norm; ctx->st.eps = eps;
    } else {
        JoinExtra ex;
        ex.Et = Ed;
        ex.Nt = N;
        ex.hmap = P<int>(ctx->sp_hidx);
        // all of this rank's query tiles: the fixed range [0, inf), no further sharding
        rc = join_relations(ctx, P<float>(ctx->sp_Eh), Rel, nh, R, d, norm, eps, 0, R, 0, LLONG_MAX, 0, ex);
        ctx->pivots_ready = false;
        if (rc != KGC_OK) return rc;
    }
    ctx->st.N = N;
    ctx->st.triplets = (double)N * (double)N * (double)R;
    ctx->st.rank = ctx->opt.rank;
    ctx->st.world = ctx->opt.world;
    ctx->st.h2d_bytes += h2d;
    if (nh == 0) {
        ctx->n_results = 0;
        ctx->have_join = true;
    }
    return KGC_OK;
}

extern "C" int kgc_join(kgc_ctx* ctx, const float* E, const float* Rel, int64_t N, int64_t R, int32_t d, int32_t norm,
                        float eps) {
    if (!ctx) return KGC_EINVAL;
    ctx->err.clear();
    ctx->n_results = -1;
    ctx->have_join = false;
    if (N < 0 || R < 0 || d < 1 || d > KGC_MAX_DIM || (norm != 1 && norm != 2) || !(eps >= 0.f) ||
        !std::isfinite(eps)) {
        set_err(ctx, "kgc_join: invalid argument (N=%lld R=%lld d=%d norm=%d eps=%g)", (long long)N, (long long)R, d,
                norm, (double)eps);
        return KGC_EINVAL;
    }
    if (N > INT_MAX / 4 || R > INT_MAX) {  // entity / relation ids are int32 in the records
        set_err(ctx, "kgc_join: N > 2^29 or R > 2^31 - 1 (32-bit entity / relation ids)");
        return KGC_EINVAL;
    }
    if (N == 0 || R == 0) {
        memset(&ctx->st, 0, sizeof ctx->st);
        ctx->st.N = N;
        ctx->st.R = R;
        ctx->st.d = d;
        ctx->st.norm = norm;
        ctx->st.eps = eps;
        ctx->st.rank = ctx->opt.rank;
        ctx->st.world = ctx->opt.world;
        ctx->n_results = 0;
        ctx->have_join = true;
        return KGC_OK;
    }
    if (!E || !Rel) {
        set_err(ctx, "kgc_join: NULL E or Rel");
        return KGC_EINVAL;
    }
    const auto host_t0 = std::chrono::steady_clock::now();
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    int rc = KGC_OK;
    bool did_split = false;
    if (ctx->opt.world > 1 && ctx->opt.tail_shard) {
        // Partition-based join (§4.7): this rank's tail partition against every
        // query (all query tiles owned: the fixed range [0, inf)); results carry global tail ids.
        const long long t0 = N * ctx->opt.rank / ctx->opt.world, t1 = N * (ctx->opt.rank + 1) / ctx->opt.world;
        if (t1 <= t0) {
            memset(&ctx->st, 0, sizeof ctx->st);
            ctx->st.N = N; ctx->st.R = R; ctx->st.d = d; ctx->st.norm = norm; ctx->st.eps = eps;
            ctx->st.rank = ctx->opt.rank; ctx->st.world = ctx->opt.world;
            ctx->st.triplets = (double)N * (double)N * (double)R;
            ctx->n_results = 0;
            ctx->have_join = true;
        } else {
            JoinExtra ex;
            ex.Nt = t1 - t0;
            ex.t_off = t0;
            rc = join_relations(ctx, E, Rel, N, R, d, norm, eps, 0, R, 0, LLONG_MAX, 0, ex);
        }
    } else if (ctx->opt.world > 1 && ctx->opt.split == 0 && !(norm == 2 && ctx->opt.l2_engine == 5)) {
        did_split = true;
        // Rank-local split: query-tile ranges balanced by an estimated per-relation cost
        // (launch_split_estimate); each rank then preprocesses only the relations its range touches.
        const long long bq = plan_bq(ctx, norm, d, N);
        const long long QT = (N + bq - 1) / bq, nq = R * QT;
        long long a = 0, b = 0, h2d = 0;
        const float *Ed = E, *Rd = Rel;
        rc = split_range(ctx, E, Rel, N, R, d, norm, eps, QT, &a, &b, &Ed, &Rd, &h2d);
        if (rc == KGC_OK && a >= b) {
            memset(&ctx->st, 0, sizeof ctx->st);
            ctx->st.N = N; ctx->st.R = R; ctx->st.d = d; ctx->st.norm = norm; ctx->st.eps = eps;
            ctx->st.rank = ctx->opt.rank; ctx->st.world = ctx->opt.world;
            ctx->st.triplets = (double)N * (double)N * (double)R;
            ctx->n_results = 0;
            ctx->have_join = true;
        } else if (rc == KGC_OK) {
            (void)nq;
            const long long r_lo = a / QT, r_hi = (b - 1) / QT + 1;
            rc = join_relations(ctx, Ed, Rd, N, R, d, norm, eps, r_lo, r_hi, a, b, QT, JoinExtra());
            ctx->st.h2d_bytes += h2d;
        }
    } else if (ctx->opt.world > 1 && ctx->opt.split == 3 && !(norm == 2 && ctx->opt.l2_engine == 5)) {
        did_split = true;
        rc = join_spatial(ctx, E, Rel, N, R, d, norm, eps);
    } else if (ctx->opt.world > 1 && ctx->opt.split == 2) {
        // Cyclic split: every rank preprocesses everything and takes query tiles q with
        // q % world == rank, so hit-dense relations spread over all ranks.
        rc = join_relations(ctx, E, Rel, N, R, d, norm, eps, 0, R, -2, -2, 0, JoinExtra());
    } else {
        rc = join_relations(ctx, E, Rel, N, R, d, norm, eps, 0, R, -1, -1, 0, JoinExtra());
    }
    if (rc != KGC_OK) {
        cudaStreamSynchronize(ctx->stream);
        cudaGetLastError();
    } else {
        ctx->st.ms_split = 0.f;
        if (did_split) cudaEventElapsedTime(&ctx->st.ms_split, ctx->ev_split[0], ctx->ev_split[1]);
        ctx->st.ms_host = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
    }
    cudaSetDevice(prev);
    return rc;
}

// ------------------------------------------------------------------ head block x tail block
// One block of the partition-based join (§4.7): the queries of a head
// block against one tail block, ids offset to the global numbering.  The ring that walks
// every tail block past every head block runs over the caller's process group
// (kgc.partition_join); this call is the per-GPU step of it.
extern "C" int kgc_join_block(kgc_ctx* ctx, const float* Eh, int64_t Nh, int64_t h_off, const float* Et, int64_t Nt,
                              int64_t t_off, const float* Rel, int64_t R, int32_t d, int32_t norm, float eps) {
    if (!ctx) return KGC_EINVAL;
    ctx->err.clear();
    ctx->n_results = -1;
    ctx->have_join = false;
    if (Nh < 0 || Nt < 0 || h_off < 0 || t_off < 0 || R < 0 || d < 1 || d > KGC_MAX_DIM || (norm != 1 && norm != 2) ||
        !(eps >= 0.f) || !std::isfinite(eps) || h_off + Nh > INT_MAX || t_off + Nt > INT_MAX || Nh > INT_MAX / 4 ||
        Nt > INT_MAX / 4 || R > INT_MAX) {
        set_err(ctx, "kgc_join_block: invalid argument (Nh=%lld h_off=%lld Nt=%lld t_off=%lld R=%lld d=%d norm=%d "
                "eps=%g)", (long long)Nh, (long long)h_off, (long long)Nt, (long long)t_off, (long long)R, d, norm,
                (double)eps);
        return KGC_EINVAL;
    }
    if (ctx->opt.world != 1 || ctx->opt.tail_shard) {
        set_err(ctx, "kgc_join_block: needs a single-shard context (world = 1); the caller orders the blocks");
        return KGC_EINVAL;
    }
    if (Nh == 0 || Nt == 0 || R == 0) {
        memset(&ctx->st, 0, sizeof ctx->st);
        ctx->st.N = Nh;
        ctx->st.R = R;
        ctx->st.d = d;
        ctx->st.norm = norm;
        ctx->st.eps = eps;
        ctx->st.world = 1;
        ctx->n_results = 0;
        ctx->have_join = true;
        return KGC_OK;
    }
    if (!Eh || !Et || !Rel) {
        set_err(ctx, "kgc_join_block: NULL Eh, Et or Rel");
        return KGC_EINVAL;
    }
    const auto host_t0 = std::chrono::steady_clock::now();
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    auto run = [&]() -> int {
        JoinExtra ex;
        ex.Et = Et;
        ex.Nt = Nt;
        ex.t_off = t_off;
        ex.h_off = h_off;
        int64_t h2d = 0;
        if (!is_device_ptr(Et, ctx->device)) {
            CK(ensure(ctx->Eb, (size_t)Nt * d * 4));
            CK(cudaMemcpyAsync(ctx->Eb.p, Et, (size_t)Nt * d * 4, cudaMemcpyDefault, ctx->stream));
            ex.Et = P<float>(ctx->Eb);
            h2d = Nt * d * 4;
        }
        const int rc = join_relations(ctx, Eh, Rel, Nh, R, d, norm, eps, 0, R, -1, -1, 0, ex);
        ctx->st.h2d_bytes += h2d;
        return rc;
    };
    const int rc = run();
    if (rc != KGC_OK) {
        cudaStreamSynchronize(ctx->stream);
        cudaGetLastError();
        ctx->n_results = -1;
        ctx->have_join = false;
    } else {
        ctx->st.triplets = (double)Nh * (double)Nt * (double)R;
        ctx->st.ms_host = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
    }
    cudaSetDevice(prev);
    return rc;
}

// ------------------------------------------------------------------ SE
// Structured Embedding: per relation, the FP64 connectors (se.cu), then the
// L1 join of fl32(W_lhs h) against fl32(W_rhs t) with the filters widened by the rounding of
// both sides, re-checked from the FP64 connectors; results appended across relations.
extern "C" int kgc_join_se(kgc_ctx* ctx, const float* E, const float* Wl, const float* Wr, int64_t N, int64_t R,
                           int32_t d, float eps) {
    if (!ctx) return KGC_EINVAL;
    ctx->n_results = -1;
    ctx->have_join = false;
    if (N < 0 || R < 0 || d < 1 || d > KGC_MAX_DIM || !(eps >= 0.f) || !std::isfinite(eps)) {
        set_err(ctx, "kgc_join_se: invalid argument (N=%lld R=%lld d=%d eps=%g)", (long long)N, (long long)R, d,
                (double)eps);
        return KGC_EINVAL;
    }
    if (ctx->opt.world != 1) {
        set_err(ctx, "kgc_join_se: needs a single-shard context (world = 1)");
        return KGC_EINVAL;
    }
    if (N == 0 || R == 0) {
        memset(&ctx->st, 0, sizeof ctx->st);
        ctx->st.N = N;
        ctx->st.R = R;
        ctx->st.d = d;
        ctx->st.norm = 1;
        ctx->st.eps = eps;
        ctx->st.world = 1;
        ctx->n_results = 0;
        ctx->have_join = true;
        return KGC_OK;
    }
    if (!E || !Wl || !Wr) {
        set_err(ctx, "kgc_join_se: NULL E, W_lhs or W_rhs");
        return KGC_EINVAL;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    const auto host_t0 = std::chrono::steady_clock::now();
    long long total = 0;
    int64_t h2d = 0;
    auto run = [&]() -> int {
        const float* Ed = E;
        if (!is_device_ptr(E, ctx->device)) {
            CK(ensure(ctx->E, (size_t)N * d * 4));
            CK(cudaMemcpyAsync(ctx->E.p, E, (size_t)N * d * 4, cudaMemcpyDefault, s));
            Ed = P<float>(ctx->E);
            h2d += N * d * 4;
        }
        const size_t wsz = (size_t)R * d * d;
        const float* Wld = Wl;
        const float* Wrd = Wr;
        if (!is_device_ptr(Wl, ctx->device) || !is_device_ptr(Wr, ctx->device)) {
            CK(ensure(ctx->se_w, wsz * 2 * 4));
            CK(cudaMemcpyAsync(ctx->se_w.p, Wl, wsz * 4, cudaMemcpyDefault, s));
            CK(cudaMemcpyAsync(P<float>(ctx->se_w) + wsz, Wr, wsz * 4, cudaMemcpyDefault, s));
            Wld = P<float>(ctx->se_w);
            Wrd = P<float>(ctx->se_w) + wsz;
            h2d += (int64_t)wsz * 8;
        }
        CK(ensure(ctx->se_a64, (size_t)N * d * 8));
        CK(ensure(ctx->se_b64, (size_t)N * d * 8));
        CK(ensure(ctx->se_af, (size_t)N * d * 4));
        CK(ensure(ctx->se_bf, (size_t)N * d * 4));
        CK(ensure(ctx->se_zero, (size_t)d * 4));
        CK(ensure(ctx->se_max, 8));
        CK(cudaMemsetAsync(ctx->se_zero.p, 0, (size_t)d * 4, s));
        kgc_stats_t acc{};
        for (long long r = 0; r < R; ++r) {
            unsigned int mx[2] = {0, 0};
            launch_se_connectors(Ed, Wld + (size_t)r * d * d, Wrd + (size_t)r * d * d, N, d, P<double>(ctx->se_a64),
                                 P<double>(ctx->se_b64), P<float>(ctx->se_af), P<float>(ctx->se_bf),
                                 P<unsigned>(ctx->se_max), P<unsigned>(ctx->se_max) + 1, s);
            CK(cudaMemcpyAsync(mx, ctx->se_max.p, 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            // |dist(fl a, fl b) - dist(a, b)| <= ||fl a - a||_1 + ||fl b - b||_1 <= 2^-24 (max||a||_1 + max||b||_1)
            const double widen = 5.9604644775390625e-08 * ((double)__uint_as_float_host(mx[0]) +
                                                           (double)__uint_as_float_host(mx[1])) * (1.0 + 1e-6);
            const float feps = nextafterf((float)((double)eps + widen), FLT_MAX);
            if (!std::isfinite(feps)) {
                set_err(ctx, "kgc_join_se: non-finite value in E, W_lhs or W_rhs (or connector values overflow float)");
                return KGC_EDATA;
            }
            JoinExtra ex;
            ex.Et = P<float>(ctx->se_bf);
            ex.filt_eps = feps;
            ex.A64 = P<double>(ctx->se_a64);
            ex.B64 = P<double>(ctx->se_b64);
            const int rc = join_impl(ctx, P<float>(ctx->se_af), P<float>(ctx->se_zero), N, 1, d, 1, eps, (int)r, -1, -1,
                                     1, ex);
            if (rc != KGC_OK) return rc;
            acc_stats(acc, ctx->st);
            acc.launches += 5;
            const int rc2 = acc_append(ctx, &total);
            if (rc2 != KGC_OK) return rc2;
        }
        const int rc = acc_finish(ctx, total);
        if (rc != KGC_OK) return rc;
        acc.query_tiles *= R;
        acc.tail_tiles *= R;
        acc.N = N;
        acc.R = R;
        acc.d = d;
        acc.norm = 1;
        acc.eps = eps;
        acc.rank = 0;
        acc.world = 1;
        acc.triplets = (double)N * (double)N * (double)R;
        acc.results = total;
        acc.h2d_bytes = h2d;
        ctx->st = acc;
        return KGC_OK;
    };
    const int rc = run();
    if (rc != KGC_OK) {
        cudaStreamSynchronize(s);
        cudaGetLastError();
        ctx->n_results = -1;
    } else {
        ctx->n_results = total;
        ctx->have_join = true;
        ctx->st.ms_host = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
    }
    cudaSetDevice(prev);
    return rc;
}

// ------------------------------------------------------------------ top-k
// The k smallest dist3 over all triplets (PAPER.md:128's statistic).
// See topk.cu for the three steps; everything but the final order of the <= k + ties
// selected records runs on the device.
namespace {
// smallest float theta >= 0 with count(theta) >= k (count monotone in theta); +inf if none
template <typename F>
int bisect_theta(F count, long long k, float* theta) {
    unsigned lo = 0u, hi = 0x7f7fffffu;  // float bit patterns of 0 and FLT_MAX (non-negative floats are ordered)
    long long c = 0;
    int rc = count(__uint_as_float_host(hi), &c);
    if (rc != KGC_OK) return rc;
    if (c < k) {
        *theta = FLT_MAX;
        return KGC_OK;
    }
    while (lo < hi) {
        const unsigned mid = lo + (hi - lo) / 2;
        rc = count(__uint_as_float_host(mid), &c);
        if (rc != KGC_OK) return rc;
        if (c >= k) hi = mid; else lo = mid + 1;
    }
    *theta = __uint_as_float_host(lo);
    return KGC_OK;
}
}  // namespace

extern "C" int64_t kgc_topk(kgc_ctx* ctx, const float* E, const float* Rel, int64_t N, int64_t R, int32_t d,
                            int32_t norm, int64_t k, int32_t exclude_self, kgc_triplet* out) {
    if (!ctx) return KGC_EINVAL;
    ctx->n_results = -1;
    if (k < 0 || N < 0 || R < 0 || d < 1 || d > KGC_MAX_DIM || (norm != 1 && norm != 2) ||
        (exclude_self != 0 && exclude_self != 1) || (k > 0 && !out)) {
        set_err(ctx, "kgc_topk: invalid arguments (k=%lld N=%lld R=%lld d=%d norm=%d)", (long long)k, (long long)N,
                (long long)R, d, norm);
        return KGC_EINVAL;
    }
    if (ctx->opt.world != 1) {
        set_err(ctx, "kgc_topk: needs a single-shard context (world = 1)");
        return KGC_EINVAL;
    }
    if (k == 0 || N == 0 || R == 0) {
        memset(&ctx->st, 0, sizeof ctx->st);  // no join ran: empty statistics, not the previous join's
        ctx->st.N = N;
        ctx->st.R = R;
        ctx->st.d = d;
        ctx->st.norm = norm;
        ctx->st.world = 1;
        ctx->n_results = 0;
        ctx->have_join = true;
        return 0;
    }
    if (!E || !Rel) {
        set_err(ctx, "kgc_topk: NULL E or Rel");
        return KGC_EINVAL;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    long long result = 0;
    auto run = [&]() -> int {
        const float* Ed = E;
        const float* Rd = Rel;
        if (!is_device_ptr(E, ctx->device)) {
            CK(ensure(ctx->E, (size_t)N * d * 4));
            CK(cudaMemcpyAsync(ctx->E.p, E, (size_t)N * d * 4, cudaMemcpyDefault, s));
            Ed = P<float>(ctx->E);
        }
        if (!is_device_ptr(Rel, ctx->device)) {
            CK(ensure(ctx->Rel, (size_t)R * d * 4));
            CK(cudaMemcpyAsync(ctx->Rel.p, Rel, (size_t)R * d * 4, cudaMemcpyDefault, s));
            Rd = P<float>(ctx->Rel);
        }
        CK(ensure(ctx->tk_cnt, 8));
        unsigned long long* dcnt = P<unsigned long long>(ctx->tk_cnt);
        // 1. sampled rows against every tail -> an upper bound of the k-th smallest distance
        const long long NR = N * R;
        long long S = std::min<long long>(NR, 256);
        CK(ensure(ctx->tk_sample, (size_t)S * N * 4));
        launch_sample_dist(Ed, Rd, N, R, d, norm, (int)S, exclude_self, P<float>(ctx->tk_sample), s);
        auto count_sample = [&](float th, long long* c) -> int {
            unsigned long long h = 0;
            launch_count_le(P<float>(ctx->tk_sample), S * N, th, dcnt, s);
            CK(cudaMemcpyAsync(&h, dcnt, 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            *c = (long long)h;
            return KGC_OK;
        };
        float theta = 0.f;
        int rc = bisect_theta(count_sample, k, &theta);
        if (rc != KGC_OK) return rc;
        // 2. the epsilon-join at theta (>= k triplets, or every triplet when theta = FLT_MAX).
        // The sample bound can be loose by orders of magnitude in result count (the closest
        // triplets come from rare rows), so first try theta * 0.9^j, j = 2, 1 (joins at a
        // smaller theta are cheap: fewer results, more pruning) and stop at the first with
        // >= k usable triplets; theta itself always suffices.
        const KgcTripletDev* res = nullptr;
        long long n = 0;
        auto count_res = [&](float th, long long* c) -> int {
            unsigned long long h = 0;
            launch_count_res_le(res, n, th, exclude_self, dcnt, s);
            CK(cudaMemcpyAsync(&h, dcnt, 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            *c = (long long)h;
            return KGC_OK;
        };
        for (int j = (theta < FLT_MAX ? 2 : 0); j >= 0; --j) {
            const float th = j ? theta * powf(0.9f, (float)j) : theta;
            rc = join_impl(ctx, Ed, Rd, N, R, d, norm, th, 0, -1, -1, R);
            if (rc != KGC_OK) return rc;
            n = ctx->n_results;
            res = reinterpret_cast<const KgcTripletDev*>(ctx->res.p);
            if (j == 0) break;
            long long have = 0;
            rc = count_res(FLT_MAX, &have);
            if (rc != KGC_OK) return rc;
            if (have >= k) break;
        }
        // 3. the k-th smallest returned distance, then the records within it, ordered on the host
        long long avail = 0;
        rc = count_res(FLT_MAX, &avail);
        if (rc != KGC_OK) return rc;
        const long long kk = std::min<long long>(k, avail);
        if (kk == 0) {
            result = 0;
            return KGC_OK;
        }
        float thk = 0.f;
        rc = bisect_theta(count_res, kk, &thk);
        if (rc != KGC_OK) return rc;
        long long m = 0;
        rc = count_res(thk, &m);
        if (rc != KGC_OK) return rc;
        CK(ensure(ctx->tk_sel, (size_t)m * 16));
        launch_compact_res_le(res, n, thk, exclude_self, reinterpret_cast<KgcTripletDev*>(ctx->tk_sel.p), dcnt, m, s);
        std::vector<kgc_triplet> sel((size_t)m);
        CK(cudaMemcpyAsync(sel.data(), ctx->tk_sel.p, (size_t)m * 16, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::sort(sel.begin(), sel.end(), [](const kgc_triplet& a, const kgc_triplet& b) {
            if (a.dist != b.dist) return a.dist < b.dist;
            if (a.h != b.h) return a.h < b.h;
            if (a.r != b.r) return a.r < b.r;
            return a.t < b.t;
        });
        CK(cudaMemcpyAsync(out, sel.data(), (size_t)kk * 16, cudaMemcpyDefault, s));
        CK(cudaStreamSynchronize(s));
        if (!is_device_ptr(out, ctx->device)) ctx->st.d2h_bytes += kk * 16;
        result = kk;
        return KGC_OK;
    };
    const int rc = run();
    if (rc != KGC_OK) {
        cudaStreamSynchronize(s);
        cudaGetLastError();
    }
    cudaSetDevice(prev);
    return rc != KGC_OK ? rc : result;
}

extern "C" int64_t kgc_results(kgc_ctx* ctx, kgc_triplet* out, int64_t capacity) {
    if (!ctx || capacity < 0) return KGC_EINVAL;
    if (ctx->n_results < 0) {
        set_err(ctx, "kgc_results: no successful join");
        return KGC_ESTATE;
    }
    long long n = std::min<long long>(ctx->n_results, capacity);
    if (out && n > 0) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(ctx->device);
        cudaError_t e = cudaMemcpyAsync(out, ctx->res.p, (size_t)n * 16, cudaMemcpyDefault, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        cudaSetDevice(prev);
        if (e != cudaSuccess) {
            set_err(ctx, "kgc_results: copy failed: %s", cudaGetErrorString(e));
            return KGC_ECUDA;
        }
        if (!is_device_ptr(out, ctx->device)) ctx->st.d2h_bytes += n * 16;
    }
    return ctx->n_results;
}

extern "C" int kgc_stats(const kgc_ctx* ctx, kgc_stats_t* out) {
    if (!ctx || !out) return KGC_EINVAL;
    if (!ctx->have_join) return KGC_ESTATE;
    *out = ctx->st;
    return KGC_OK;
}

extern "C" int64_t kgc_inspect(kgc_ctx* ctx, int32_t what, void* out, int64_t bytes) {
    if (!ctx || bytes < 0) return KGC_EINVAL;
    if (!ctx->have_join || ctx->N == 0 || ctx->R == 0) return KGC_ESTATE;
    struct DevGuard {
        int prev = 0;
        explicit DevGuard(int dev) { cudaGetDevice(&prev); cudaSetDevice(dev); }
        ~DevGuard() { cudaSetDevice(prev); }
    } guard(ctx->device);
    const void* src = nullptr;
    int64_t n = 0;
    switch (what) {
        case KGC_INSPECT_TAIL_KEYS: src = ctx->K > 1 ? ctx->mpkt.p : ctx->kt.p; n = ctx->N * 4 * ctx->K; break;
        case KGC_INSPECT_QUERY_KEYS:
            if (ctx->K > 1 && ctx->l2f) {  // L2: materialise the keys the join computed on the fly
                if (ensure(ctx->mpkq, (size_t)ctx->N * ctx->R * ctx->K * 4) != cudaSuccess) return KGC_ECUDA;
                launch_mp_qkeys_all(P<double>(ctx->mpB), P<double>(ctx->mpA), P<double>(ctx->mpC), ctx->N, ctx->R,
                                    ctx->K, P<float>(ctx->mpkq), ctx->stream);
            }
            src = ctx->K > 1 ? ctx->mpkq.p : ctx->kq.p;
            n = ctx->N * ctx->R * 4 * ctx->K;
            break;
        case KGC_INSPECT_TILE_LIST: src = ctx->tile_list.p; n = ctx->list_len * 4; break;
        case KGC_INSPECT_GATHER_LIST: src = ctx->glist.p; n = ctx->glist_len * 4; break;
        case KGC_INSPECT_GATHER_COST: src = ctx->glist_len ? ctx->gblk.p : nullptr; n = src ? ctx->R * (int64_t)ctx->QT * 8 : 0; break;
        case KGC_INSPECT_TAIL_PERM: src = ctx->tperm.p; n = ctx->N * 4; break;
        case KGC_INSPECT_QUERY_PERM: src = ctx->qperm.p; n = ctx->N * ctx->R * 4; break;
        case KGC_INSPECT_TILE_RANGES: src = ctx->ranges.p; n = ctx->R * (int64_t)ctx->QT * 8; break;
        case KGC_INSPECT_QUERY_COST: src = ctx->cum.p; n = ctx->R * (int64_t)ctx->QT * 8; break;
        case KGC_INSPECT_PIVOTS: src = ctx->K > 1 ? ctx->mpP.p : nullptr; n = src ? (int64_t)ctx->K * ctx->d * 4 : 0; break;
        default: return KGC_EINVAL;
    }
    if (out && bytes > 0 && n > 0) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(ctx->device);
        cudaError_t e = cudaMemcpyAsync(out, src, (size_t)std::min(n, bytes), cudaMemcpyDefault, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        cudaSetDevice(prev);
        if (e != cudaSuccess) return KGC_ECUDA;
    }
    return n;
}
