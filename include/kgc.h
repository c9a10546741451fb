/*
 * kgc.h -- C ABI of the B200-native TransE completion join (libkgc.so).
 *
 * What it computes.  Knowledge-graph completion, Definition 1 of arXiv
 * 2307.12059, for TransE:
 *
 *     R(eps) = { (h, r, t) in [0,N) x [0,R) x [0,N) :  || E_h + Rel_r - E_t ||_p <= eps }
 *
 * with p = norm in {1, 2}, L2 the non-squared Euclidean norm, the bound
 * inclusive, self edges (h == t) included, every relation vector independent.
 * ``eps`` is the DISTANCE threshold theta: a caller holding a score threshold
 * s* (score >= s*) passes eps = -s* because dist3 = -score.
 *
 * How: the triple problem is recast as a binary similarity join
 * q = h + r against t; pivot distances and sorting
 * give contiguous surviving tail-tile ranges per query
 * tile by Lemma 1 and Lemma 2, so whole tiles are skipped;
 * surviving tiles are verified on the GPU (tcgen05 TF32 tensor-core filter
 * with a rigorous guard band for L2, FP32 SIMT for L1) and every candidate is
 * re-checked in FP64 before it is emitted ("verify if the
 * results are valid").  The filtering is lossless: the
 * result set is the brute-force set.
 *
 * Conventions for every call:
 *   - int-returning calls return a kgc_status (0 = OK, < 0 = error); the
 *     message of the last error is available from kgc_last_error().
 *   - No call keeps a pointer passed by the caller after it returns.
 *   - A context is not thread-safe: one context per host thread.
 *   - Pointers may be host (pageable or pinned) or device memory of the
 *     context's device; the library detects which with
 *     cudaPointerGetAttributes.
 */
#ifndef KGC_H_
#define KGC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define KGC_ABI_VERSION 3  /* 2: kgc_options.tail_shard, kgc_stats_t.gathered_pairs; 3: kgc_options.relation_batch,
                              kgc_join_block */

/* Opaque context: owns device buffers, the stream, per-join statistics. */
typedef struct kgc_ctx kgc_ctx;

typedef enum {
    KGC_OK = 0,
    KGC_EINVAL = -1,   /* bad argument: NULL pointer, N<0, R<0, d<1 or d>KGC_MAX_DIM, norm not 1/2, eps<0 or non-finite */
    KGC_EDATA = -2,    /* a non-finite value in E or Rel */
    KGC_ENOMEM = -3,   /* device or host allocation failed */
    KGC_ECUDA = -4,    /* CUDA runtime error (message in kgc_last_error) */
    KGC_ENODEV = -5,   /* no CUDA device / not an sm_100 device */
    KGC_ESTATE = -6    /* call out of order (e.g. kgc_results before any successful kgc_join) */
} kgc_status;

#define KGC_MAX_DIM 1024

/* One result record, 16 bytes.  dist is the non-squared L_p distance
 * computed in FP64 and rounded to float. */
typedef struct {
    int32_t h, r, t;
    float dist;
} kgc_triplet;

/* Options for kgc_create.  Fill with kgc_default_options() first. */
typedef struct {
    int32_t device;           /* CUDA device ordinal; -1 = the current device                      */
    int32_t rank, world;      /* this context computes shard `rank` of `world` of the work list     */
                              /* (query tiles split by predicted cost; results stay sharded)       */
    int32_t prune;            /* 1 = Lemma 1/2 tile pruning (default); 0 = every tile (naive control,*/
                              /*     PAPER.md:473 "naive GPU approach")                            */
    int32_t pivot;            /* 0 = zero vector (default); 1 = mean of the tails      */
    int32_t l2_engine;        /* 0 = auto (3 when N * pad8(d) * 4 > 48 MiB, else 1; 2 if d > 256);  */
                              /* 1 = tcgen05 TF32 filter; 2 = FP32 SIMT filter; 3 = tcgen05 TF32 on */
                              /* CTA pairs (cta_group::2, 256-row query tiles); 4 = tcgen05 TF32 */
                              /* on gathered tail blocks (needs pivots >= 2: per 128-row query tile */
                              /* only the tails whose own K keys pass the test against the tile's   */
                              /* key box, 256 per block; falls back to 1 when the lists would      */
                              /* exceed 8 GiB); 5 = relation-factored tcgen05 TF32 (no pruning: one */
                              /* G = H T^T tile per (head tile, tail tile) serves all R relations   */
                              /* in the epilogue; for data where tiles do not prune)                */
                              /* 6 = CTA pairs (as 3) on gathered tail blocks when pivots >= 2:    */
                              /* per 256-row query tile the tails passing the per-tail K-pivot     */
                              /* test, 256 per block, each CTA gathering its 128 rows with cp.async */
    int32_t chunk_tiles;      /* max tail tiles per work item (load-balance granularity); 0 = auto */
    int32_t pivots;           /* 0/1 = one pivot (default); 2..8, 12, 16, 24, 32, 48, */
                              /* 64, 96 or 128 = multi-pivot tile pruning (L_inf over K pivot       */
                              /* distances; needs d <= 256, prune = 1; otherwise one  */
                              /* pivot is used); other values: KGC_EINVAL at kgc_create; more than  */
                              /* 32 with norm 1: KGC_EINVAL at the join (the L1 keys support 32).   */
                              /* The per-tail test of the gathered engines uses the first 8 pivots  */
    int64_t result_capacity;  /* initial result-buffer capacity in triplets; 0 = auto (grows)       */
    void*   stream;           /* cudaStream_t to run on; NULL = a stream the context creates       */
    int32_t l1_engine;        /* 0 = auto (3 with multi-pivot pruning, else 2); 1 = FP16x2 SIMT    */
                              /* filter with rigorous band (only when every |E|, |Rel| <= 1000);    */
                              /* 2 = FP32 SIMT on 64 x 64 tiles; 3 = FP32 SIMT on gathered tails:   */
                              /* inside each surviving tile pair only the tails whose own K pivot   */
                              /* keys pass the test against the query tile's box (needs pivots >= 2; */
                              /* also used for the L2 SIMT engine when set explicitly)              */
    int32_t split;            /* world > 1: 0 = rank-local (default: rank k takes query tiles       */
                              /* [k nq/W, (k+1) nq/W) and preprocesses only the relations they      */
                              /* touch; tails are replicated); 1 = global cost-balanced split (every */
                              /* rank preprocesses everything, shards by surviving-tile counts);   */
                              /* 2 = cyclic (every rank preprocesses everything and takes query    */
                              /* tiles q with q % world == rank: hit-dense relations spread out);   */
                              /* 3 = spatial block-cyclic head split (split.cu): every rank orders */
                              /* the heads along the same space-filling curve (Morton order of the */
                              /* distances to 4 pivots), cuts it into W*m chunks of ~4096 heads    */
                              /* (m >= 2) and joins the heads of chunks k, k+W, ... for every       */
                              /* relation against all N tails; no cost estimate, compact query     */
                              /* tiles, every rank a stratified sample of the space.  Records carry */
                              /* global ids; stats.N and triplets are those of the whole join       */
    int32_t tail_shard;       /* world > 1: 1 = partition-based join (§4.7): rank */
                              /* k holds only tails [k N/W, (k+1) N/W) and joins every query       */
                              /* against them (split is ignored); 0 = tails replicated (default)   */
    int32_t relation_batch;   /* relations per internal join pass; 0 = auto (as many as keep N x     */
                              /* batch <= 2^28 query rows).  A join over more relations runs as    */
                              /* consecutive batches whose results are appended (each batch is a   */
                              /* complete join of its relations, so the union is R(eps)); this is   */
                              /* what lifts N x R beyond 32-bit row ids (10^6 x 1000) */
} kgc_options;

/* Per-join statistics (of the last successful kgc_join). */
typedef struct {
    int64_t N, R;
    int32_t d, norm;
    float eps;
    int32_t rank, world;
    double triplets;              /* N*N*R candidate triplets (PAPER.md:460 counts 14951^2 x 2690) */
    int64_t query_tile_rows;      /* rows per query tile (128 tensor cores / FP16x2, 64 FP32 SIMT) */
    int64_t tail_tile_rows;       /* rows per tail tile (256 tensor cores, 128 FP16x2, 64 FP32 SIMT) */
    int64_t query_tiles;          /* per relation                                                  */
    int64_t tail_tiles;
    int64_t tile_pairs_total;     /* R * query_tiles * tail_tiles                                  */
    int64_t tile_pairs_surviving; /* after Lemma 1/2 pruning, all shards                           */
    int64_t tile_pairs_mine;      /* processed by this context's shard                             */
    int64_t work_items_mine;
    int64_t candidates;           /* pairs that passed the GPU filter (this shard)                 */
    int64_t results;              /* triplets emitted (this shard)                                 */
    int64_t h2d_bytes, d2h_bytes; /* host<->device bytes moved inside kgc_join                     */
    int32_t launches;             /* kernels launched by the last kgc_join                         */
    int32_t reruns;               /* capacity-overflow reruns                                      */
    /* device time per phase (CUDA events on the context's stream), milliseconds */
    float ms_total, ms_h2d, ms_keys, ms_sort, ms_ranges, ms_stage, ms_tiles, ms_recheck;
    int32_t pivots_used;          /* 1, or K of the multi-pivot pruning                            */
    int32_t engine;               /* tile engine used: 1 tcgen05 TF32, 2 FP32 SIMT, 3 FP16x2 SIMT,   */
                                  /* 4 tcgen05 TF32 on CTA pairs, 5 FP32 SIMT on gathered tails,      */
                                  /* 6 tcgen05 TF32 on gathered tail blocks, 7 relation-factored,     */
                                  /* 8 tcgen05 TF32 on CTA pairs over gathered tail blocks            */
    float ms_split;               /* device time of the rank-local split estimate (world > 1)       */
    float ms_host;                /* host wall time of the whole kgc_join call                      */
    int64_t gathered_pairs;       /* engine 5: (query row, tail) pairs left after the per-tail K-pivot */
                                  /* test inside surviving tiles (sentinel padding excluded)          */
} kgc_stats_t;

/* Fill *opt with defaults: device -1, rank 0, world 1, prune 1, pivot 0,
 * l2_engine 0, chunk_tiles 0, pivots 1, result_capacity 0, stream NULL,
 * l1_engine 0, split 0, tail_shard 0, relation_batch 0. */
void kgc_default_options(kgc_options* opt);

/* Create a context.  opt == NULL means defaults.  Returns KGC_ENODEV when no
 * sm_100 device is present.  *out is set to NULL on error. */
int kgc_create(kgc_ctx** out, const kgc_options* opt);

/* Run the join R(eps) above.
 *   E   : N x d float32, row-major, contiguous (entity embeddings)
 *   Rel : R x d float32, row-major, contiguous (relation embeddings)
 *   norm: 1 or 2; eps: distance threshold >= 0, finite.
 * N == 0 or R == 0 is valid and yields 0 results (E / Rel may then be NULL).
 * Limits: N < 2^29 and R < 2^31 (int32 ids in kgc_triplet); larger N x R than
 * 2^28 query rows runs in relation batches (kgc_options.relation_batch), bounded
 * only by device memory.  Otherwise KGC_EINVAL.
 * Stream order: every device operation runs on the context's stream (opt.stream /
 * kgc_set_stream, else a non-blocking stream of the context).  Device-memory E /
 * Rel must therefore be complete before the call, or be produced on the stream the
 * context runs on (pass the producer's stream with kgc_set_stream).
 * Blocks until the result count is known.  On error the previous results are
 * dropped and the context stays usable. */
int kgc_join(kgc_ctx* ctx, const float* E, const float* Rel, int64_t N, int64_t R, int32_t d,
             int32_t norm, float eps);

/* Copy min(count, capacity) result records of the last join into `out`
 * (host or device memory, caller-owned) and return the total count (>= 0),
 * or a negative kgc_status.  out may be NULL to query the count.  Record
 * order is unspecified (each triplet appears exactly once). */
int64_t kgc_results(kgc_ctx* ctx, kgc_triplet* out, int64_t capacity);

/* Statistics of the last successful join. */
int kgc_stats(const kgc_ctx* ctx, kgc_stats_t* out);

/* Message of the last error on this context ("" if none).  Owned by the
 * context; valid until the next call on it.  ctx == NULL gives the last
 * kgc_create error. */
const char* kgc_last_error(const kgc_ctx* ctx);

/* Use `stream` (a cudaStream_t) for subsequent joins; NULL = the context's own. */
int kgc_set_stream(kgc_ctx* ctx, void* stream);

/* Release every resource of the context.  NULL is a no-op. */
void kgc_destroy(kgc_ctx* ctx);

/* Inspection hooks for tests: copy an intermediate array of the last join to
 * host memory `out` (capacity `bytes`); returns the number of bytes the array
 * has (copies min of the two), or a negative kgc_status.
 *   KGC_INSPECT_TAIL_KEYS   float[N]     d(t, p) per tail, original order (K1)
 *   KGC_INSPECT_QUERY_KEYS  float[R*N]   d(h + r, p), [r][h] (K1)
 *   KGC_INSPECT_TAIL_PERM   int32[N]     sorted position -> tail index (K2)
 *   KGC_INSPECT_QUERY_PERM  int32[R*N]   per relation, sorted position -> head (K2)
 *   KGC_INSPECT_TILE_RANGES int32[R*QT*2] surviving tail-tile range [sb, eb] per query tile (K3)
 *   KGC_INSPECT_QUERY_COST  int64[R*QT]  exclusive prefix of surviving tiles per query tile (K3)
 *   KGC_INSPECT_TILE_LIST   int32[mine]  multi-pivot: this shard's surviving tail tiles, query tile by
 *                                        query tile (offset of tile q = cost prefix[q] - prefix[first])
 *   KGC_INSPECT_GATHER_LIST int32[64*mine] engine 5: per query tile q of this shard, its surviving sorted
 *                                        tail positions in ascending order, padded with N to whole blocks
 *                                        of 64, at offset 64 * (cost prefix[q] - prefix[first]) (the
 *                                        tile list's offsets; entries past q's blocks are unused)
 *   KGC_INSPECT_GATHER_COST int64[R*QT]  engine 5: 64-tail blocks per query tile (0 outside this shard)
 *   KGC_INSPECT_PIVOTS      float[K*d]   multi-pivot: the K pivots p_k, row-major (0 bytes with one pivot)
 * With multi-pivot pruning (pivots_used = K > 1) the key arrays hold K floats
 * per row: TAIL_KEYS float[N][K], QUERY_KEYS float[R][N][K]. */
enum {
    KGC_INSPECT_TAIL_KEYS = 1,
    KGC_INSPECT_QUERY_KEYS = 2,
    KGC_INSPECT_TAIL_PERM = 3,
    KGC_INSPECT_QUERY_PERM = 4,
    KGC_INSPECT_TILE_RANGES = 5,
    KGC_INSPECT_QUERY_COST = 6,
    KGC_INSPECT_TILE_LIST = 7,
    KGC_INSPECT_GATHER_LIST = 8,
    KGC_INSPECT_GATHER_COST = 9,
    KGC_INSPECT_PIVOTS = 10
};
/* After a join that ran in relation batches the arrays are those of the last batch. */
int64_t kgc_inspect(kgc_ctx* ctx, int32_t what, void* out, int64_t bytes);

/* Pure host function (no device needed), used by split = 1: the shard of
 * query tiles owned by `rank` of `world`, given the exclusive prefix sums
 * `cum` (length n) of the per-query-tile surviving-tile counts and their grand total.  Query tile q
 * belongs to rank min(world-1, floor(world * cum[q] / total)) (total == 0:
 * everything to rank 0).  Writes the half-open range [*begin, *end) and
 * returns its cost (surviving tiles), or KGC_EINVAL.  The device uses the
 * same rule. */
int64_t kgc_shard_range(const int64_t* cum, int64_t n, int64_t total, int32_t rank, int32_t world,
                        int64_t* begin, int64_t* end);

/* Pure host function (no device needed), used by split = 3: the chunks of the
 * space-filling-curve order of N heads that `rank` of `world` joins.  The order
 * is cut into nch = min(N, world * m) equal chunks, m = max(2, round(N / (world *
 * chunk))) (chunk: target heads per chunk; the library uses 4096), chunk c spans
 * sorted positions [c N / nch, (c + 1) N / nch) and belongs to rank c mod world.
 * Writes up to `cap` (begin, len) pairs in chunk order and returns the number of
 * chunks the rank owns (call with cap = 0 to size the arrays), or KGC_EINVAL.
 * Over all ranks the chunks partition [0, N) exactly. */
int64_t kgc_spatial_chunks(int64_t N, int32_t world, int32_t rank, int64_t chunk, int64_t* begin, int64_t* len,
                           int64_t cap);

/* One block of the partition-based join (PAPER.md:419-422 [§4.7]: "divide both
 * datasets into several partitions ... join each pair of partitions"): every
 * (h, r, t) with h in [h_off, h_off + Nh), t in [t_off, t_off + Nt), r in [0, R) and
 * || Eh[h - h_off] + Rel_r - Et[t - t_off] ||_norm <= eps; records carry the global
 * ids h, r, t.  Eh: Nh x d, Et: Nt x d, Rel: R x d, row-major fp32, host or device.
 * The per-GPU step of kgc.partition_join, which keeps one entity block per GPU
 * and passes the tail blocks around a ring of ranks, so that no GPU holds all of
 * E.  Needs world == 1 and tail_shard == 0 (the caller orders the blocks);
 * kgc_stats().triplets = Nh * Nt * R.  Errors as kgc_join (h_off + Nh and
 * t_off + Nt must fit int32). */
int kgc_join_block(kgc_ctx* ctx, const float* Eh, int64_t Nh, int64_t h_off, const float* Et, int64_t Nt,
                   int64_t t_off, const float* Rel, int64_t R, int32_t d, int32_t norm, float eps);

/* Structured Embedding (SE, PAPER.md:193 [§4.3]): every (h, r, t) with
 * dist3 = || W_r^lhs h - W_r^rhs t ||_1 <= eps, i.e. the same join with
 * connector_1(h, r) = W_r^lhs h, connector_2(t, r) = W_r^rhs t, dist = L1 ("SE is
 * also transformable to a metric space").  E: N x d row-major fp32; Wl, Wr: R x d x d
 * row-major fp32 (W_r[k][j] multiplies h_j into component k), host or device.
 * Per relation the connectors are formed in FP64 (the re-check uses them) and
 * rounded once to fp32 for the filters, whose threshold is widened by
 * 2^-24 (max_h ||a_h||_1 + max_t ||b_t||_1) so the filtering stays lossless.
 * Results (h, r, t, dist) via kgc_results, stats via kgc_stats (summed over
 * relations).  Needs world == 1.  Errors as kgc_join. */
int kgc_join_se(kgc_ctx* ctx, const float* E, const float* Wl, const float* Wr, int64_t N, int64_t R, int32_t d,
                float eps);

/* The k smallest distances over all N*R*N triplets, ascending, ties ordered by
 * (h, r, t): the paper's minimum-distance statistic min_{i,j,k} ||h_i + r_j - t_k||
 * (PAPER.md:128 [§2, Table 1], with and without self edges h = t), SURVEY §8(f)
 * row 4.  E, Rel, N, R, d, norm as for kgc_join; k >= 0; exclude_self 0 or 1
 * (1 drops every triplet with h == t).  `out` (host or device memory, k records)
 * receives min(k, available) records; the return value is that count, or a
 * negative kgc_status.  Method: FP64 distances of up to 256 sampled (h, r) rows
 * against every tail give an upper bound theta of the k-th smallest distance (k
 * actual triplets lie within it); epsilon-joins (every §8(a) step) at theta *
 * 0.9^j, j = 2, 1, 0, until one returns >= k triplets (j = 0 always does); the
 * k-th smallest returned distance is found by bisection on the device.  Distances are K6's (FP64, rounded to float).  Afterwards
 * kgc_results / kgc_stats return the epsilon-join that was kept, i.e. the one at
 * theta * 0.9^j for the first j (2, 1, 0) that returned >= k triplets; its
 * threshold is kgc_stats().eps.  k == 0, N == 0 or R == 0 returns 0 with empty
 * statistics.  Needs world == 1 (KGC_EINVAL otherwise). */
int64_t kgc_topk(kgc_ctx* ctx, const float* E, const float* Rel, int64_t N, int64_t R, int32_t d, int32_t norm,
                 int64_t k, int32_t exclude_self, kgc_triplet* out);

/* ABI version compiled into the library (== KGC_ABI_VERSION). */
int kgc_abi_version(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* KGC_H_ */
