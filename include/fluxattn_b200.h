/*
 * fluxattn_b200.h -- C-ABI of the B200-native Fluxion sparse-decode hot path.
 *
 * Plain pointers and sizes only: no CUDA or torch types cross this boundary.
 * Device-memory arguments are marked [dev]; host-memory ones [host].  All
 * kernels run on the context's stream; calls are asynchronous unless stated.
 * Every function returns FX_OK (0) or a negative status; the thread-local
 * message from fx_last_error() then starts with the reference's stable error
 * code ("empty-context: ...", "invalid-granularity: ...", ...).
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   fx_build_metadata(_levels)  <- build_metadata      src/block_index.cpp:10-39
 *   fx_block_scores             <- block_score          src/block_index.cpp:41-53
 *   fx_topk_blocks              <- topk_blocks          src/block_index.cpp:55-83
 *        (batched: fx_decode_step, sel_bits output)
 *   fx_blocks_for_budget        <- blocks_for_budget    src/block_index.cpp:96-103
 *   fx_plan_groups              <- plan_group/volume/budget_at src/selector.cpp:9-46
 *   fx_predict                  <- predict/forward      src/predictor.cpp:161-185
 *   fx_decode_step              <- execute_task         src/scheduler.cpp:78-96
 *        (default_kv_attention attention.cpp:143-151, sparse_attention
 *         block_index.cpp:85-94, merge_into attention.cpp:89-104, fused)
 *   fx_gathered_attention       <- gathered_attention_unchecked attention.cpp:57-87
 *   fx_merge_partials           <- combine_partials/merge_into attention.cpp:89-129
 *   fx_decode_step              <- run(queue, profile, RunMode::Executed)
 *                                  src/scheduler.cpp:283-287 over one decode step
 *                                  of run_decode (src/pipeline.cpp:292-363)
 *   fx_cp_candidates/threshold/select/combine
 *                               <- topk_blocks + merge_into (block_index.cpp:55-83,
 *                                  attention.cpp:89-104) split over context-parallel
 *                                  shards (the 1M-token C5 case; the reference has no
 *                                  multi-device code)
 */
#ifndef FLUXATTN_B200_H
#define FLUXATTN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FX_ABI_VERSION 5

#if defined(__GNUC__)
#define FX_API __attribute__((visibility("default")))
#else
#define FX_API
#endif

/* status codes */
#define FX_OK 0
#define FX_ERR_INVALID (-1)  /* bad argument / shape ("bad-shape", "invalid-granularity", ...) */
#define FX_ERR_CUDA (-2)     /* CUDA runtime failure */
#define FX_ERR_NOMEM (-3)    /* device allocation failed */
#define FX_ERR_STATE (-4)    /* "no-context", "stale-selection", ... */

/* storage types of K/V/metadata */
#define FX_F32 0
#define FX_BF16 1

/* plan modes of fx_decode_step */
#define FX_PLAN_PROPS 0 /* head properties -> on-device plan_group (pipeline.cpp:329) */
#define FX_PLAN_FIXED 1 /* one (blk, bgt) for every head (pipeline.cpp:304-311)      */
#define FX_PLAN_FULL 2  /* blk 128, bgt 1 (pipeline.cpp:298-303)                     */
#define FX_PLAN_GIVEN 3 /* caller-provided [dev] blk per group + budget per head     */

typedef struct fx_ctx fx_ctx;

/* Batched, device-resident KV: K and V are [batch][kv_heads][l_cap][head_dim]
 * in `dtype`, each (b, g) row range in position order
 * sink | cpu | local | new  (kv_cache.hpp:13-18), i.e. rows
 * [0, l_sink) sink, [l_sink, l_sink+l_cpu) cpu, then l_local local rows,
 * then decode-time rows appended at l_sink+l_cpu+l_local+step.
 * Query head h of sequence b belongs to group h / group_size. */
typedef struct fx_layout {
    int32_t batch;
    int32_t kv_heads;
    int32_t group_size;
    int32_t head_dim;
    int32_t dtype;
    int32_t reserved;
    int64_t l_sink;
    int64_t l_cpu;
    int64_t l_local;
    int64_t l_cap;
} fx_layout;

/* Per-step arguments of fx_decode_step.  [dev] unless noted. */
typedef struct fx_step_args {
    const void* k;               /* [B][Hkv][l_cap][D] */
    const void* v;
    const void* meta[4];         /* levels blk 16/32/64/128: [B][Hkv][nblk][2][D] (min row, max row) */
    const float* absmax;         /* [B][Hkv][D] max_row |k_cpu[row][d]| (from fx_build_metadata_levels) */
    int64_t l_new;               /* decode rows already appended */
    const float* q;              /* [B][H][D] f32 */
    int32_t plan_mode;           /* FX_PLAN_* */
    int32_t fixed_block_size;    /* FX_PLAN_FIXED */
    double fixed_budget;         /* FX_PLAN_FIXED */
    const double* bgt0;          /* FX_PLAN_PROPS: [B][H] head properties (budget_oracle.hpp:17-21) */
    const double* kslope;
    const int32_t* streaming;
    int32_t* plan_blk;           /* in (GIVEN) / out: [B][Hkv] chosen granularity, 0 = streaming group */
    double* plan_budgets;        /* in (GIVEN) / out: [B][H] per-head budget */
    double* plan_volume;         /* out, optional: [B][Hkv] V(blk*) (selector.cpp:12) */
    double* plan_cand_volumes;   /* out, optional: [B][Hkv][4] */
    int32_t* plan_kblocks;       /* out, optional: [B][H] blocks_for_budget */
    uint32_t* sel_bits;          /* out, optional: [B][H][sel_words] bit i = block i selected */
    int32_t sel_words;           /* words per head in sel_bits (>= ceil(nblk16/32)) */
    float* o;                    /* out: [B][H][D] f32 attention output (defaults (+) sparse) */
    float* lse;                  /* out, optional: [B][H] natural-log LSE of the merged output */
    /* context-parallel shard (C5); all zero on a single device */
    int64_t l_cpu_total;         /* cpu rows of the WHOLE sequence: plan_group and blocks_for_budget
                                    use it (0 = lay->l_cpu) */
    int64_t cpu_offset;          /* global row of this shard's first cpu row (multiple of 128) */
    const uint32_t* sel_in;      /* given selection [B][H][sel_words] over this shard's blocks at
                                    plan_blk: skips score/select (requires FX_PLAN_GIVEN) */
    /* optional fused append (append_new, kv_cache.hpp:68-73): [B][Hkv][D] f32 rows written
       as decoded row l_new of every (b, g) before this step attends l_new + 1 rows -- the
       previous step's token, saving the separate fx_append_kv launch */
    const float* append_k;
    const float* append_v;
} fx_step_args;

/* ---- context, errors, memory ------------------------------------------ */
FX_API const char* fx_last_error(void);
FX_API int fx_abi_version(void);
FX_API int fx_ctx_create(int device, fx_ctx** out);
FX_API int fx_ctx_destroy(fx_ctx* ctx);
/* Run on an external cudaStream_t (passed as void*); NULL = the legacy default
 * stream.  Until this is called the ctx uses its own non-blocking stream. */
FX_API int fx_ctx_set_stream(fx_ctx* ctx, void* stream);
FX_API void* fx_ctx_stream(fx_ctx* ctx);
/* Waits for the ctx stream, then reports device-detected argument errors of
 * the work since the last call (FX_ERR_INVALID "invalid-granularity: ..." when
 * a FX_PLAN_GIVEN plan held a block size outside {0, 16, 32, 64, 128}; such
 * groups are attended over their resident defaults only, like blk 0). */
FX_API int fx_ctx_synchronize(fx_ctx* ctx);
/* Kernels launched through this context so far. */
FX_API uint64_t fx_ctx_launches(fx_ctx* ctx);

/* Optional CUDA-event timing of each kernel launch on the ctx stream. */
#define FX_KERNEL_PLAN 0     /* K5 prepare/plan          */
#define FX_KERNEL_SCORE 1    /* K2a approximate scores   */
#define FX_KERNEL_SELECT 2   /* K2b exact top-k select   */
#define FX_KERNEL_WORKLIST 3 /* union -> boxes           */
#define FX_KERNEL_ATTEND 4   /* K3+K4 attention          */
#define FX_KERNEL_METADATA 5 /* K1 metadata levels       */
#define FX_KERNEL_APPEND 6   /* decode-row append        */
#define FX_KERNEL_MERGE 7    /* unit-partial merge (TMA) */
#define FX_KERNEL_COUNT 8
FX_API int fx_ctx_set_timing(fx_ctx* ctx, int enable);
/* Accumulated milliseconds and launch count of one kernel id (synchronizes). */
FX_API int fx_ctx_kernel_time(fx_ctx* ctx, int32_t kernel, double* total_ms, int64_t* launches);
FX_API int fx_ctx_reset_timing(fx_ctx* ctx);
FX_API int fx_malloc(fx_ctx* ctx, size_t bytes, void** dptr);
FX_API int fx_free(fx_ctx* ctx, void* dptr);
FX_API int fx_memcpy_h2d(fx_ctx* ctx, void* dst, const void* src, size_t bytes);
FX_API int fx_memcpy_d2h(fx_ctx* ctx, void* dst, const void* src, size_t bytes);
/* device -> device on the ctx stream (asynchronous) */
FX_API int fx_memcpy_d2d(fx_ctx* ctx, void* dst, const void* src, size_t bytes);
FX_API int fx_memset(fx_ctx* ctx, void* dptr, int value, size_t bytes);

/* ---- sizes -------------------------------------------------------------- */
FX_API int64_t fx_block_count(int64_t rows, int32_t block_size);
/* bytes of one metadata level for the whole batch */
FX_API size_t fx_meta_level_bytes(const fx_layout* lay, int32_t block_size);
/* device scratch fx_decode_step needs (allocated lazily inside the ctx), for the
 * ctx's device (its SM count sets the attention grid); ctx NULL = the current device */
FX_API size_t fx_step_scratch_bytes(fx_ctx* ctx, const fx_layout* lay);

/* ---- K1: metadata -------------------------------------------------------- */
/* All four candidate levels of every (b, g) in one streaming pass over the cpu
 * segment, plus absmax[b][g][d] = max_row |k[row][d]| used by the selection
 * error bound.  meta*: [B][Hkv][nblk(blk)][2][D] in lay->dtype. */
FX_API int fx_build_metadata_levels(fx_ctx* ctx, const fx_layout* lay, const void* k, void* meta16,
                             void* meta32, void* meta64, void* meta128, float* absmax);
/* The same pass with per-block MEAN keys as well (north-star item 1: min /
 * max / mean representative keys per block at every candidate granularity;
 * the reference's Quest score uses min / max only, block_index.hpp:16-22):
 * levels[i] as meta16..meta128 above, means[i] [dev] [B][Hkv][nblk(16 << i)][D]
 * f32 = the block's row sum / row count. */
FX_API int fx_build_metadata_means(fx_ctx* ctx, const fx_layout* lay, const void* k, void* const levels[4],
                                   float* absmax, float* const means[4]);
/* One matrix at any granularity >= 1 (the per-head reference API). k: [dev]
 * [rows][dim] in dtype; meta: [dev] [nblk][2][dim] in dtype. */
FX_API int fx_build_metadata(fx_ctx* ctx, const void* k, int32_t dtype, int64_t rows, int32_t dim,
                      int32_t block_size, void* meta);

/* ---- K2: scoring and selection ------------------------------------------- */
/* Exact f64 Quest scores of every block (block_score for b = 0..nblk-1). */
FX_API int fx_block_scores(fx_ctx* ctx, const float* q, const void* meta, int32_t dtype, int64_t nblk,
                    int32_t dim, double* scores);
/* topk_blocks for one query: blocks_out [dev] [min(k,nblk)] in selection order
 * (score desc, id asc); *k_eff [host] = min(k, nblk); *clamped [host] = k > nblk. */
FX_API int fx_topk_blocks(fx_ctx* ctx, const float* q, const void* meta, int32_t dtype, int64_t nblk,
                   int32_t dim, int64_t k, uint32_t* blocks_out, int64_t* k_eff, int32_t* clamped);

/* The selection prefilter's approximate f32 scores of every block of every
 * head at the group granularity blk [dev] [B][Hkv] -> out [dev] [B][H][nblk16]
 * (row stride nblk16), and the bound scale c of |approx - exact| <= c *
 * sum_d |q_d| absmax_d that fx_decode_step uses ([host] *eps_scale). */
FX_API int fx_approx_scores(fx_ctx* ctx, const fx_layout* lay, const void* const meta[4],
                            const float* q, const int32_t* blk, float* out, double* eps_scale);

/* ---- K5: selector and predictor ------------------------------------------ */
/* plan_group for n groups of G heads (props [dev] [n][G]) plus blocks_for_budget
 * of each head at the chosen granularity. Outputs [dev]. */
FX_API int fx_plan_groups(fx_ctx* ctx, int32_t n_groups, int32_t group_size, int64_t l_cpu,
                   const double* bgt0, const double* kslope, const int32_t* streaming,
                   int32_t* blk, double* budgets, double* volume, double* cand_volumes,
                   int32_t* kblocks);
/* blocks_for_budget on device for n (budget, blk) pairs. */
FX_API int fx_blocks_for_budget(fx_ctx* ctx, int32_t n, const double* budgets, const int32_t* blk,
                         int64_t l_cpu, int32_t* kblocks);

typedef struct fx_model fx_model;
/* Upload a 41->256->384->3 predictor: weights row-major [out][in] f64 and the
 * 41 (mu, sigma) normalization pairs, all [host].  A model holds device scratch
 * (hidden activations, per-row-tile counters of its layer-2 kernel): use it
 * from one stream at a time. */
FX_API int fx_model_create(fx_ctx* ctx, const double* w1, const double* b1, const double* w2,
                    const double* b2, const double* w3, const double* b3, const double* mu,
                    const double* sigma, fx_model** out);
FX_API int fx_model_destroy(fx_model* m);
/* predict() for n raw feature vectors [dev] [n][41] f64 -> head properties
 * bgt0 = clamp(z0,0,1), k = z1, streaming = sigmoid(z2) >= 0.5 (pipeline.cpp:287-288).
 * z [dev, optional] [n][3] raw logits. */
/* Rows are tiled (8 per CTA) so each weight is read once per tile; a model
 * keeps one activation scratch, so calls sharing a model are serialized by
 * the caller (one stream). */
FX_API int fx_predict(fx_ctx* ctx, const fx_model* m, int32_t n, const double* features, double* bgt0,
               double* kslope, int32_t* streaming, double* z);

/* ---- K3/K4: attention ----------------------------------------------------- */
/* One whole decode step of the batch: plan -> score/select -> sparse GQA
 * attention over defaults + selected blocks with the fused LSE merge. */
FX_API int fx_decode_step(fx_ctx* ctx, const fx_layout* lay, const fx_step_args* args);
/* The step's two halves (SURVEY §8b batched extension):
 * fx_plan_select -- plan (any plan mode) + approximate scores + bit-exact top-k:
 *   fills plan_blk / plan_budgets / plan_kblocks and sel_bits (all required),
 *   no attention (topk_blocks for every head, block_index.cpp:55-83);
 * fx_sparse_decode -- attention over the defaults and a given selection
 *   (args->sel_in, plan mode FX_PLAN_GIVEN) with the fused LSE merge
 *   (sparse_attention + merge_into, block_index.cpp:85-94, attention.cpp:89-104). */
FX_API int fx_plan_select(fx_ctx* ctx, const fx_layout* lay, const fx_step_args* args);
FX_API int fx_sparse_decode(fx_ctx* ctx, const fx_layout* lay, const fx_step_args* args);
/* gathered_attention_unchecked for one query over rows idx[0..n) (ascending)
 * of k/v [dev] [rows][dim]; o [dev] [dim] f32, lse [dev] f32 (-inf if n == 0). */
FX_API int fx_gathered_attention(fx_ctx* ctx, const float* q, const void* k, const void* v,
                          int32_t dtype, int64_t rows, int32_t dim, const uint32_t* idx,
                          int64_t n, float* o, float* lse);
/* merge of n partials ([dev] o [n][dim], lse [n]; lse = -inf marks an empty
 * partial) -> o [dev] [dim], lse [dev]. */
FX_API int fx_merge_partials(fx_ctx* ctx, int32_t n, int32_t dim, const float* o_parts,
                      const float* lse_parts, float* o, float* lse);
/* Write decode row `row` (= l_sink+l_cpu+l_local+step) of every (b, g) from
 * k_new/v_new [dev] [B][Hkv][D] f32 (append_new, kv_cache.hpp:68-73). */
FX_API int fx_append_kv(fx_ctx* ctx, const fx_layout* lay, void* k, void* v, int64_t row,
                 const float* k_new, const float* v_new);
/* Convert f32 -> dtype on device (n elements). */
FX_API int fx_convert(fx_ctx* ctx, const float* src, void* dst, int32_t dtype, size_t n);

/* ---- output-aware budget oracle (labels) ---------------------------------- */
/* The oracle head properties of every query head of the batch
 * (pipeline.cpp:256-276, replaces per head: cache_attention attention.cpp:131-141,
 * max_output_norm budget_oracle.cpp:37-41, label_streaming :107-116,
 * min_budget :54-105 at blk 1/16/32/64/128, fit_curve :149-172).
 * k, v: the layout's cache [dev] with l_new decoded rows; meta: the four levels
 * of fx_build_metadata_levels (blk 16..128; may be NULL when l_cpu == 0);
 * q [dev] [B][H][D] f32; criterion 0 = step normalizer max_h ||o_full_h|| of
 * each sequence b (Output+Budget), 1 = ||o_full_h|| (OutputOnly).
 * Outputs [dev]: o_full [B][H][D] f64, normalizer [B], budgets [B][H][5]
 * (min_budget .budget per blk), blocks [B][H][5] (optional), bgt0, kslope
 * [B][H], streaming [B][H] int32.  Synchronizes the ctx stream (the
 * degenerate-normalizer check).  Errors: degenerate-normalizer, bad-shape,
 * empty-context, no-context. */
FX_API int fx_label_heads(fx_ctx* ctx, const fx_layout* lay, const void* k, const void* v,
                          int64_t l_new, const void* const meta[4], const float* q, double tau,
                          int32_t criterion, double* o_full, double* normalizer, double* budgets,
                          int64_t* blocks, double* bgt0, double* kslope, int32_t* streaming);

/* ---- predictor features (features.cpp) ------------------------------------ */
#define FX_STATS_SCALARS 32 /* flat PrefillStats record: 32 scalars + 3 * head_dim */
/* prefill_stats (features.cpp:86-157) for every head, on the prefill cache
 * (no decoded rows): rec [dev] [B][H][32 + 3 D] f64 -- [0] layer [1] head
 * [2] l_cpu [3] l_sink [4] l_local [5] cpu_empty [6..7] sink key/value norm
 * means [8..11] / [12..15] cpu key / value row-norm moments [16..19] z_anchor
 * moments [20..22] anchor lse sink/cpu/local [23..25] anchor output norms
 * [26..29] budget features (min_budget at blk 16..128 for the anchor, the
 * step normalizer; pipeline.cpp:37-46) [30] cross_head_max_anchor
 * [31] ||anchor||, then mean_k_cpu[D], mean_v_cpu[D], anchor[D].
 * anchor [dev] [B][H][D] f32.  Synchronizes the ctx stream. */
FX_API int fx_prefill_stats(fx_ctx* ctx, const fx_layout* lay, const void* k, const void* v,
                            const void* const meta[4], const float* anchor, double tau,
                            int32_t layer, double* rec);
/* decode_features (features.cpp:172-224) for every head: features [dev]
 * [B][H][41] f64 from the step's q [dev] [B][H][D], the cache with l_new
 * decoded rows and the prefill records; feature 39 (cross_head_max_q) is the
 * max over the heads of each sequence of gpu_output_norm (features.cpp:81-84).
 * Feed to fx_predict. */
FX_API int fx_decode_features(fx_ctx* ctx, const fx_layout* lay, const void* k, const void* v,
                              int64_t l_new, const float* q, const double* rec, double* features);
/* decode_features + normalize + predict for every head (features.cpp:162-233,
 * predictor.cpp:161-185, pipeline.cpp:277-290).  The features take two
 * launches: the f64 default-segment attention as 64-row chunk partials over
 * the whole machine, then one merge launch in which the Hkv groups of a
 * sequence run as one thread-block cluster and exchange the cross-head
 * maximum (feature 39) through distributed shared memory; then the
 * predictor's second layer with the output layer fused into its last CTA per
 * row tile.  append_k / append_v [dev] [B][Hkv][D] f32
 * (nullable, together): the previous token (append_new, pipeline.cpp:406-412)
 * is written at decoded row l_new first and counted in (l_new + 1 decoded rows
 * attended) -- pass l_new + 1 to the step that follows.  Writes the head
 * properties bgt0 / kslope / streaming [dev] [B][H] (feed them to
 * fx_decode_step, FX_PLAN_PROPS); features [dev] [B][H][41] and raw logits z
 * [dev] [B][H][3] are optional.  Shapes the split kernels do not cover (group
 * size outside {1,2,4,7,8}, head_dim not 64/128, kv_heads > 8) take the
 * fx_decode_features kernels instead, with the same results. */
FX_API int fx_predict_props(fx_ctx* ctx, const fx_layout* lay, void* k, void* v, int64_t l_new,
                            const float* append_k, const float* append_v, const float* q,
                            const double* rec, const fx_model* model, double* features, double* z,
                            double* bgt0, double* kslope, int32_t* streaming);

/* ---- synthetic workload generator (workload.cpp) ------------------------- */
/* WorkloadSpec (workload.hpp:16-54), same fields and defaults semantics. */
typedef struct fx_workload_spec {
    uint64_t seed;
    int32_t layers, heads, group_size, head_dim, context_len, sink_tokens, local_tokens,
        decode_steps;
    double streaming_frac, retrieval_frac, sink_frac, diffuse_frac;
    int32_t needles, needle_tokens;
    double needle_strength, payload_gain, local_boost, query_jitter, streaming_jitter,
        decoy_strength, decoy_payload_strength;
    int32_t decoy_tokens, decoy_payload_tokens;
    double query_drift;
} fx_workload_spec;
/* generate(spec) (workload.cpp:154-308) into the device cache: batch entry b
 * is layer layers[b] of the workload seeded seeds[b] [host arrays, B each]
 * (the reference has no batch: b = an independent Workload).  K/V bulk on the
 * device (counter-based SplitMix64), the O(d)-per-head structure on the host.
 * Outputs [dev, optional]: anchor_q [B][H][D], step_q [steps][B][H][D],
 * step_new_k / step_new_v [steps][B][Hkv][D] (decode trace, workload.cpp:280-305);
 * archetypes [host, optional] [B][H] (0 streaming, 1 retrieval, 2 sink decoy,
 * 3 diffuse).  The layout must match the spec (heads / group_size groups,
 * head_dim, sink / cpu / local lengths).  Synchronizes the ctx stream.
 * Errors: infeasible-spec, bad-shape. */
FX_API int fx_generate(fx_ctx* ctx, const fx_workload_spec* spec, const fx_layout* lay,
                       const uint64_t* seeds, const int32_t* layers, void* k, void* v,
                       float* anchor_q, int32_t steps, float* step_q, float* step_new_k,
                       float* step_new_v, int32_t* archetypes);

/* ---- FXT1 workload traces (workload.cpp:311-433) ------------------------- */
typedef struct fx_trace_info {
    uint64_t input_hash, seed;
    int32_t layers, heads, group_size, head_dim, context_len, sink_tokens, local_tokens,
        decode_steps;
} fx_trace_info;
/* Read an FXT1 header (import_trace's checks: corrupt-trace / io-error). */
FX_API int fx_trace_info_read(const char* path, fx_trace_info* info);
/* import_trace for one layer into batch entry b of the device cache (f32 ->
 * layout dtype); optional outputs [dev]: anchor_q [H][D], step_q [steps][H][D],
 * new_k / new_v [steps][Hkv][D]; archetypes [host] [H]. */
FX_API int fx_trace_load(fx_ctx* ctx, const char* path, int32_t layer, const fx_layout* lay,
                         int32_t b, void* k, void* v, float* anchor_q, float* step_q,
                         float* new_k, float* new_v, int32_t* archetypes);
/* export_trace: layer ly of the trace = batch entry entries[ly] [host] of the
 * device cache; per-layer arrays [dev] anchor_q [layers][H][D], step_q
 * [layers][steps][H][D], new_k / new_v [layers][steps][Hkv][D] (NULL = zeros);
 * archetypes [host] [layers][H] (NULL = diffuse), needle_count [host]
 * [layers][H] with needles [host] (start, end) pairs in that order (NULL = none). */
FX_API int fx_trace_save(fx_ctx* ctx, const char* path, const fx_trace_info* info,
                         const fx_layout* lay, const int32_t* entries, const void* k,
                         const void* v, const float* anchor_q, const float* step_q,
                         const float* new_k, const float* new_v, const int32_t* archetypes,
                         const int32_t* needle_count, const uint32_t* needles);

/* ---- context-parallel decode (C5) ------------------------------------------
 * The cpu segment is split into contiguous 128-row-aligned shards, one per
 * rank (sink rows on rank 0, local + decoded rows on the last rank), so block
 * b of every granularity lives whole on one shard and keeps its global id.
 * The global top-k of each head (topk_blocks, block_index.cpp:55-83) is
 * reproduced bit-exactly from the shards' local top-k lists:
 *   1. fx_cp_candidates: every shard selects its min(k, nblk_local) best
 *      blocks and emits them with exact reference scores;
 *   2. exchange kth (all-gather) -> fx_cp_threshold: T = max over shards of
 *      the local k-th key, a lower bound of the global k-th score;
 *   3. exchange the entries with key >= T (all-gather) -> fx_cp_select: the
 *      global (score desc, id asc) rank of each own entry, bits for rank < k;
 *   4. fx_decode_step (FX_PLAN_GIVEN + sel_in) -> the shard's (o, lse);
 *   5. exchange (o, lse) (all-gather) -> fx_cp_combine (merge_into).
 * Keys are order-preserving u64 images of the f64 scores (0 = empty slot). */
/* Plan with args->l_cpu_total (plan_* outputs as in fx_decode_step), select this
 * shard's best min(k, nblk_local) blocks per head and emit them sorted (score
 * desc, id asc): keys/ids [dev] [B*H][cap] (global block ids, zero-filled past
 * count), count [dev] [B*H], kth [dev] [B*H] = key of the k-th entry when the
 * shard holds >= k blocks, else 0. */
FX_API int fx_cp_candidates(fx_ctx* ctx, const fx_layout* lay, const fx_step_args* args,
                            int64_t cap, uint64_t* keys, uint32_t* ids, int32_t* count,
                            uint64_t* kth);
/* thresh [dev] [n] = max over the R shards of kth_all [dev] [R][n];
 * keep [dev] [n] = entries of this shard's sorted keys [n][cap] with key >= thresh. */
FX_API int fx_cp_threshold(fx_ctx* ctx, int32_t ranks, int64_t n, int64_t cap,
                           const uint64_t* keys, const uint64_t* kth_all, uint64_t* thresh,
                           int32_t* keep);
/* From the gathered candidates gkeys/gids [dev] [R][n = B*H][m] (each shard's
 * first m sorted entries; slots with key < thresh or key 0 are ignored), set
 * bit (id - cpu_offset/blk) of sel_out [dev] [B*H][sel_words] for every entry
 * of shard `self` whose global rank by (key desc, id asc) is < kblocks[h]. */
FX_API int fx_cp_select(fx_ctx* ctx, const fx_layout* lay, int32_t ranks, int32_t self, int64_t m,
                        const uint64_t* gkeys, const uint32_t* gids, const uint64_t* thresh,
                        const int32_t* kblocks, const int32_t* blk, int64_t cpu_offset,
                        uint32_t* sel_out, int32_t sel_words);
/* merge_into over the R shard partials: o_parts [dev] [R][n][dim], lse_parts
 * [dev] [R][n] (natural log, -inf = empty) -> o [dev] [n][dim], lse [dev] [n]. */
FX_API int fx_cp_combine(fx_ctx* ctx, int32_t ranks, int64_t n, int32_t dim, const float* o_parts,
                         const float* lse_parts, float* o, float* lse);

/* ---- context-parallel exchanges over peer memory (no NCCL) ---------------
 * One-shot alternative to steps 2, 3 and 5 above: every rank's buffers are
 * mapped into every rank (CUDA IPC over NVLink; plain device pointers when the
 * shards share a process) and the kernels read the peers' candidate lists and
 * (o, lse) partials directly, after waiting on each peer's ready flag -- no
 * all-gather, no host round trip for the exchange size.  Pointers [dev]. */
#define FX_CP_MAX_RANKS 16
typedef struct fx_cp_peer {
    const uint64_t* keys;   /* [n][cap] sorted candidate (or band) keys */
    const uint32_t* ids;    /* [n][cap] global block ids */
    const uint64_t* kth;    /* [n] local k-th key (candidate protocol) */
    const float* o;         /* [n][dim] attention partial of the shard */
    const float* lse;       /* [n] */
    const uint64_t* flags;  /* [4] step stamps: 0 candidates / stats, 1 histograms,
                               2 bands, 3 partials */
    int64_t cap;
    const double* stats;    /* [n][4] approx-score min, max, error bound, non-finite (bracket protocol) */
    const int32_t* hist;    /* [n][2048] approx-score histogram over the global range */
    const int32_t* defc;    /* [n][2] blocks certainly in the top-k, band length */
} fx_cp_peer;
/* flags[slot] = stamp after every prior op of the stream is visible system-wide. */
FX_API int fx_cp_signal(fx_ctx* ctx, uint64_t* flags, int32_t slot, uint64_t stamp);
/* Waits for peers[r].flags[0] >= stamp, then threshold + global rank in one
 * kernel (fx_cp_threshold + fx_cp_select over the peers' lists in place). */
FX_API int fx_cp_select_peer(fx_ctx* ctx, const fx_layout* lay, int32_t ranks, int32_t self,
                             const fx_cp_peer* peers, uint64_t stamp, const int32_t* kblocks,
                             const int32_t* blk, int64_t cpu_offset, uint32_t* sel_out,
                             int32_t sel_words);
/* The single-device selection (K2b's bracket) distributed over the ranks --
 * nothing but the band around the global k-th score is ever exact-scored or
 * sorted.  Phases, each launched for every local shard before the next:
 *   0  plan + approximate scores into `approx`; per-head min / max / error
 *      bound -> own stats; (then fx_cp_signal slot 0)
 *   1  wait stats of all ranks; histogram of the local scores over the global
 *      range -> own hist; (signal 1)
 *   2  wait hists; the summed histogram brackets the global k-th score: blocks
 *      above it -> sel_out bits, their count and the band length -> own defc;
 *      the band is exact-scored and sorted (score desc, id asc) -> own keys /
 *      ids; (signal 2)
 *   3  wait bands; global rank of each own band entry among all ranks' bands,
 *      bits for rank < k - sum(defc).
 * args: the shard's step arguments (q, meta, absmax, plan, l_cpu_total,
 * cpu_offset; sel_bits = sel_out).  approx [dev] [n][approx_stride] f32. */
FX_API int fx_cp_dist_phase(fx_ctx* ctx, const fx_layout* lay, const fx_step_args* args,
                            int32_t phase, int32_t ranks, int32_t self, const fx_cp_peer* peers,
                            uint64_t stamp, float* approx, int64_t approx_stride);
/* Waits for peers[r].flags[3] >= stamp, then merge_into over the peers' (o, lse). */
FX_API int fx_cp_combine_peer(fx_ctx* ctx, int32_t ranks, int64_t n, int32_t dim,
                              const fx_cp_peer* peers, uint64_t stamp, float* o, float* lse);
/* CUDA IPC for the peer tables: export the allocation holding dptr (64-byte
 * handle + dptr's offset in it), map a peer's handle into this context's
 * device (add the offset), unmap. */
FX_API int fx_ipc_handle(const void* dptr, unsigned char handle[64], int64_t* offset);
FX_API int fx_ipc_open(fx_ctx* ctx, const unsigned char handle[64], void** dptr);
FX_API int fx_ipc_close(fx_ctx* ctx, void* dptr);

#ifdef __cplusplus
}
#endif
#endif /* FLUXATTN_B200_H */
