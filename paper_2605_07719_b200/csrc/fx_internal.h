// fx_internal.h -- host-side internals shared by the .cu translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "fluxattn_b200.h"

namespace fx {

// Rows per TMA box / per attention "box" (one 16-token slab of one (b, g)).
constexpr int kBoxRows = 16;
// Virtual boxes appended to every (b, g) run when the attention grid splits the
// global box sequence: a run's fixed cost (q load, partial flush, merge) is
// ~this many boxes of streaming, so CTAs covering many short runs get fewer
// boxes.  Virtual boxes are never loaded.
constexpr int kRunPad = 16;
// Batches up to this many (b, g) runs get their run starts rebuilt in smem
// by the attention kernels from the worklist's per-run counts.
constexpr int kMaxRunPrefix = 1024;
// Attention work unit of the TMA kernel: up to this many consecutive boxes of
// one (b, g) (4 pipeline tiles).  The worklist publishes a group's units to a
// queue as soon as the group's boxes exist; persistent attention CTAs claim
// units in publication order.
constexpr int kUnitBoxes = 64;
// Unit queue flag word: epoch (32) | bg (19) | unit index in the group (13).
constexpr int kUnitBgBits = 19, kUnitIdxBits = 13;
// Candidate granularities, selector.hpp:12.
constexpr int kLevels[4] = {16, 32, 64, 128};

struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] inline void fail(int status, const std::string& msg) { throw Error(status, msg); }

#define FX_CUDA(call)                                                                       \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            ::fx::fail(FX_ERR_CUDA, std::string("cuda-error: ") + cudaGetErrorString(e_) + \
                                        " (" #call ")");                                    \
    } while (0)

#define FX_REQUIRE(cond, status, msg)            \
    do {                                         \
        if (!(cond)) ::fx::fail((status), (msg)); \
    } while (0)

// Box descriptor: rows [row, row + n) of one (b, g) (or, for index boxes,
// entries [row, row + n) of an index list); `mask` bit h = query head h of
// the group attends these rows.
struct Box {
    int32_t row;
    uint16_t n;
    uint16_t mask;
};
static_assert(sizeof(Box) == 8, "Box is 8 bytes");

// Device-side bookkeeping of one decode step (lives in ctx scratch).
struct StepCounters {
    int32_t total_boxes;  // filled after the worklist kernel (prefix of per-(b,g) counts)
    int32_t pad[31];
};

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Launch as a programmatic dependent of the previous kernel on the stream
// (see pdl_wait / pdl_trigger in fx_common.cuh).
// PDL is switched off while per-kernel event timing is on (fx_ctx_set_timing),
// so an event pair brackets one kernel alone instead of its programmatic wait
// on the previous one.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    FX_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}
inline int64_t level_blocks(int64_t l_cpu, int blk) { return cdiv(l_cpu, blk); }

// ---- kernel launchers (one per .cu) --------------------------------------
// fx_metadata.cu
// mean (optional): per-block mean keys of the four levels, f32 [B*Hkv][nblk][D]
void launch_meta_levels(const fx_layout& L, const void* k, void* m16, void* m32, void* m64,
                        void* m128, float* absmax, cudaStream_t s, float* const mean[4] = nullptr);
void launch_meta_generic(const void* k, int dtype, int64_t rows, int dim, int blk, void* meta,
                         cudaStream_t s);

// fx_plan.cu
// optional fused append of one decoded row per (b, g) (kv_cache.hpp:68-73)
struct AppendArgs {
    void* k = nullptr;
    void* v = nullptr;
    const float* kn = nullptr;
    const float* vn = nullptr;
    int64_t l_cap = 0, row = 0;
    int D = 0, bf16 = 0;
};
void launch_prepare(const fx_layout& L, int64_t l_plan, int plan_mode, int fixed_blk, double fixed_budget,
                    const double* bgt0, const double* kslope, const int32_t* streaming,
                    int32_t* blk, double* budgets, double* volume, double* cand, int32_t* kblocks,
                    int32_t* bg_done, cudaStream_t s, const AppendArgs& ap = AppendArgs(),
                    int32_t* err = nullptr);
void launch_blocks_for_budget(int n, const double* budgets, const int32_t* blk, int64_t l_cpu,
                              int32_t* kblocks, cudaStream_t s);
// the 41-256-384-3 predictor as tiled f64 layer kernels; scratch holds the
// hidden activations (predict_scratch_bytes(n)); tiles = the model's
// monotonic row-tile counters (predict_row_tiles(n) ints, zeroed once): the
// last layer-2 CTA of a row tile runs the output layer
size_t predict_scratch_bytes(int n);
int predict_row_tiles(int n);
void launch_predict(int n, const double* w1t, const double* b1, const double* w2t,
                    const double* b2, const double* w3t, const double* b3, const double* mu,
                    const double* sigma, const double* feats, double* bgt0, double* kslope,
                    int32_t* streaming, double* z, void* scratch, int32_t* tiles, cudaStream_t s);
// layers 2 and 3 + the head properties from the first hidden layer's output
// a1 [n][256]; a2 [n][384] scratch (the fused feature path computes layer 1)
void launch_predict_tail(int n, const double* a1, const double* w2t, const double* b2, const double* w3t,
                         const double* b3, double* bgt0, double* kslope, int32_t* streaming, double* z,
                         double* a2, int32_t* tiles, cudaStream_t s);

// fx_score.cu / fx_topk.cu / fx_select.cu
double approx_eps_scale(const fx_layout& L);
void launch_approx_scores(const fx_layout& L, const void* const meta[4], const float* q,
                          const int32_t* blk, const int32_t* kblocks, float* approx,
                          int64_t approx_stride, int num_sms, cudaStream_t s, bool rank_all = false);
struct WorklistArgs;
// The attention unit queue a worklist publishes into (words == nullptr: none).
struct UnitQueue {
    uint64_t* words = nullptr;  // [unit_capacity] epoch-tagged flag words
    int32_t* ctl = nullptr;     // [4]: tail, groups, claim, (spare); zeroed by k_prepare
    int32_t* ubase = nullptr;   // [n_bg] first unit id of each group (for the unit merge)
    uint32_t epoch = 0;
};
// wl != nullptr: the selection kernel also builds the attention boxes (fused
// worklist); sel_done = [n_bg] per-group head counters, zeroed by k_prepare.
void launch_select(const fx_layout& L, const void* const meta[4], const float* absmax,
                   const float* q, const int32_t* blk, const int32_t* kblocks,
                   const float* approx, int64_t approx_stride, uint32_t* sel_bits, int sel_words,
                   uint64_t* cand_keys, uint32_t* cand_ids, cudaStream_t s,
                   const WorklistArgs* wl = nullptr, int32_t* sel_done = nullptr);
void launch_worklist(const fx_layout& L, int64_t l_new, const int32_t* blk,
                     const uint32_t* sel_bits, int sel_words, Box* boxes, int64_t box_stride,
                     int32_t* bg_count, int32_t* bg_start, int32_t* done, cudaStream_t s,
                     const UnitQueue& uq = UnitQueue());
void launch_exact_scores(const float* q, const void* meta, int dtype, int64_t nblk, int dim,
                         double* scores, cudaStream_t s);
// exact scores of all blocks, sorted (score desc, id asc); first k ids out.
// tmp arrays hold `cap` (power of two >= nblk) entries.
void launch_topk_exact(const float* q, const void* meta, int dtype, int64_t nblk, int dim,
                       int64_t k, uint32_t* blocks_out, uint64_t* tmp_keys, uint32_t* tmp_ids,
                       int64_t cap, cudaStream_t s);
void launch_meta_absmax(const void* meta, int dtype, int64_t nblk, int dim, float* absmax,
                        cudaStream_t s);

// Flat PrefillStats record (features.hpp:85-110), kStatsN + 3 D doubles per
// head: [0] layer [1] head [2] l_cpu [3] l_sink [4] l_local [5] cpu_empty
// [6] sink_key_norm_mean [7] sink_value_norm_mean [8..11] k_cpu_norms
// [12..15] v_cpu_norms [16..19] z_anchor [20..22] lse sink/cpu/local anchor
// [23..25] out norm sink/cpu/local anchor [26..29] budget_features
// [30] cross_head_max_anchor [31] ||anchor||, then mean_k_cpu[D],
// mean_v_cpu[D], anchor_query[D] (the oracle's fxo_prefill_stats layout).
constexpr int kStatsN = 32;
constexpr double kEmptyLseDev = -1e6;  // kEmptyLse, features.hpp:16

// fx_label.cu: output-aware head labels (budget_oracle.cpp); device outputs.
// prefill_rec != nullptr: q is the anchor and the anchor-side record fields
// are written too (features.cpp:86-157).
size_t label_scratch_bytes(const fx_layout& L, int64_t l_new);
void launch_label(const fx_layout& L, const void* k, const void* v, int64_t l_new, const float* q,
                  const void* const meta[4], double tau, int criterion, void* scratch,
                  double* o_full, double* normalizer, double* budgets, int64_t* blocks,
                  double* bgt0, double* kslope, int32_t* streaming, int32_t* err, cudaStream_t s,
                  double* prefill_rec = nullptr, int layer = 0);
// fx_features.cu: KV-only prefill fields (group statistics) and decode features
void launch_prefill_group(const fx_layout& L, const void* k, const void* v, double* rec,
                          void* scratch, cudaStream_t s);
size_t prefill_group_scratch_bytes(const fx_layout& L);
size_t decode_features_scratch_bytes(const fx_layout& L, int64_t l_new);
void launch_decode_features(const fx_layout& L, const void* k, const void* v, int64_t l_new,
                            const float* q, const double* rec, double* feats, void* scratch,
                            cudaStream_t s);

// fx_predict_step.cu: decode features of every head -- chunk partials over the
// machine, then one clustered merge; l_new counts the appended row (if any)
bool feat_fused_supported(const fx_layout& L);
size_t feat_fused_scratch_bytes(const fx_layout& L, int64_t l_new);
// layer1 = {w1t, b1, mu, sigma} (nullable): the merge kernel also normalizes
// the features and runs the predictor's first layer into a1 [heads][256]
void launch_feat_fused(const fx_layout& L, void* k, void* v, int64_t l_new, const float* q, const double* rec,
                       double* feats, void* scratch, cudaStream_t s, const float* append_k = nullptr,
                       const float* append_v = nullptr, const double* const layer1[4] = nullptr,
                       double* a1 = nullptr, int num_sms = 148);

// fx_workload.cu: generate(spec) into the device cache
void generate_workload(const fx_layout& L, const fx_workload_spec& sp, const uint64_t* seeds,
                       const int32_t* layers, void* k, void* v, float* anchor_q, int32_t steps,
                       float* step_q, float* step_new_k, float* step_new_v, int32_t* archetypes,
                       void* scratch_alloc(size_t, void*), void* alloc_ctx, cudaStream_t s);

// fx_trace.cu: FXT1 traces
void trace_info(const char* path, fx_trace_info* info);
void trace_load(const char* path, int32_t layer, const fx_layout& L, int32_t b, void* k, void* v,
                float* anchor_q, float* step_q, float* new_k, float* new_v, int32_t* archetypes,
                void* scratch_alloc(size_t, void*), void* alloc_ctx, cudaStream_t s);
void trace_save(const char* path, const fx_trace_info& h, const fx_layout& L, const int32_t* entries,
                const void* k, const void* v, const float* anchor_q, const float* step_q,
                const float* new_k, const float* new_v, const int32_t* archetypes,
                const int32_t* needle_count, const uint32_t* needles, cudaStream_t s);
void launch_convert(const float* src, void* dst, int dtype, size_t n, cudaStream_t s);

// fx_cp.cu: peer-memory exchanges
void launch_cp_signal(uint64_t* flags, int slot, uint64_t stamp, cudaStream_t s);
void launch_cp_select_peer(const fx_layout& L, int R, int self, const fx_cp_peer* peers, uint64_t stamp,
                           const int32_t* kblocks, const int32_t* blk, int64_t cpu_offset,
                           uint32_t* sel_out, int sel_words, cudaStream_t s);
void launch_cp_combine_peer(int R, int64_t n, int dim, const fx_cp_peer* peers, uint64_t stamp, float* o,
                            float* lse, cudaStream_t s);
void launch_cp_dist_phase(const fx_layout& L, int phase, int R, int self, const fx_cp_peer* peers,
                          uint64_t stamp, const float* approx, int64_t astride, const float* q,
                          const float* absmax, const void* const meta[4], const int32_t* blk,
                          const int32_t* kblocks, int64_t l_total, int64_t cpu_offset, uint32_t* sel,
                          int sel_words, cudaStream_t s);

// fx_attend.cu
// 3-D TMA map of a bf16 [rows][D] matrix: {64 columns, rows, D/64 chunks},
// box {64, box_rows, D/64}, 128-byte swizzle (D multiple of 64).
CUtensorMap make_row_map(const void* base, int D, int64_t rows, int box_rows);
struct AttendArgs {
    fx_layout L;
    const void* k;
    const void* v;
    const float* q;           // [B][H][D]
    const uint32_t* idx;      // index boxes (API path) or nullptr
    const Box* boxes;         // [n_bg][box_stride]
    int64_t box_stride;
    const int32_t* bg_start;  // [n_bg + 1] exclusive prefix of (box count + pad), for n_bg > 1024
    const int32_t* bg_count;  // [n_bg] box counts (run starts rebuilt in smem for n_bg <= 1024)
    int pad;                  // virtual boxes at the end of each run (kRunPad or 0)
    float* part_o;            // generic: [(grid + n_bg)][G][D]; TMA: [unit][G][D]
    float* part_lse;          // generic: [(grid + n_bg)][G];    TMA: [unit][G]
    int32_t* bg_done;         // [n_bg], zeroed before the launch
    float* o;                 // [B][H][D]
    float* lse;               // [B][H] or nullptr
    // unit queue of the TMA kernel (published by the worklist; see kUnitBoxes)
    UnitQueue uq;             // TMA kernel only; epoch != 0
};
// Units a step can publish at most (partial slots of the TMA kernel).
int64_t unit_capacity(int64_t n_bg, int64_t box_stride);
// The f32 warp-stream kernel (k_attend_f32w) runs this layout; its chunk
// partial slots.
bool f32w_supported(const fx_layout& L, bool has_idx);
int64_t chunk_capacity(int64_t n_bg, int64_t box_stride);
bool attend_uses_tma(const fx_layout& L, bool has_idx);
int attend_grid(const fx_layout& L, bool has_idx, int num_sms);
// the partial merge that follows launch_attend (PDL): the TMA kernel's unit
// partials, or the generic kernel's runs cut by CTA range ends; returns the
// number of kernels launched
int launch_unit_merge(const AttendArgs& a, int grid, bool allow_tma, cudaStream_t s);
// returns the number of kernels launched
int launch_attend(const AttendArgs& a, int grid, bool allow_tma, cudaStream_t s);
void launch_index_boxes(int64_t n, Box* boxes, int32_t* bg_start, int32_t* bg_count,
                        int32_t* bg_done, cudaStream_t s);
void launch_merge_partials(int n, int dim, const float* o_parts, const float* lse_parts, float* o,
                           float* lse, cudaStream_t s);
void launch_append(const fx_layout& L, void* k, void* v, int64_t row, const float* kn,
                   const float* vn, cudaStream_t s);
void launch_convert(const float* src, void* dst, int dtype, size_t n, cudaStream_t s);

// fx_cp.cu (context-parallel shards, config C5)
void launch_cp_candidates(const fx_layout& L, const void* const meta[4], const float* q,
                          const int32_t* blk, const int32_t* kblocks, const uint32_t* sel_bits,
                          int sel_words, int64_t cpu_offset, int64_t cap, uint64_t* keys,
                          uint32_t* ids, int32_t* count, uint64_t* kth, cudaStream_t s);
void launch_cp_threshold(int R, int64_t n, int64_t cap, const uint64_t* keys,
                         const uint64_t* kth_all, uint64_t* thresh, int32_t* keep, cudaStream_t s);
void launch_cp_select(const fx_layout& L, int R, int self, int64_t m, const uint64_t* gkeys,
                      const uint32_t* gids, const uint64_t* thresh, const int32_t* kblocks,
                      const int32_t* blk, int64_t cpu_offset, uint32_t* sel_out, int sel_words,
                      cudaStream_t s);
void launch_cp_combine(int R, int64_t n, int dim, const float* o_parts, const float* lse_parts,
                       float* o, float* lse, cudaStream_t s);

}  // namespace fx
