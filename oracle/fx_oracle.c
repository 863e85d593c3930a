/*
 * fx_oracle.c -- CPU restatement of the Fluxion sparse-decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_2605_07719_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links or calls it (there is no CPU fallback).
 *
 * Parity pinning: every function below is checked against the compiled
 * reference (oracle/_ref/libfluxref.so, built from /root/reference/proj/src
 * by oracle/Makefile) on the golden vectors in tests/golden/ and on the SPEC
 * known-answer examples (tests/test_oracle.py).
 *
 * Arithmetic rules copied from the reference semantics (not its code):
 *   - storage f32 row-major [rows x dim]; all accumulation in f64, in
 *     sequential index order (matrix.hpp:74-78 `dot`).
 *   - no FMA contraction: the reference is built without -march, so its f64
 *     arithmetic is unfused; this file is compiled with -ffp-contract=off.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define FXO_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------ */
/* Block metadata -- block_index.cpp:10-39, block_index.hpp:16-30       */
/* ------------------------------------------------------------------ */

FXO_API size_t fxo_block_count(size_t rows, int blk) {
    if (blk <= 0) return 0;
    return (rows + (size_t)blk - 1) / (size_t)blk;
}

/* mins/maxs: [nblk x dim].  Returns 0, or -1 for blk <= 0
 * ("invalid-granularity", block_index.cpp:11-12). */
FXO_API int fxo_build_metadata(const float* k, size_t rows, size_t dim, int blk,
                               float* mins, float* maxs) {
    if (blk <= 0) return -1;
    const size_t nblk = fxo_block_count(rows, blk);
    for (size_t b = 0; b < nblk; ++b) {
        const size_t r0 = b * (size_t)blk;
        size_t r1 = r0 + (size_t)blk;
        if (r1 > rows) r1 = rows;
        float* mn = mins + b * dim;
        float* mx = maxs + b * dim;
        memcpy(mn, k + r0 * dim, dim * sizeof(float));
        memcpy(mx, k + r0 * dim, dim * sizeof(float));
        for (size_t r = r0 + 1; r < r1; ++r) {
            const float* row = k + r * dim;
            for (size_t d = 0; d < dim; ++d) {
                /* std::min(a,b) = (b < a) ? b : a ; std::max = (a < b) ? b : a */
                if (row[d] < mn[d]) mn[d] = row[d];
                if (mx[d] < row[d]) mx[d] = row[d];
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Quest block score -- block_index.cpp:41-53                          */
/* ------------------------------------------------------------------ */

FXO_API double fxo_block_score(const float* q, const float* mn, const float* mx, size_t dim) {
    double s = 0.0;
    for (size_t d = 0; d < dim; ++d) {
        const double lo = (double)q[d] * (double)mn[d];
        const double hi = (double)q[d] * (double)mx[d];
        s += (lo < hi) ? hi : lo; /* std::max(lo, hi) */
    }
    return s;
}

typedef struct {
    double score;
    uint32_t id;
} fxo_scored;

/* (score desc, id asc) -- block_index.cpp:68-72 */
static int fxo_cmp_scored(const void* a, const void* b) {
    const fxo_scored* x = (const fxo_scored*)a;
    const fxo_scored* y = (const fxo_scored*)b;
    if (x->score != y->score) return x->score > y->score ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id ? 1 : 0);
}

/* All block scores, [nblk]. */
FXO_API void fxo_block_scores(const float* q, const float* mins, const float* maxs,
                              size_t nblk, size_t dim, double* scores) {
    for (size_t b = 0; b < nblk; ++b)
        scores[b] = fxo_block_score(q, mins + b * dim, maxs + b * dim, dim);
}

/* topk_blocks -- block_index.cpp:55-83.
 * blocks_out: [k_eff] ids in selection order (score desc, id asc).
 * Returns k_eff = min(k, nblk); *clamped = (k > nblk). */
FXO_API size_t fxo_topk_blocks(const float* q, const float* mins, const float* maxs,
                               size_t nblk, size_t dim, size_t k, uint32_t* blocks_out,
                               double* scores_out, int* clamped) {
    int cl = 0;
    if (k > nblk) {
        k = nblk;
        cl = 1;
    }
    if (clamped) *clamped = cl;
    if (k == 0 || nblk == 0) return 0;
    fxo_scored* s = (fxo_scored*)malloc(nblk * sizeof(fxo_scored));
    for (size_t b = 0; b < nblk; ++b) {
        s[b].score = fxo_block_score(q, mins + b * dim, maxs + b * dim, dim);
        s[b].id = (uint32_t)b;
    }
    qsort(s, nblk, sizeof(fxo_scored), fxo_cmp_scored);
    for (size_t i = 0; i < k; ++i) {
        blocks_out[i] = s[i].id;
        if (scores_out) scores_out[i] = s[i].score;
    }
    free(s);
    return k;
}

/* Score of the (k+1)-th ranked block minus the k-th (>= 0), used by the
 * tests to report "mismatch where reference gap < 1e-6" separately. */
FXO_API double fxo_boundary_gap(const float* q, const float* mins, const float* maxs,
                                size_t nblk, size_t dim, size_t k) {
    if (k == 0 || k >= nblk) return INFINITY;
    fxo_scored* s = (fxo_scored*)malloc(nblk * sizeof(fxo_scored));
    for (size_t b = 0; b < nblk; ++b) {
        s[b].score = fxo_block_score(q, mins + b * dim, maxs + b * dim, dim);
        s[b].id = (uint32_t)b;
    }
    qsort(s, nblk, sizeof(fxo_scored), fxo_cmp_scored);
    const double gap = s[k - 1].score - s[k].score;
    free(s);
    return gap;
}

/* token_indices for a selection, ascending (block_index.cpp:77-80).
 * Returns the token count. */
static int fxo_cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

FXO_API size_t fxo_selection_tokens(const uint32_t* blocks, size_t k, int blk, size_t l_cpu,
                                    uint32_t* tokens_out) {
    size_t n = 0;
    for (size_t i = 0; i < k; ++i) {
        const size_t t0 = (size_t)blocks[i] * (size_t)blk;
        size_t t1 = t0 + (size_t)blk;
        if (t1 > l_cpu) t1 = l_cpu;
        for (size_t t = t0; t < t1; ++t) tokens_out[n++] = (uint32_t)t;
    }
    qsort(tokens_out, n, sizeof(uint32_t), fxo_cmp_u32);
    return n;
}

/* blocks_for_budget -- block_index.cpp:96-103 */
FXO_API size_t fxo_blocks_for_budget(double budget, size_t l_cpu, int blk) {
    if (budget <= 0.0 || l_cpu == 0) return 0;
    const size_t nblk = (l_cpu + (size_t)blk - 1) / (size_t)blk;
    const double raw = budget * (double)l_cpu / (double)blk;
    size_t k = (size_t)ceil(raw - 1e-12);
    if (k < 1) k = 1;
    return k < nblk ? k : nblk;
}

/* ------------------------------------------------------------------ */
/* Attention core -- attention.cpp:26-104                              */
/* ------------------------------------------------------------------ */

static double fxo_dot(const float* a, const float* b, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += (double)a[i] * (double)b[i];
    return s;
}

/* gathered_attention_unchecked (attention.cpp:57-87).  idx == NULL means
 * rows 0..n-1 (segment_attention_unchecked, attention.cpp:26-55).
 * o: [dim] f64.  Returns tokens (0 = merge identity; lse = -inf). */
FXO_API size_t fxo_gathered_attention(const float* q, const float* k, const float* v,
                                      size_t dim, const uint32_t* idx, size_t n, double* o,
                                      double* lse) {
    *lse = -INFINITY;
    if (n == 0) return 0;
    const double inv_sqrt_d = 1.0 / sqrt((double)dim);
    double* s = (double*)malloc(n * sizeof(double));
    double m = -INFINITY;
    for (size_t i = 0; i < n; ++i) {
        const size_t r = idx ? idx[i] : i;
        s[i] = fxo_dot(q, k + r * dim, dim) * inv_sqrt_d;
        if (m < s[i]) m = s[i];
    }
    for (size_t j = 0; j < dim; ++j) o[j] = 0.0;
    double denom = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const size_t r = idx ? idx[i] : i;
        const double w = exp(s[i] - m);
        denom += w;
        const float* vr = v + r * dim;
        for (size_t j = 0; j < dim; ++j) o[j] += w * (double)vr[j];
    }
    for (size_t j = 0; j < dim; ++j) o[j] /= denom;
    *lse = m + log(denom);
    free(s);
    return n;
}

/* merge_into (attention.cpp:89-104).  Empty (tokens == 0) is the identity. */
FXO_API void fxo_merge_into(double* acc_o, double* acc_lse, size_t* acc_tokens, const double* o,
                            double lse, size_t tokens, size_t dim) {
    if (tokens == 0) return;
    if (*acc_tokens == 0) {
        memcpy(acc_o, o, dim * sizeof(double));
        *acc_lse = lse;
        *acc_tokens = tokens;
        return;
    }
    const double a = *acc_lse;
    const double tot = a > lse ? a + log1p(exp(lse - a)) : lse + log1p(exp(a - lse));
    const double wa = exp(a - tot);
    const double wb = exp(lse - tot);
    for (size_t j = 0; j < dim; ++j) acc_o[j] = wa * acc_o[j] + wb * o[j];
    *acc_lse = tot;
    *acc_tokens += tokens;
}

/* ------------------------------------------------------------------ */
/* Selector -- selector.cpp:9-46                                       */
/* ------------------------------------------------------------------ */

static const int fxo_candidates[4] = {16, 32, 64, 128}; /* selector.hpp:12 */

static double fxo_clamp01(double x) { return x < 0.0 ? 0.0 : (1.0 < x ? 1.0 : x); }

FXO_API double fxo_volume(int blk, size_t l_cpu, const double* budgets, int n) {
    double sum = 0.0;
    for (int i = 0; i < n; ++i) sum += fxo_clamp01(budgets[i]);
    return 2.0 * (double)l_cpu / (double)blk + 2.0 * (double)l_cpu * sum;
}

FXO_API double fxo_budget_at(double bgt0, double kslope, int streaming, int blk) {
    if (streaming) return 0.0;
    const double k = kslope > 0.0 ? kslope : 0.0; /* std::max(k, 0.0) */
    return fxo_clamp01(bgt0 + k * log2((double)blk));
}

/* plan_group.  budgets_out: [G].  Returns 1 for a streaming group (no
 * task; blk_out = 0), else 0. */
FXO_API int fxo_plan_group(const double* bgt0, const double* kslope, const int* streaming, int G,
                           size_t l_cpu, int* blk_out, double* budgets_out, double* volume_out,
                           double* cand_volumes) {
    int all_streaming = 1;
    for (int h = 0; h < G; ++h)
        if (!streaming[h]) all_streaming = 0;
    *blk_out = 0;
    *volume_out = 0.0;
    for (int c = 0; c < 4; ++c) cand_volumes[c] = 0.0;
    if (all_streaming) return 1;
    double best = 0.0;
    double* tmp = (double*)malloc((size_t)G * sizeof(double));
    for (int c = 0; c < 4; ++c) {
        const int blk = fxo_candidates[c];
        for (int h = 0; h < G; ++h) tmp[h] = fxo_budget_at(bgt0[h], kslope[h], streaming[h], blk);
        const double v = fxo_volume(blk, l_cpu, tmp, G);
        cand_volumes[c] = v;
        if (*blk_out == 0 || v <= best) { /* ties go to the larger blk */
            best = v;
            *blk_out = blk;
            memcpy(budgets_out, tmp, (size_t)G * sizeof(double));
        }
    }
    *volume_out = best;
    free(tmp);
    return 0;
}

/* ------------------------------------------------------------------ */
/* execute_task for one group -- scheduler.cpp:78-96                   */
/* ------------------------------------------------------------------ */

/* One GQA group in the position-ordered layout sink | cpu | local | new
 * ([l_total x dim] f32 each for K and V).  Metadata at plan blk over the
 * cpu segment.  Per head h: defaults (sink, local, new merged in that
 * order, attention.cpp:143-151), then k = blocks_for_budget, topk, sparse
 * gathered attention, merge.  out_o: [G x dim] f64, out_lse: [G]. */
FXO_API void fxo_execute_group(const float* k, const float* v, size_t dim, size_t l_sink,
                               size_t l_cpu, size_t l_local, size_t l_new, const float* queries,
                               int G, int blk, const double* budgets, const float* mins,
                               const float* maxs, double* out_o, double* out_lse,
                               uint64_t* out_tokens) {
    const size_t nblk = fxo_block_count(l_cpu, blk);
    const size_t seg_off[3] = {0, l_sink + l_cpu, l_sink + l_cpu + l_local};
    const size_t seg_len[3] = {l_sink, l_local, l_new};
    double* part = (double*)malloc(dim * sizeof(double));
    uint32_t* sel = (uint32_t*)malloc((nblk ? nblk : 1) * sizeof(uint32_t));
    uint32_t* tok = (uint32_t*)malloc((l_cpu ? l_cpu : 1) * sizeof(uint32_t));
    for (int h = 0; h < G; ++h) {
        const float* q = queries + (size_t)h * dim;
        double* acc = out_o + (size_t)h * dim;
        double acc_lse = -INFINITY;
        size_t acc_tok = 0;
        for (size_t j = 0; j < dim; ++j) acc[j] = 0.0;
        for (int s = 0; s < 3; ++s) {
            if (seg_len[s] == 0) continue;
            double lse;
            const size_t t = fxo_gathered_attention(q, k + seg_off[s] * dim, v + seg_off[s] * dim,
                                                    dim, NULL, seg_len[s], part, &lse);
            fxo_merge_into(acc, &acc_lse, &acc_tok, part, lse, t, dim);
        }
        const size_t kb = blk > 0 ? fxo_blocks_for_budget(budgets[h], l_cpu, blk) : 0;
        if (kb > 0) {
            const size_t ke = fxo_topk_blocks(q, mins, maxs, nblk, dim, kb, sel, NULL, NULL);
            const size_t nt = fxo_selection_tokens(sel, ke, blk, l_cpu, tok);
            double lse;
            const size_t t = fxo_gathered_attention(q, k + l_sink * dim, v + l_sink * dim, dim,
                                                    tok, nt, part, &lse);
            fxo_merge_into(acc, &acc_lse, &acc_tok, part, lse, t, dim);
        }
        out_lse[h] = acc_lse;
        if (out_tokens) out_tokens[h] = acc_tok;
    }
    free(part);
    free(sel);
    free(tok);
}

/* ------------------------------------------------------------------ */
/* Predictor inference -- predictor.cpp:40-53, 161-185                 */
/* ------------------------------------------------------------------ */

/* C[out] = b + sum_i a[i] * W[o][i], bias-first sequential accumulation. */
static void fxo_linear(const double* w, const double* b, size_t in, size_t out, const double* a,
                       double* c) {
    for (size_t o = 0; o < out; ++o) {
        double s = b[o];
        const double* wr = w + o * in;
        for (size_t i = 0; i < in; ++i) s += a[i] * wr[i];
        c[o] = s;
    }
}

/* 41 -> 256 -> 384 -> 3 ReLU MLP on a raw feature vector; normalize with
 * (x - mu)/sigma, zero-sigma dims -> 0 (features.cpp:226-233).
 * out: {bgt0 = clamp(z0,0,1), k = z1, s_prob = sigmoid(z2)}, z_raw: z. */
FXO_API void fxo_predict(const double* w1, const double* b1, const double* w2, const double* b2,
                         const double* w3, const double* b3, const double* mu,
                         const double* sigma, const double* raw, double* out, double* z_raw) {
    double x[41], a1[256], a2[384], z[3];
    for (int i = 0; i < 41; ++i) x[i] = sigma[i] > 0.0 ? (raw[i] - mu[i]) / sigma[i] : 0.0;
    fxo_linear(w1, b1, 41, 256, x, a1);
    for (int i = 0; i < 256; ++i) a1[i] = a1[i] > 0.0 ? a1[i] : 0.0;
    fxo_linear(w2, b2, 256, 384, a1, a2);
    for (int i = 0; i < 384; ++i) a2[i] = a2[i] > 0.0 ? a2[i] : 0.0;
    fxo_linear(w3, b3, 384, 3, a2, z);
    out[0] = fxo_clamp01(z[0]);
    out[1] = z[1];
    out[2] = 1.0 / (1.0 + exp(-z[2]));
    if (z_raw) memcpy(z_raw, z, sizeof z);
}

/* ------------------------------------------------------------------ */
/* Synthetic-input RNG -- rng.hpp:12-64 (SplitMix64 + Box-Muller)      */
/* ------------------------------------------------------------------ */

FXO_API uint64_t fxo_rng_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

FXO_API uint64_t fxo_rng_fork(uint64_t state, uint64_t stream) {
    uint64_t s = state ^ (0xd1b54a32d192ed03ULL * (stream + 1));
    fxo_rng_next(&s);
    return s;
}

FXO_API double fxo_rng_uniform(uint64_t* state) {
    return (double)(fxo_rng_next(state) >> 11) * 0x1.0p-53;
}

FXO_API double fxo_rng_normal(uint64_t* state) {
    double u1 = fxo_rng_uniform(state);
    while (u1 <= 0.0) u1 = fxo_rng_uniform(state);
    const double u2 = fxo_rng_uniform(state);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

/* Fill [n] floats with N(0,1) draws from a SplitMix64 stream. */
FXO_API void fxo_rng_normals(uint64_t seed, float* out, size_t n) {
    uint64_t s = seed;
    for (size_t i = 0; i < n; ++i) out[i] = (float)fxo_rng_normal(&s);
}

/* ------------------------------------------------------------------ */
/* Predictor initialization -- predictor.cpp:26-37 (make_layer),        */
/* 140-148 (make_model): Rng(seed ^ 0xf1c5a77e5eed), w ~ N(0,1)*sqrt(2/in), */
/* biases 0, layers drawn in order from one stream.                    */
/* ------------------------------------------------------------------ */
FXO_API void fxo_make_model(uint64_t seed, double* w1, double* b1, double* w2, double* b2,
                            double* w3, double* b3) {
    uint64_t s = seed ^ 0xf1c5a77e5eedULL;
    double* ws[3] = {w1, w2, w3};
    double* bs[3] = {b1, b2, b3};
    const size_t ins[3] = {41, 256, 384}, outs[3] = {256, 384, 3};
    for (int l = 0; l < 3; ++l) {
        const double scale = sqrt(2.0 / (double)ins[l]);
        for (size_t i = 0; i < ins[l] * outs[l]; ++i) ws[l][i] = fxo_rng_normal(&s) * scale;
        for (size_t o = 0; o < outs[l]; ++o) bs[l][o] = 0.0;
    }
}

/* ------------------------------------------------------------------ */
/* Output-aware budget oracle -- budget_oracle.cpp:13-105, 149-172     */
/* ------------------------------------------------------------------ */

/* l2_norm / l2_distance over f64 (matrix.hpp:86-99): sequential sums. */
static double fxo_l2_norm(const double* x, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += x[i] * x[i];
    return sqrt(s);
}
static double fxo_l2_distance(const double* a, const double* b, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double d = a[i] - b[i];
        s += d * d;
    }
    return sqrt(s);
}

/* max_output_norm (budget_oracle.cpp:37-41): max_h ||o_h||. outs [n][dim]. */
FXO_API double fxo_max_output_norm(const double* outs, size_t n, size_t dim) {
    double m = 0.0;
    for (size_t h = 0; h < n; ++h) {
        const double x = fxo_l2_norm(outs + h * dim, dim);
        if (m < x) m = x;
    }
    return m;
}

/* Segments of one group cache in the position layout sink | cpu | local | new. */
typedef struct {
    const float* k;
    const float* v;
    size_t dim, l_sink, l_cpu, l_local, l_new;
} fxo_cache;

/* default_kv_attention (attention.cpp:143-151): sink, local, new merged in
 * that order.  Returns tokens (0 = empty). */
static size_t fxo_default_partial(const fxo_cache* c, const float* q, double* o, double* lse,
                                  double* part) {
    const size_t off[3] = {0, c->l_sink + c->l_cpu, c->l_sink + c->l_cpu + c->l_local};
    const size_t len[3] = {c->l_sink, c->l_local, c->l_new};
    size_t tok = 0;
    *lse = -INFINITY;
    for (size_t j = 0; j < c->dim; ++j) o[j] = 0.0;
    for (int s = 0; s < 3; ++s) {
        if (len[s] == 0) continue;
        double l;
        const size_t t = fxo_gathered_attention(q, c->k + off[s] * c->dim, c->v + off[s] * c->dim,
                                                c->dim, NULL, len[s], part, &l);
        fxo_merge_into(o, lse, &tok, part, l, t, c->dim);
    }
    return tok;
}

/* cache_attention (attention.cpp:131-141): sink, cpu, local, new merged in
 * position order.  o_full [dim].  Returns -1 on an empty cache. */
FXO_API int fxo_cache_attention(const float* k, const float* v, size_t dim, size_t l_sink,
                                size_t l_cpu, size_t l_local, size_t l_new, const float* q,
                                double* o_full) {
    const size_t off[4] = {0, l_sink, l_sink + l_cpu, l_sink + l_cpu + l_local};
    const size_t len[4] = {l_sink, l_cpu, l_local, l_new};
    double* part = (double*)malloc(dim * sizeof(double));
    double lse = -INFINITY;
    size_t tok = 0;
    for (size_t j = 0; j < dim; ++j) o_full[j] = 0.0;
    for (int s = 0; s < 4; ++s) {
        if (len[s] == 0) continue;
        double l;
        const size_t t = fxo_gathered_attention(q, k + off[s] * dim, v + off[s] * dim, dim, NULL,
                                                len[s], part, &l);
        fxo_merge_into(o_full, &lse, &tok, part, l, t, dim);
    }
    free(part);
    return tok == 0 ? -1 : 0;
}

/* reconstruction_deviation (budget_oracle.cpp:13-20). */
static double fxo_deviation(const double* o, size_t tokens, const double* o_full, size_t dim,
                            double normalizer) {
    if (tokens == 0) return fxo_l2_norm(o_full, dim) / normalizer;
    return fxo_l2_distance(o, o_full, dim) / normalizer;
}

/* label_streaming (budget_oracle.cpp:107-116): 1 = streaming.  Returns -1
 * (degenerate-normalizer) when normalizer == 0 and the cpu segment is
 * non-empty. */
FXO_API int fxo_label_streaming(const float* k, const float* v, size_t dim, size_t l_sink,
                                size_t l_cpu, size_t l_local, size_t l_new, const float* q,
                                const double* o_full, double normalizer, double tau) {
    if (l_cpu == 0) return 1;
    if (normalizer == 0.0) return -1;
    const fxo_cache c = {k, v, dim, l_sink, l_cpu, l_local, l_new};
    double* o = (double*)malloc(dim * sizeof(double));
    double* part = (double*)malloc(dim * sizeof(double));
    double lse;
    const size_t t = fxo_default_partial(&c, q, o, &lse, part);
    const int r = fxo_deviation(o, t, o_full, dim, normalizer) <= tau;
    free(o);
    free(part);
    return r;
}


/* min_budget (budget_oracle.cpp:54-105).  Scans block prefixes in score
 * order; the first whose reconstruction deviation is <= tau wins.
 * Outputs budget (realized token fraction), blocks, saturated.  Returns -1
 * when normalizer == 0 (degenerate-normalizer), -2 on a bad granularity. */
FXO_API int fxo_min_budget(const float* k, const float* v, size_t dim, size_t l_sink, size_t l_cpu,
                           size_t l_local, size_t l_new, const float* q, int blk,
                           const double* o_full, double normalizer, double tau, double* budget,
                           size_t* blocks, int* saturated) {
    if (normalizer == 0.0) return -1;
    if (blk <= 0) return -2;
    const fxo_cache c = {k, v, dim, l_sink, l_cpu, l_local, l_new};
    double* def_o = (double*)malloc(dim * sizeof(double));
    double* part = (double*)malloc(dim * sizeof(double));
    double* acc = (double*)malloc(dim * sizeof(double));
    double* merged = (double*)malloc(dim * sizeof(double));
    double def_lse;
    const size_t def_t = fxo_default_partial(&c, q, def_o, &def_lse, part);
    *budget = 0.0;
    *blocks = 0;
    *saturated = 0;
    if (fxo_deviation(def_o, def_t, o_full, dim, normalizer) <= tau || l_cpu == 0) goto out;
    {
        const float* kc = k + l_sink * dim;
        const float* vc = v + l_sink * dim;
        const size_t nblk = fxo_block_count(l_cpu, blk);
        float* mins = (float*)malloc(nblk * dim * sizeof(float));
        float* maxs = (float*)malloc(nblk * dim * sizeof(float));
        fxo_build_metadata(kc, l_cpu, dim, blk, mins, maxs);
        fxo_scored* sc = (fxo_scored*)malloc(nblk * sizeof(fxo_scored));
        for (size_t b = 0; b < nblk; ++b) {
            sc[b].score = fxo_block_score(q, mins + b * dim, maxs + b * dim, dim);
            sc[b].id = (uint32_t)b;
        }
        qsort(sc, nblk, sizeof(fxo_scored), fxo_cmp_scored); /* score_order: strict total order */
        double acc_lse = -INFINITY;
        size_t acc_t = 0, tokens = 0, i;
        for (i = 0; i < nblk; ++i) {
            const size_t b = sc[i].id;
            const size_t r0 = b * (size_t)blk;
            const size_t r1 = r0 + (size_t)blk < l_cpu ? r0 + (size_t)blk : l_cpu;
            double l;
            const size_t t = fxo_gathered_attention(q, kc + r0 * dim, vc + r0 * dim, dim, NULL,
                                                    r1 - r0, part, &l);
            fxo_merge_into(acc, &acc_lse, &acc_t, part, l, t, dim);
            tokens += r1 - r0;
            /* merged = defaults (+) cpu_acc */
            memcpy(merged, def_o, dim * sizeof(double));
            double m_lse = def_lse;
            size_t m_t = def_t;
            fxo_merge_into(merged, &m_lse, &m_t, acc, acc_lse, acc_t, dim);
            if (fxo_deviation(merged, m_t, o_full, dim, normalizer) <= tau) {
                *budget = (double)tokens / (double)l_cpu;
                *blocks = i + 1;
                break;
            }
        }
        if (i == nblk) {
            *budget = 1.0;
            *blocks = nblk;
            *saturated = 1;
        }
        free(mins);
        free(maxs);
        free(sc);
    }
out:
    free(def_o);
    free(part);
    free(acc);
    free(merged);
    return 0;
}

/* fit_curve (budget_oracle.cpp:149-172): least-squares slope of budget on
 * log2(blk); intercept reported only.  Returns -1 (underdetermined) with
 * fewer than 2 distinct block sizes. */
FXO_API int fxo_fit_curve(const int* blks, const double* budgets, int n, double* k_out,
                          double* free_intercept, double* max_abs_residual) {
    int distinct = 0;
    for (int i = 0; i < n; ++i) {
        int seen = 0;
        for (int j = 0; j < i; ++j)
            if (blks[j] == blks[i]) seen = 1;
        distinct += !seen;
    }
    if (distinct < 2) return -1;
    double sx = 0.0, sy = 0.0;
    for (int i = 0; i < n; ++i) {
        sx += log2((double)blks[i]);
        sy += budgets[i];
    }
    const double nn = (double)n, mx = sx / nn, my = sy / nn;
    double sxx = 0.0, sxy = 0.0;
    for (int i = 0; i < n; ++i) {
        const double dx = log2((double)blks[i]) - mx;
        sxx += dx * dx;
        sxy += dx * (budgets[i] - my);
    }
    const double k = sxy / sxx;
    *k_out = k;
    *free_intercept = my - k * mx;
    double r = 0.0;
    for (int i = 0; i < n; ++i) {
        const double pred = *free_intercept + k * log2((double)blks[i]);
        const double e = fabs(pred - budgets[i]);
        if (r < e) r = e;
    }
    *max_abs_residual = r;
    return 0;
}

/* The oracle-source HeadProperties of one head (pipeline.cpp:256-276):
 * label_streaming, else min_budget at blk 1/16/32/64/128 and fit_curve over
 * the last four with the blk-1 budget as bgt0.  budgets_out [5] (zeros for a
 * streaming head).  Returns the fxo_min_budget / fxo_fit_curve error, or 0. */
FXO_API int fxo_oracle_props(const float* k, const float* v, size_t dim, size_t l_sink,
                             size_t l_cpu, size_t l_local, size_t l_new, const float* q,
                             const double* o_full, double normalizer, double tau, double* bgt0,
                             double* kslope, int* streaming, double* budgets_out) {
    static const int label_blocks[5] = {1, 16, 32, 64, 128}; /* budget_oracle.hpp:26 */
    for (int i = 0; i < 5; ++i) budgets_out[i] = 0.0;
    *bgt0 = *kslope = 0.0;
    const int st = fxo_label_streaming(k, v, dim, l_sink, l_cpu, l_local, l_new, q, o_full,
                                       normalizer, tau);
    if (st < 0) return st;
    *streaming = st;
    if (st) return 0;
    for (int i = 0; i < 5; ++i) {
        size_t nb;
        int sat;
        const int rc = fxo_min_budget(k, v, dim, l_sink, l_cpu, l_local, l_new, q, label_blocks[i],
                                      o_full, normalizer, tau, &budgets_out[i], &nb, &sat);
        if (rc) return rc;
    }
    double icpt, res;
    const int rc = fxo_fit_curve(label_blocks + 1, budgets_out + 1, 4, kslope, &icpt, &res);
    *bgt0 = budgets_out[0];
    return rc;
}

/* ------------------------------------------------------------------ */
/* Features -- features.cpp:26-224                                    */
/* ------------------------------------------------------------------ */

#define FXO_EMPTY_LSE (-1e6) /* kEmptyLse, features.hpp:16 */
#define FXO_STATS_N 32        /* scalar fields of the flat PrefillStats record */

/* compute_moments (features.cpp:26-46): mean, population var, skew, excess kurt. */
FXO_API void fxo_moments(const double* x, size_t n, double* out4) {
    double mean = 0.0, m2 = 0.0, m3 = 0.0, m4 = 0.0;
    out4[0] = out4[1] = out4[2] = out4[3] = 0.0;
    if (n == 0) return;
    for (size_t i = 0; i < n; ++i) mean += x[i];
    mean /= (double)n;
    for (size_t i = 0; i < n; ++i) {
        const double d = x[i] - mean;
        m2 += d * d;
        m3 += d * d * d;
        m4 += d * d * d * d;
    }
    m2 /= (double)n;
    m3 /= (double)n;
    m4 /= (double)n;
    out4[0] = mean;
    out4[1] = m2;
    if (m2 > 0.0) {
        out4[2] = m3 / pow(m2, 1.5);
        out4[3] = m4 / (m2 * m2) - 3.0;
    }
}

static double fxo_l2_norm_f(const float* x, size_t n) { /* matrix.hpp:80-84 */
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += (double)x[i] * (double)x[i];
    return sqrt(s);
}

/* segment_summary (features.cpp:66-77): lse and output norm of one segment. */
static void fxo_segment_summary(const float* q, const float* k, const float* v, size_t rows,
                                size_t dim, double* lse, double* out_norm) {
    *lse = FXO_EMPTY_LSE;
    *out_norm = 0.0;
    if (rows == 0) return;
    double* o = (double*)malloc(dim * sizeof(double));
    fxo_gathered_attention(q, k, v, dim, NULL, rows, o, lse);
    *out_norm = fxo_l2_norm(o, dim);
    free(o);
}

/* gpu_output_norm (features.cpp:81-84): ||default_kv_attention||, 0 if empty. */
FXO_API double fxo_gpu_output_norm(const float* k, const float* v, size_t dim, size_t l_sink,
                                   size_t l_cpu, size_t l_local, size_t l_new, const float* q) {
    const fxo_cache c = {k, v, dim, l_sink, l_cpu, l_local, l_new};
    double* o = (double*)malloc(dim * sizeof(double));
    double* part = (double*)malloc(dim * sizeof(double));
    double lse;
    const size_t t = fxo_default_partial(&c, q, o, &lse, part);
    const double r = t == 0 ? 0.0 : fxo_l2_norm(o, dim);
    free(o);
    free(part);
    return r;
}

/* prefill_stats (features.cpp:86-157) as a flat record of FXO_STATS_N + 3 dim
 * doubles: [0] layer [1] head [2] l_cpu [3] l_sink [4] l_local [5] cpu_empty
 * [6] sink_key_norm_mean [7] sink_value_norm_mean [8..11] k_cpu_norms
 * [12..15] v_cpu_norms [16..19] z_anchor [20..22] lse sink/cpu/local anchor
 * [23..25] out norm sink/cpu/local anchor [26..29] budget_features
 * [30] cross_head_max_anchor [31] ||anchor||, then mean_k_cpu[dim],
 * mean_v_cpu[dim], anchor_query[dim]. */
FXO_API void fxo_prefill_stats(const float* k, const float* v, size_t dim, size_t l_sink,
                               size_t l_cpu, size_t l_local, const float* anchor,
                               const double* budget_features, double cross_head_max_anchor,
                               int layer, int head, double* rec) {
    for (size_t i = 0; i < FXO_STATS_N + 3 * dim; ++i) rec[i] = 0.0;
    double* mk = rec + FXO_STATS_N;
    double* mv = mk + dim;
    double* an = mv + dim;
    rec[0] = layer;
    rec[1] = head;
    rec[2] = (double)l_cpu;
    rec[3] = (double)l_sink;
    rec[4] = (double)l_local;
    rec[5] = l_cpu == 0;
    for (size_t j = 0; j < dim; ++j) an[j] = (double)anchor[j];
    for (int i = 0; i < 4; ++i) rec[26 + i] = budget_features[i];
    rec[30] = cross_head_max_anchor;
    rec[31] = fxo_l2_norm_f(anchor, dim);
    const size_t nmax = l_cpu > l_sink ? l_cpu : l_sink;
    double* tmp = (double*)malloc((nmax ? nmax : 1) * sizeof(double));
    if (l_sink > 0) {
        double s = 0.0;
        for (size_t i = 0; i < l_sink; ++i) tmp[i] = fxo_l2_norm_f(k + i * dim, dim);
        for (size_t i = 0; i < l_sink; ++i) s += tmp[i];
        rec[6] = s / (double)l_sink;
        s = 0.0;
        for (size_t i = 0; i < l_sink; ++i) tmp[i] = fxo_l2_norm_f(v + i * dim, dim);
        for (size_t i = 0; i < l_sink; ++i) s += tmp[i];
        rec[7] = s / (double)l_sink;
    }
    const float* kc = k + l_sink * dim;
    const float* vc = v + l_sink * dim;
    if (l_cpu > 0) {
        for (size_t i = 0; i < l_cpu; ++i)
            for (size_t j = 0; j < dim; ++j) {
                mk[j] += (double)kc[i * dim + j];
                mv[j] += (double)vc[i * dim + j];
            }
        for (size_t j = 0; j < dim; ++j) {
            mk[j] /= (double)l_cpu;
            mv[j] /= (double)l_cpu;
        }
        for (size_t i = 0; i < l_cpu; ++i) tmp[i] = fxo_l2_norm_f(kc + i * dim, dim);
        fxo_moments(tmp, l_cpu, rec + 8);
        for (size_t i = 0; i < l_cpu; ++i) tmp[i] = fxo_l2_norm_f(vc + i * dim, dim);
        fxo_moments(tmp, l_cpu, rec + 12);
        const double qn = rec[31];
        for (size_t i = 0; i < l_cpu; ++i) tmp[i] = 0.0;
        if (qn > 0.0) {
            const double denom = qn * sqrt((double)dim);
            for (size_t i = 0; i < l_cpu; ++i) tmp[i] = fxo_dot(anchor, kc + i * dim, dim) / denom;
        }
        fxo_moments(tmp, l_cpu, rec + 16);
        fxo_segment_summary(anchor, kc, vc, l_cpu, dim, &rec[21], &rec[24]);
    } else {
        rec[21] = FXO_EMPTY_LSE;
    }
    fxo_segment_summary(anchor, k, v, l_sink, dim, &rec[20], &rec[23]);
    const size_t lo = l_sink + l_cpu;
    fxo_segment_summary(anchor, k + lo * dim, v + lo * dim, l_local, dim, &rec[22], &rec[25]);
    free(tmp);
}

/* approx_lse_cpu (features.cpp:159-170). */
static double fxo_approx_lse_cpu(const float* q, const double* rec, size_t dim) {
    const size_t l_cpu = (size_t)rec[2];
    if (l_cpu == 0) return FXO_EMPTY_LSE;
    const double qn = fxo_l2_norm_f(q, dim);
    if (qn == 0.0) return log((double)l_cpu);
    const double* mk = rec + FXO_STATS_N;
    double qk = 0.0;
    for (size_t j = 0; j < dim; ++j) qk += (double)q[j] * mk[j];
    const double mu_q = qk / (qn * sqrt((double)dim));
    return log((double)l_cpu) + qn * mu_q + 0.5 * qn * qn * rec[17];
}

/* decode_features (features.cpp:172-224) -> out[41]. */
FXO_API void fxo_decode_features(const float* k, const float* v, size_t dim, size_t l_sink,
                                 size_t l_cpu, size_t l_local, size_t l_new, const float* q,
                                 const double* rec, double cross_head_max_now, double* f) {
    const double* mk = rec + FXO_STATS_N;
    const double* mv = mk + dim;
    const double* an = mv + dim;
    for (int i = 0; i < 41; ++i) f[i] = 0.0;
    f[0] = rec[0];
    f[1] = rec[1];
    f[2] = rec[2];
    f[3] = rec[3] + rec[4] + (double)l_new;
    f[4] = rec[6];
    f[5] = rec[7];
    f[6] = fxo_l2_norm(mk, dim);
    f[7] = fxo_l2_norm(mv, dim);
    for (int i = 0; i < 4; ++i) {
        f[8 + i] = rec[8 + i];
        f[12 + i] = rec[12 + i];
        f[17 + i] = rec[16 + i];
    }
    const double qn = fxo_l2_norm_f(q, dim);
    if (qn > 0.0 && rec[5] == 0.0) {
        double qk = 0.0;
        for (size_t j = 0; j < dim; ++j) qk += (double)q[j] * mk[j];
        f[16] = qk / (qn * sqrt((double)dim));
    }
    double lse_s, on_s, lse_l, on_l;
    fxo_segment_summary(q, k, v, l_sink, dim, &lse_s, &on_s);
    const size_t lo = l_sink + l_cpu;
    fxo_segment_summary(q, k + lo * dim, v + lo * dim, l_local, dim, &lse_l, &on_l);
    f[21] = lse_s;
    f[22] = fxo_approx_lse_cpu(q, rec, dim);
    f[23] = lse_l;
    f[24] = rec[20];
    f[25] = rec[21];
    f[26] = rec[22];
    f[27] = on_s;
    f[28] = on_l;
    f[29] = rec[23];
    f[30] = rec[24];
    f[31] = rec[25];
    /* ||anchor|| over the float anchor (l2_norm of span<const float>) */
    const double anorm = rec[31];
    f[32] = qn;
    f[33] = anorm;
    if (qn > 0.0 && anorm > 0.0) {
        double d = 0.0;
        for (size_t j = 0; j < dim; ++j) d += (double)q[j] * an[j];
        f[34] = d / (qn * anorm);
    }
    for (int i = 0; i < 4; ++i) f[35 + i] = rec[26 + i];
    f[39] = cross_head_max_now;
    f[40] = rec[30];
}
