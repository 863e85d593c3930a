// fx_topk.cu -- K2b: bit-exact budgeted top-k block selection per head,
// topk_blocks (block_index.cpp:55-83): the k highest reference scores, ties to
// the lower block id, k clamped to the block count.
//
// One CTA per head over the approximate scores of fx_score.cu, which satisfy
// |a - s| <= eps for the reference score s:
//   1. a linear value-range histogram of a (2048 bins) locates the bin b* that
//      holds the k-th largest approximate score A_k, so A_k lies in
//      [e_lo, e_hi] = bin b*'s value range widened by one bin on each side
//      (the widening absorbs the f32 rounding of the bin map);
//   2. a > e_hi + 2 eps  =>  s > A_k + eps >= (true k-th score): in the
//      reference top-k whatever the tie rule;  a < e_lo - 2 eps  =>  out;
//      everything else is the "band" (typically tens of blocks);
//   3. band blocks are re-scored with the reference recipe -- products in f64
//      (exact) by a warp, the sum in dimension order by one lane, unfused --
//      and ranked by (score desc, id asc); the rest of the k come from there.
// Output: the selection as a bitmask over the group's blocks.
#include <algorithm>

#include "fx_common.cuh"

namespace fx {
namespace {

// threads per selection CTA: 256 (four CTAs per SM) when the heads outnumber
// the SMs; 512 / 1024 when two / one CTA per SM hold every head and a head
// has >= 16 blocks per thread at blk 16, so a small batch of long contexts
// (C3, C5) splits each head's passes over more threads
constexpr int kTMin = 256, kTMax = 1024;
constexpr int kBins = 2048;
// the histogram is stored with one padding word per 32 bins (bin b at
// b + b / 32): lanes whose bins differ by a multiple of 32 hit different banks
constexpr int kHistWords = kBins + kBins / 32;
__device__ __forceinline__ int hidx(int b) { return b + (b >> 5); }
constexpr int kMaxWords = 4096;   // nblk <= 131072 at the chosen granularity
constexpr int kSmemKeys = 16384;  // approximate scores staged in smem up to this many
constexpr int kSmallCand = 512;   // band ranked in smem up to this size (a power of two)
constexpr int kSortCand = 192;    // ... by counting up to this size, by a bitonic sort above

#ifdef FX_TRACE  // profiling build only: per-head phase times and band sizes
__device__ long long g_sel_trace[16 * 8192];
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SEL_MARK(i) \
    if (threadIdx.x == 0 && blockIdx.x < 8192) g_sel_trace[blockIdx.x * 16 + (i)] = gtimer();
#else
#define SEL_MARK(i)
#endif
}  // namespace
}  // namespace fx
#define WL_MARK(i) SEL_MARK(i)
#include "fx_worklist.cuh"
namespace fx {
namespace {

struct MetaPtrs {
    const void* p[4];
};
__device__ __forceinline__ const void* level_ptr(const void* const* meta, int blk) {
    return meta[blk == 16 ? 0 : blk == 32 ? 1 : blk == 64 ? 2 : 3];
}

// Reference score of one block by one thread (block_index.cpp:41-53): f64
// products (exact), summed in dimension order, unfused.  q is f64 in smem;
// the metadata row (smem or global, generic 16-byte loads) in vectors.
__device__ __forceinline__ double score_step(double s, double qd, float lo, float hi) {
    const double a = __dmul_rn(qd, (double)lo), c = __dmul_rn(qd, (double)hi);
    return __dadd_rn(s, (a < c) ? c : a);
}
__device__ double exact_score_vec(const double* __restrict__ qs, const __nv_bfloat16* __restrict__ mn,
                                  const __nv_bfloat16* __restrict__ mx, int D) {
    double s = 0.0;
    if ((D & 7) == 0) {
#pragma unroll 4
        for (int d = 0; d < D; d += 8) {
            const uint4 a = *reinterpret_cast<const uint4*>(mn + d);
            const uint4 c = *reinterpret_cast<const uint4*>(mx + d);
            const uint32_t av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                s = score_step(s, qs[d + 2 * u], bf16lo_to_f(av[u]), bf16lo_to_f(cv[u]));
                s = score_step(s, qs[d + 2 * u + 1], bf16hi_to_f(av[u]), bf16hi_to_f(cv[u]));
            }
        }
        return s;
    }
    for (int d = 0; d < D; ++d) s = score_step(s, qs[d], __bfloat162float(mn[d]), __bfloat162float(mx[d]));
    return s;
}
__device__ double exact_score_vec(const double* __restrict__ qs, const float* __restrict__ mn,
                                  const float* __restrict__ mx, int D) {
    double s = 0.0;
    if ((D & 3) == 0) {
        for (int d = 0; d < D; d += 4) {
            const float4 a = *reinterpret_cast<const float4*>(mn + d);
            const float4 c = *reinterpret_cast<const float4*>(mx + d);
            s = score_step(s, qs[d], a.x, c.x);
            s = score_step(s, qs[d + 1], a.y, c.y);
            s = score_step(s, qs[d + 2], a.z, c.z);
            s = score_step(s, qs[d + 3], a.w, c.w);
        }
        return s;
    }
    for (int d = 0; d < D; ++d) s = score_step(s, qs[d], mn[d], mx[d]);
    return s;
}

// Same sum over a row in shared (or global) memory, 16-byte reads.
__device__ __forceinline__ double exact_score_smem(const double* qs, const __nv_bfloat16* mn,
                                                   const __nv_bfloat16* mx, int D) {
    return exact_score_vec(qs, mn, mx, D);
}
__device__ __forceinline__ double exact_score_smem(const double* qs, const float* mn,
                                                   const float* mx, int D) {
    return exact_score_vec(qs, mn, mx, D);
}

template <int DT, int kT>
__device__ __forceinline__ void select_head(
    MetaPtrs meta, const float* __restrict__ absmax, const float* __restrict__ q,
    const int32_t* __restrict__ blk_arr, const int32_t* __restrict__ kblocks, int Hkv, int G,
    int D, int64_t l_cpu, const float* __restrict__ approx, int64_t astride, double eps_scale,
    uint32_t* __restrict__ sel_bits, int sel_words, uint64_t* __restrict__ cand_keys,
    uint32_t* __restrict__ cand_ids, int64_t cand_stride, int keys_cap) {
    using T = typename Elem<DT>::T;
    constexpr int kNW = kT / 32;
    // dynamic smem: keys[keys_cap] f32 | hist[kHistWords] | q[D] f64 | ck[kSmallCand] | ci[kSmallCand]
    extern __shared__ __align__(16) unsigned char dsm[];
    float* s_keys = reinterpret_cast<float*>(dsm);
    int32_t* hist = reinterpret_cast<int32_t*>(dsm + (size_t)keys_cap * 4);
    double* s_q = reinterpret_cast<double*>(hist + kHistWords);
    uint64_t* ck = reinterpret_cast<uint64_t*>(s_q + D);
    uint32_t* ci = reinterpret_cast<uint32_t*>(ck + kSmallCand);
    __shared__ float red[2][kNW];
    __shared__ int s_wsum[2][kNW];
    __shared__ int s_bin;
    __shared__ int s_ncand;
    __shared__ double s_eps;

    const int64_t head = blockIdx.x;
    const int64_t H = (int64_t)Hkv * G;
    const int b = (int)(head / H), h = (int)(head % H), g = h / G;
    const int bg = b * Hkv + g;
    // the plan comes from k_prepare (two launches back, complete before the
    // scorer began, hence before this grid launched); read through L2
    const int blk = __ldcg(blk_arr + bg);
    const int64_t k = __ldcg(kblocks + head);
    uint32_t* bits = sel_bits + head * sel_words;
    const int64_t nblk = blk > 0 ? cdiv_dev(l_cpu, blk) : 0;
    const int W = (int)cdiv_dev(nblk, 32);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

    if (nblk == 0 || k <= 0) {
        for (int j = t; j < W; j += kT) bits[j] = 0u;
        return;
    }
    if (k >= nblk) {  // clamped: every block (block_index.cpp:61-64)
        for (int j = t; j < W; j += kT) {
            const int64_t rem = nblk - (int64_t)j * 32;
            bits[j] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
        }
        return;
    }
    SEL_MARK(0);
    const T* mbase = static_cast<const T*>(level_ptr(meta.p, blk)) + (int64_t)bg * nblk * 2 * D;
    const float* qh = q + head * D;
    const float* sc = approx + head * astride;
    const bool staged = nblk <= keys_cap;

    // everything that does not depend on the scorer first: q, the error bound,
    // the histogram; then the programmatic wait for the scorer's output
    for (int i = t; i < kHistWords; i += kT) hist[i] = 0;
    if (t == 0) s_ncand = 0;
    for (int d = t; d < D; d += kT) s_q[d] = (double)qh[d];
    if (warp == 0) {
        double a = 0.0;
        for (int d = lane; d < D; d += 32)
            a += fabs((double)qh[d]) * (double)absmax[(int64_t)bg * D + d];
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) s_eps = a * eps_scale * 1.01 + 1e-30;
    }
    pdl_wait();
    // ---- 0. stage (128-bit loads, several in flight), min/max, error bound ----
    float mx = -INFINITY, mn = INFINITY;
    bool fin_all = true;
    auto see = [&](float a) {
        if (isfinite(a)) {
            mx = fmaxf(mx, a);
            mn = fminf(mn, a);
        } else {
            fin_all = false;
        }
    };
    {
        const int64_t n4 = nblk >> 2;
        const float4* sc4 = reinterpret_cast<const float4*>(sc);
#pragma unroll 4
        for (int64_t i = t; i < n4; i += kT) {
            const float4 v = __ldg(sc4 + i);
            if (staged) reinterpret_cast<float4*>(s_keys)[i] = v;
            see(v.x);
            see(v.y);
            see(v.z);
            see(v.w);
        }
        for (int64_t i = n4 * 4 + t; i < nblk; i += kT) {
            const float a = sc[i];
            if (staged) s_keys[i] = a;
            see(a);
        }
    }
    // one barrier round for max, min and finiteness
    mx = warp_max(mx);
    mn = -warp_max(-mn);
    if (lane == 0) {
        red[0][warp] = mx;
        red[1][warp] = mn;
    }
    const bool sane_local = __syncthreads_and(fin_all);
    float gmx = -INFINITY, gmn = INFINITY;
#pragma unroll
    for (int i = 0; i < kNW; ++i) {
        gmx = fmaxf(gmx, red[0][i]);
        gmn = fminf(gmn, red[1][i]);
    }
    const bool sane = sane_local && isfinite(s_eps);
    const float* src = staged ? s_keys : sc;
    const double eps = s_eps;
    SEL_MARK(1);

    // ---- 1. bracket A_k ----
    double e_lo = -INFINITY, e_hi = INFINITY;  // non-finite prefilter: band = everything
    if (sane && !(gmx > gmn)) {
        e_lo = e_hi = (double)gmx;  // all equal: A_k is that value
    } else if (sane) {
        const float scale = (float)kBins / (gmx - gmn);
        for (int64_t i = t; i < nblk; i += kT) {
            const float f = (src[i] - gmn) * scale;
            atomicAdd(&hist[hidx(f >= (float)(kBins - 1) ? kBins - 1 : (f <= 0.f ? 0 : (int)f))], 1);
        }
        __syncthreads();
        // bin holding the k-th largest: each thread owns kBins/kT bins; suffix
        // sums over threads (from the top) locate the owner, which scans them
        constexpr int PB = kBins / kT;
        static_assert(PB >= 2 && PB <= 8, "kBins / kT consecutive bins per thread");
        int hb[PB];  // this thread's PB consecutive bins (one padded row of 32 holds them)
#pragma unroll
        for (int i = 0; i < PB; ++i) hb[i] = hist[hidx(t * PB + i)];
        int c = 0;
#pragma unroll
        for (int i = 0; i < PB; ++i) c += hb[i];
        int x = c;  // suffix sum within the warp (lanes >= lane)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_down_sync(0xffffffffu, x, o);
            if (lane + o < 32) x += y;
        }
        if (lane == 0) s_wsum[0][warp] = x;
        __syncthreads();
        int S = x;
        for (int w = warp + 1; w < kNW; ++w) S += s_wsum[0][w];
        if (S >= k && S - c < k) {
            int above = S - c;
#pragma unroll
            for (int i = PB - 1; i >= 0; --i) {
                above += hb[i];
                if (above >= k) {
                    s_bin = t * PB + i;
                    break;
                }
            }
        }
        __syncthreads();
        const double w = ((double)gmx - (double)gmn) / kBins;
        e_lo = (double)gmn + (s_bin - 1) * w;
        e_hi = (double)gmn + (s_bin + 2) * w;
    }
    const double hi = e_hi + 2.0 * eps, lo = e_lo - 2.0 * eps;
    SEL_MARK(2);

    // ---- 2. classify in one warp pass: definite-in bits, band ids appended
    // through a shared counter (one atomic per warp word that has any).  The
    // band's order is irrelevant: it is ranked by (exact score, id) below. ----
    uint32_t* cids = cand_ids + head * cand_stride;
    uint64_t* ckeys = cand_keys + head * cand_stride;
    int wdef = 0;  // this warp's definite count (all lanes)
    for (int j = warp; j < W; j += kNW) {
        const int64_t i = (int64_t)j * 32 + lane;
        const bool in = i < nblk;
        const double a = in ? (double)src[i] : 0.0;
        const uint32_t bd = __ballot_sync(0xffffffffu, in && a > hi);
        const bool cand = in && !(a > hi) && a >= lo;
        const uint32_t bc = __ballot_sync(0xffffffffu, cand);
        if (lane == 0) bits[j] = bd;
        wdef += __popc(bd);
        if (bc) {
            int base = 0;
            if (lane == 0) base = atomicAdd(&s_ncand, __popc(bc));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (cand) {
                const int pos = base + __popc(bc & ((1u << lane) - 1u));
                if (pos < kSmallCand) ci[pos] = (uint32_t)i;
                cids[pos] = (uint32_t)i;  // (read only when the band outgrows ci)
                // the row is exact-scored next: start it towards L2 now
                if (pos < kSmallCand && ((2 * D * sizeof(T)) & 15) == 0)
                    prefetch_l2_bulk(mbase + (int64_t)i * 2 * D, (uint32_t)(2 * D * sizeof(T)));
            }
        }
    }
    if (lane == 0) s_wsum[0][warp] = wdef;
    __syncthreads();
    int64_t n_def = 0;
#pragma unroll
    for (int w = 0; w < kNW; ++w) n_def += s_wsum[0][w];
    const int64_t n_cand = s_ncand;
    const bool small = n_cand <= kSmallCand;
    const int64_t need = k - n_def;
    __syncthreads();
    SEL_MARK(3);
#ifdef FX_TRACE
    if (t == 0 && blockIdx.x < 8192) g_sel_trace[blockIdx.x * 16 + 6] = n_cand | (n_def << 32);
    if (t == 0 && blockIdx.x < 8192) g_sel_trace[blockIdx.x * 16 + 7] = k | ((int64_t)nblk << 32);
#endif

    // ---- 3. exact reference scores of the band ----
    // bf16: the terms max(q_d mn_d, q_d mx_d) (exact f64 products) are formed
    // in parallel -- 8 dims per thread straight from the metadata row, one
    // round trip -- into smem (over the no longer needed keys + histogram),
    // then one thread per candidate adds its D terms in dimension order: the
    // reference sum, with only the dependent adds left serial.
    constexpr bool kTerms = DT == FX_BF16;
    // term layout of a candidate: dims in groups of 8 with a one-double skew
    // per group (index (d / 8) * 9 + d % 8), so the 16 writers of a candidate
    // (8 dims each) hit 16 distinct bank pairs; odd candidate pitch, so the
    // serial readers (one candidate each) spread over the banks too
    const int tpitch = (D / 8) * 9 + 1;  // doubles
    const int per_round_t = ((int)((size_t)keys_cap * 4 + kHistWords * 4)) / (tpitch * 8);
    // a band of more than two term rounds: one candidate per thread instead,
    // its row read straight from L2 in 16-byte vectors (all candidates at once)
    const bool direct = kTerms && (D & 7) == 0 && n_cand > 2 * (int64_t)per_round_t;
    if (direct) {
        for (int64_t c = t; c < n_cand; c += kT) {
            const uint32_t id = small ? ci[c] : cids[c];
            const T* row = mbase + (int64_t)id * 2 * D;
            const double sc_ = exact_score_vec(s_q, row, row + D, D);
            if (small) ck[c] = f64_key(sc_);
            else ckeys[c] = f64_key(sc_);
        }
    } else if (kTerms && (D & 7) == 0 && per_round_t >= 1) {
        double* term = reinterpret_cast<double*>(dsm);
        const int v8 = D / 8;
        // a thread's 8 dims are the same for every candidate (kT % v8 == 0):
        // its q slice in registers, read from global (L1) -- the shared copy's
        // 64-byte-strided reads were 8-way bank conflicts
        double qv[8];
        const bool qreg = kT % v8 == 0;
        if (qreg) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(qh + 8 * (t % v8)));
            const float4 c = __ldg(reinterpret_cast<const float4*>(qh + 8 * (t % v8)) + 1);
            qv[0] = a.x, qv[1] = a.y, qv[2] = a.z, qv[3] = a.w;
            qv[4] = c.x, qv[5] = c.y, qv[6] = c.z, qv[7] = c.w;
        }
        for (int64_t c0 = 0; c0 < n_cand; c0 += per_round_t) {
            const int nc = (int)(n_cand - c0 < per_round_t ? n_cand - c0 : per_round_t);
            for (int e = t; e < nc * v8; e += kT) {
                const int cc = e / v8, u = e % v8;
                const uint32_t id = small ? ci[c0 + cc] : cids[c0 + cc];
                const T* row = mbase + (int64_t)id * 2 * D;
                const uint4 a = __ldg(reinterpret_cast<const uint4*>(row) + u);
                const uint4 c = __ldg(reinterpret_cast<const uint4*>(row + D) + u);
                const uint32_t av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
                double* tr = term + (size_t)cc * tpitch + 9 * u;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const double q0 = qreg ? qv[2 * j] : s_q[8 * u + 2 * j];
                    const double q1 = qreg ? qv[2 * j + 1] : s_q[8 * u + 2 * j + 1];
                    const double x0 = __dmul_rn(q0, (double)bf16lo_to_f(av[j]));
                    const double y0 = __dmul_rn(q0, (double)bf16lo_to_f(cv[j]));
                    const double x1 = __dmul_rn(q1, (double)bf16hi_to_f(av[j]));
                    const double y1 = __dmul_rn(q1, (double)bf16hi_to_f(cv[j]));
                    tr[2 * j] = (x0 < y0) ? y0 : x0;
                    tr[2 * j + 1] = (x1 < y1) ? y1 : x1;
                }
            }
            __syncthreads();
            for (int cc = t; cc < nc; cc += kT) {
                const double* tr = term + (size_t)cc * tpitch;
                double sum = 0.0;
                for (int g8 = 0; g8 < D / 8; ++g8)  // dimension order
#pragma unroll
                    for (int j = 0; j < 8; ++j) sum = __dadd_rn(sum, tr[9 * g8 + j]);
                const int64_t c = c0 + cc;
                if (small) ck[c] = f64_key(sum);
                else ckeys[c] = f64_key(sum);
            }
            __syncthreads();
        }
    } else {
        const int row_b = 2 * D * (int)sizeof(T);
        const int pitch = row_b + 16;  // 16-byte skew: conflict-free row-parallel reads
        const int per_round = ((int)((size_t)keys_cap * 4 + kHistWords * 4)) / pitch;
        const bool vec = (row_b & 15) == 0 && per_round >= 1;
        unsigned char* stage = dsm;
        for (int64_t c0 = 0; c0 < n_cand; c0 += (vec ? per_round : n_cand)) {
            const int64_t step_ = vec ? (int64_t)per_round : n_cand;
            const int nc = (int)(n_cand - c0 < step_ ? n_cand - c0 : step_);
            if (vec) {
                const int v16 = row_b / 16;
                for (int e = t; e < nc * v16; e += kT) {
                    const int cc = e / v16, u = e % v16;
                    const uint32_t id = small ? ci[c0 + cc] : cids[c0 + cc];
                    const uint4 x = __ldg(reinterpret_cast<const uint4*>(mbase + (int64_t)id * 2 * D) + u);
                    *reinterpret_cast<uint4*>(stage + (size_t)cc * pitch + u * 16) = x;
                }
                __syncthreads();
            }
            for (int cc = t; cc < nc; cc += kT) {
                const int64_t c = c0 + cc;
                const uint32_t id = small ? ci[c] : cids[c];
                const T* mrow = vec ? reinterpret_cast<const T*>(stage + (size_t)cc * pitch)
                                    : mbase + (int64_t)id * 2 * D;
                const double sc_ = exact_score_smem(s_q, mrow, mrow + D, D);
                if (small) ck[c] = f64_key(sc_);
                else ckeys[c] = f64_key(sc_);
            }
            __syncthreads();
        }
    }
    __syncthreads();
    SEL_MARK(4);
    if (small && n_cand > kSortCand) {
        // a wide band: bitonic sort of the (key, id) pairs in place, best
        // first (key desc, id asc; pad entries (0, ~0u) sort last), then the
        // first `need` are in -- log2(p) (log2(p) + 1) / 2 barrier stages
        // instead of the O(n^2) ranking below
        const int nc = (int)n_cand;
        int p = 1;
        while (p < nc) p <<= 1;
        for (int i = nc + t; i < p; i += kT) {
            ck[i] = 0ull;
            ci[i] = 0xffffffffu;
        }
        __syncthreads();
        for (int size = 2; size <= p; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int i = t; i < (p >> 1); i += kT) {
                    const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                    const uint64_t ka = ck[lo], kb = ck[hi];
                    const uint32_t ia = ci[lo], ib = ci[hi];
                    const bool b_first = (kb > ka) || (kb == ka && ib < ia);
                    const bool a_first = (ka > kb) || (ka == kb && ia < ib);
                    if ((lo & size) == 0 ? b_first : a_first) {
                        ck[lo] = kb;
                        ck[hi] = ka;
                        ci[lo] = ib;
                        ci[hi] = ia;
                    }
                }
                __syncthreads();
            }
        }
        const int take = (int)(need < (int64_t)nc ? need : (int64_t)nc);
        for (int i = t; i < take; i += kT) atomicOr(&bits[ci[i] >> 5], 1u << (ci[i] & 31));
    } else if (small) {
        // rank of each candidate by counting the ones ahead of it; four
        // (key, id) pairs per 16-byte shared read (ck / ci are 16-byte
        // aligned unless D is odd), stopping once `need` are ahead (it is out)
        const int nc = (int)n_cand, nc4 = (D & 1) ? 0 : nc & ~3;
        for (int c = t; c < nc; c += kT) {
            const uint64_t kc = ck[c];
            const uint32_t idc = ci[c];
            int rank = 0;
            auto ahead = [&](uint64_t kj, uint32_t ij) { return (int)((kj > kc) || (kj == kc && ij < idc)); };
            int j = 0;
            for (; j < nc4 && rank < need; j += 4) {
                const ulonglong2 k01 = *reinterpret_cast<const ulonglong2*>(ck + j);
                const ulonglong2 k23 = *reinterpret_cast<const ulonglong2*>(ck + j + 2);
                const uint4 i4 = *reinterpret_cast<const uint4*>(ci + j);
                rank += ahead(k01.x, i4.x) + ahead(k01.y, i4.y) + ahead(k23.x, i4.z) + ahead(k23.y, i4.w);
            }
            for (; j < nc && rank < need; ++j) rank += ahead(ck[j], ci[j]);
            if (rank < need) atomicOr(&bits[idc >> 5], 1u << (idc & 31));
        }
    } else {
        // Large band (degenerate data, e.g. equal keys): block-wide radix select
        // of the need-th largest key K* (8 passes of 8 bits over the band in
        // global scratch), every key > K* in, then the tied keys == K* lowest
        // id first -- the take-th smallest id by a second radix select.
        int32_t* h = reinterpret_cast<int32_t*>(dsm);  // 256 bins (the keys area is free)
        __shared__ uint64_t s_pref;
        __shared__ int64_t s_cnt;
        uint64_t pref = 0, msk = 0;
        int64_t above = 0;
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int i = t; i < 256; i += kT) h[i] = 0;
            __syncthreads();
            for (int64_t c = t; c < n_cand; c += kT) {
                const uint64_t kc = ckeys[c];
                if ((kc & msk) == pref) atomicAdd(&h[(kc >> shift) & 255], 1);
            }
            __syncthreads();
            if (t == 0) {  // highest digit whose cumulative count from the top reaches need
                int64_t cum = above;
                int d = 255;
                for (; d > 0; --d) {
                    if (cum + h[d] >= need) break;
                    cum += h[d];
                }
                s_pref = pref | ((uint64_t)d << shift);
                s_cnt = cum;  // keys above digit d's bucket
            }
            __syncthreads();
            pref = s_pref;
            above = s_cnt;
            msk |= 0xffull << shift;
        }
        const uint64_t kstar = pref;
        const int64_t take = need - above;  // >= 1 keys equal to K*
        for (int64_t c = t; c < n_cand; c += kT)
            if (ckeys[c] > kstar) atomicOr(&bits[cids[c] >> 5], 1u << (cids[c] & 31));
        uint32_t ipref = 0, imsk = 0;
        int64_t below = 0;
        for (int shift = 24; shift >= 0; shift -= 8) {
            for (int i = t; i < 256; i += kT) h[i] = 0;
            __syncthreads();
            for (int64_t c = t; c < n_cand; c += kT) {
                const uint32_t ic = cids[c];
                if (ckeys[c] == kstar && (ic & imsk) == ipref) atomicAdd(&h[(ic >> shift) & 255], 1);
            }
            __syncthreads();
            if (t == 0) {  // lowest digit whose cumulative count from the bottom reaches take
                int64_t cum = below;
                int d = 0;
                for (; d < 255; ++d) {
                    if (cum + h[d] >= take) break;
                    cum += h[d];
                }
                s_pref = ipref | ((uint32_t)d << shift);
                s_cnt = cum;
            }
            __syncthreads();
            ipref = (uint32_t)s_pref;
            below = s_cnt;
            imsk |= 0xffu << shift;
        }
        for (int64_t c = t; c < n_cand; c += kT)  // ids are distinct: exactly `take` of them
            if (ckeys[c] == kstar && cids[c] <= ipref) atomicOr(&bits[cids[c] >> 5], 1u << (cids[c] & 31));
    }
    __syncthreads();
    SEL_MARK(5);
}

// One CTA per head.  With `wl.boxes` set, the CTA that completes the last head
// of a group (sel_done[bg] reaches G) goes on to build that group's attention
// boxes (fx_worklist.cuh) -- the union of the G selections is final then.
template <int DT, int kT>
__global__ void __launch_bounds__(kT) k_select(
    MetaPtrs meta, const float* __restrict__ absmax, const float* __restrict__ q,
    const int32_t* __restrict__ blk_arr, const int32_t* __restrict__ kblocks, int Hkv, int G,
    int D, int64_t l_cpu, const float* __restrict__ approx, int64_t astride, double eps_scale,
    uint32_t* __restrict__ sel_bits, int sel_words, uint64_t* __restrict__ cand_keys,
    uint32_t* __restrict__ cand_ids, int64_t cand_stride, int keys_cap, WorklistArgs wl,
    int32_t* __restrict__ sel_done) {
    pdl_trigger();  // select_head waits for the scorer once its independent setup is done
    SEL_MARK(10);
    select_head<DT, kT>(meta, absmax, q, blk_arr, kblocks, Hkv, G, D, l_cpu, approx, astride,
                    eps_scale, sel_bits, sel_words, cand_keys, cand_ids, cand_stride, keys_cap);
    SEL_MARK(11);
    if (wl.boxes == nullptr) return;
    __shared__ int s_last;
    __shared__ int64_t s_wsum[kT + 1];
    const int bg = (int)(blockIdx.x / G);
    __syncthreads();  // this head's bits written; the release below publishes them
    if (threadIdx.x == 0) s_last = atomic_add_acq_rel_gpu(sel_done + bg, 1) == G - 1;
    __syncthreads();
    if (!s_last) return;
    fence_acq_rel_gpu();
    // dynamic smem (keys | histogram | ...) is free now: the per-word box counts
    extern __shared__ __align__(16) unsigned char dsm[];
    int32_t* wcnt = reinterpret_cast<int32_t*>(dsm);
    SEL_MARK(8);
    worklist_group(wl, bg, wcnt, s_wsum);
    worklist_publish(wl, (int)(gridDim.x / G));
    SEL_MARK(9);
}

}  // namespace

double approx_eps_scale(const fx_layout& L);

void launch_select(const fx_layout& L, const void* const meta[4], const float* absmax,
                   const float* q, const int32_t* blk, const int32_t* kblocks,
                   const float* approx, int64_t approx_stride, uint32_t* sel_bits, int sel_words,
                   uint64_t* cand_keys, uint32_t* cand_ids, cudaStream_t s, const WorklistArgs* wl,
                   int32_t* sel_done) {
    MetaPtrs mp{{meta[0], meta[1], meta[2], meta[3]}};
    FX_REQUIRE(level_blocks(L.l_cpu, 16) <= (int64_t)kMaxWords * 32, FX_ERR_INVALID,
               "bad-shape: cpu segment too long for one selection CTA");
    FX_REQUIRE(L.head_dim <= 256, FX_ERR_INVALID, "bad-shape: head_dim must be <= 256");
    const int64_t heads = (int64_t)L.batch * L.kv_heads * L.group_size;
    const int64_t nmax = level_blocks(L.l_cpu, 16);
    const int keys_cap = (int)((std::min<int64_t>(nmax, kSmemKeys) + 3) & ~int64_t(3));
    size_t smem = (size_t)keys_cap * 4 + (size_t)kHistWords * 4 + (size_t)L.head_dim * 8 +
                  (size_t)kSmallCand * 12;
    WorklistArgs w{};
    if (wl) {
        FX_REQUIRE(L.group_size <= 16, FX_ERR_INVALID, "bad-shape: group_size must be <= 16");
        w = *wl;
        smem = std::max(smem, (size_t)kMaxWords * 4);  // fused worklist: the word counts
    }
    const double eps = approx_eps_scale(L);
    // widest CTA whose residency (64 registers per thread; the dynamic smem)
    // still holds every head in one wave
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
            cudaGetLastError();
            sms = 148;
        }
    }
    int nt = kTMin;
    for (int c = kTMax; c > kTMin; c >>= 1) {
        if (nmax < (int64_t)c * 16) continue;  // short heads: the extra warps only add barrier cost
        const int64_t by_regs = 65536 / (c * 64);
        const int64_t by_smem = (int64_t)(227 * 1024) / (int64_t)(smem + 1024);
        if (heads <= (int64_t)sms * std::min(by_regs, by_smem)) {
            nt = c;
            break;
        }
    }
    auto go = [&](auto kern) {
        FX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        launch_pdl(kern, (unsigned)heads, nt, smem, s,
            mp, absmax, q, blk, kblocks, L.kv_heads, L.group_size, L.head_dim, L.l_cpu, approx,
            approx_stride, eps, sel_bits, sel_words, cand_keys, cand_ids, approx_stride, keys_cap,
            w, sel_done);
    };
    if (L.dtype == FX_BF16) {
        if (nt == 1024) go(k_select<FX_BF16, 1024>);
        else if (nt == 512) go(k_select<FX_BF16, 512>);
        else go(k_select<FX_BF16, kTMin>);
    } else {
        if (nt == 1024) go(k_select<FX_F32, 1024>);
        else if (nt == 512) go(k_select<FX_F32, 512>);
        else go(k_select<FX_F32, kTMin>);
    }
    FX_CUDA(cudaGetLastError());
}

#ifdef FX_TRACE
extern "C" FX_API int fx_debug_sel_trace(long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_sel_trace, sizeof(long long) * n) == cudaSuccess ? 0 : -2;
}
extern "C" FX_API int fx_debug_sel_trace_clear(void) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_sel_trace) != cudaSuccess) return -2;
    return cudaMemset(p, 0, sizeof(g_sel_trace)) == cudaSuccess ? 0 : -2;
}
#endif

}  // namespace fx
