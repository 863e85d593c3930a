// fx_attend.cu -- K3 + K4: block-sparse GQA split-K decode attention with the
// fused log-sum-exp merge.
//
// Reference semantics (per head h of a group, scheduler.cpp:78-96):
//   acc = default_kv_attention(q, cache)          attention.cpp:143-151
//   acc = merge_into(acc, sparse_attention(q, cache, topk(...)))
// i.e. exact softmax attention of q over  sink + local + new  and the
// selected cpu-segment blocks, merged by LSE (attention.cpp:89-104).
//
// Work decomposition.  The worklist (fx_worklist.cuh; fused into k_select)
// lays every (b, g) out as a list of 16-row "boxes" (defaults first, then the
// union of the group's selected blocks) with a G-bit head mask per box.
//
// k_attend_tma (bf16, D in {64, 128}, G <= 8) is fed by a unit queue: as soon
// as a group's boxes exist, the worklist publishes them as units of
// kUnitBoxes boxes (epoch-tagged flag words, release/acquire), and the
// persistent CTAs -- resident while the selection of later groups is still
// running -- claim units in publication order with one atomic each.  A
// single-unit group is written final; otherwise every unit leaves an (o, lse)
// partial and k_merge_units (launched behind this kernel, PDL) folds them in
// unit order, so the result does not depend on which CTA ran what.  Dynamic
// claiming also balances the per-SM bandwidth differences at the end.
//   warp 4        producer: claims units, one 3-D TMA per 16-row box and
//                 tensor (SWIZZLE_128B) into a kStages-deep ring of 8-box
//                 tiles plus a 1-D bulk copy of the unit's q rows, mbarrier
//                 completion;
//   warp 5        epilogue: combines the consumer warps' states of a unit,
//                 writes the partial / final output -- off the consumers'
//                 path;
//   warps 0..3    consumers: two boxes each per 8-box tile;
//                 S^T[16 tok x 8 heads] = K . Q^T  (mma.sync m16n8k16 bf16,
//                 q split hi+lo so q keeps ~16 mantissa bits),
//                 online softmax in f32 (exp2 domain),
//                 O^T[D x 8] += V^T . P^T (P^T transposed in-register with
//                 movmatrix, V^T via ldmatrix.trans).
//   G <= 8 heads fill the n8 side of the MMA, so one MMA serves all heads of
//   the group and K/V are read from HBM exactly once per (b, g, token).
//   tcgen05 needs M >= 64 rows of one operand; with one query token per head
//   the widest dense side is G <= 8, so the legacy m16n8k16 shape is the
//   right tool here (the kernel is HBM-bound: ~4 flop/byte).
// k_attend_generic: any dtype (f32 path of config 1), any G <= 16, D <= 256,
//   and index lists (the per-query reference API); CUDA-core f32 math; the
//   global box sequence split into equal contiguous ranges over a persistent
//   grid, runs cut by a range end merged by their last contributor.
#include <cuda.h>

#include "fx_common.cuh"

namespace fx {
namespace {

constexpr int kCWarps = 4;      // consumer warps
constexpr int kBPW = 2;         // boxes per consumer warp per tile (32 tokens: 2 MMA m-tiles)
constexpr int kTileBoxes = kCWarps * kBPW;  // boxes per pipeline tile
constexpr int kStages = 3;      // 64 KB stages (K + V of 8 boxes)
// TMA kernel warps: kCWarps consumers + one producer
constexpr int kProducer = kCWarps, kTmaThreads = (kCWarps + 1) * 32;
constexpr int kGen = 128;       // threads of the generic kernel
constexpr int kGenMaxG = 16;
constexpr int kGenMaxD = 256;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kLog2e = 1.4426950408889634f;
// tile flags: first / last tile of a run; the run lies wholly in this CTA
// (its partial is the final output); end of the CTA's range
constexpr int F_FIRST = 1, F_LAST = 2, F_END = 4, F_SOLE = 8;

struct TileHdr {
    int32_t bg, flags, nb;
    int32_t u, c, nun;  // unit id, its index in the group, the group's unit count
    int32_t unused[2];
    Box box[kTileBoxes];
};

struct View {
    int n_bg, Hkv, G, D;
    int64_t l_cap;
    const void* k;
    const void* v;
    const float* q;
    const uint32_t* idx;
    const Box* boxes;
    int64_t box_stride;
    const int32_t* bg_start;  // global run starts (used when n_bg > kMaxPrefix)
    const int32_t* bg_count;  // per-(b, g) box counts (run starts rebuilt in smem)
    int pad;  // virtual boxes ending each run in the split (never loaded)
    float* part_o;
    float* part_lse;
    int32_t* bg_done;  // [n_bg] contributor counters, zeroed before the launch
    float* o;
    float* lse;
};

__device__ __forceinline__ int cta_of(int64_t x, int64_t NB, int grid) {
    return (int)(((x + 1) * grid - 1) / NB);
}
// Warp-cooperative find_bg: every lane counts the run starts <= x over a
// strided slice (independent loads, all in flight at once), then a warp sum.
// One L2 round trip instead of log2(n_bg) dependent ones.
__device__ __forceinline__ int find_bg_warp(const int32_t* start, int n_bg, int64_t x, int lane) {
    int cnt = 0;
    for (int j = 1 + lane; j < n_bg; j += 32) cnt += start[j] <= x ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    return cnt;  // start[] is non-decreasing and start[0] = 0 <= x
}
__device__ __forceinline__ int find_bg(const int32_t* start, int n_bg, int64_t x) {
    int lo = 0, hi = n_bg - 1;  // largest bg with start[bg] <= x
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (start[mid] <= x) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Whether CTA c of the generic kernel's static split has any box (with fewer
// boxes than CTAs some ranges are empty and leave no partial).
__device__ __forceinline__ bool cta_nonempty(int c, int64_t NB, int grid) {
    return NB * c / grid < NB * (c + 1) / grid;
}

constexpr int kMaxPrefix = kMaxRunPrefix;  // (b, g) runs whose starts are rebuilt in smem

// Run starts of the global box sequence: exclusive prefix of (box count +
// pad) over the (b, g) runs, rebuilt by every CTA in smem from the
// worklist's counts (one coalesced round trip), so the worklist publishes no
// grid-wide prefix and the producer's run walk never touches global memory.
// Larger batches fall back to the worklist's global bg_start.
__device__ const int32_t* run_starts(const View& p, int32_t* s_start, int* wtmp, int t, int nt) {
    if (p.n_bg > kMaxPrefix) return p.bg_start;
    const int lane = t & 31, warp = t >> 5, nw = nt >> 5;
    int carry = 0;
    for (int c0 = 0; c0 < p.n_bg; c0 += nt) {
        const int i = c0 + t;
        const int v = i < p.n_bg ? __ldcg(p.bg_count + i) + p.pad : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wtmp[warp] = x;
        __syncthreads();
        int off = carry, tot = 0;
        for (int w = 0; w < nw; ++w) {
            if (w < warp) off += wtmp[w];
            tot += wtmp[w];
        }
        if (i < p.n_bg) s_start[i] = off + x - v;
        __syncthreads();
        carry += tot;
    }
    if (t == 0) s_start[p.n_bg] = carry;
    __syncthreads();
    return s_start;
}

// Runs with no real boxes (a context-parallel shard whose group selected
// nothing there and holds no default rows; a streaming group without defaults)
// reach no tile.  Their output is the merge identity -- o = 0, lse = -inf
// (merge_into with an empty partial, attention.cpp:89-104) -- written by the
// CTA whose range holds the run's first (virtual) box.
__device__ void write_empty_runs(const View& p, const int32_t* starts, int64_t r0, int64_t r1,
                                 int t, int nt) {
    if (r0 >= r1) return;
    for (int bg = find_bg(starts, p.n_bg, r0); bg < p.n_bg && starts[bg] < r1; ++bg) {
        if (starts[bg] < r0 || starts[bg + 1] - starts[bg] > p.pad) continue;
        const int64_t head0 = (int64_t)(bg / p.Hkv) * p.Hkv * p.G + (int64_t)(bg % p.Hkv) * p.G;
        for (int i = t; i < p.G * p.D; i += nt) p.o[head0 * p.D + i] = 0.f;
        if (p.lse)
            for (int h = t; h < p.G; h += nt) p.lse[head0 + h] = -INFINITY;
    }
}


// ---------------------------------------------------------------------------
// TMA + mma.sync kernel, fed by the unit queue
// ---------------------------------------------------------------------------
// Tensor maps of K (0) and V (1) viewed 3-D {64 cols, rows, D/64 chunks}
// (strides: row D*2 B, chunk 128 B); box = 16 rows x all chunks, 128-B swizzle.
struct KvMaps {
    CUtensorMap box[2];
};

// One attention unit = up to kUnitBoxes consecutive boxes of one (b, g)
// (fx_worklist.cuh publish_units).  A unit of a single-unit group writes the
// final (o, lse); otherwise one (o, lse) partial per unit, folded by
// k_merge_units.
struct QView {
    int n_bg, Hkv, G;
    int64_t l_cap;
    const float* q;
    const Box* boxes;
    int64_t box_stride;
    const int32_t* bg_count;
    UnitQueue uq;      // ctl zeroed by k_prepare
    float* part_o;     // [unit][G][D]
    float* part_lse;   // [unit][G] (natural log)
    float* o;
    float* lse;
};

constexpr int kEpi = kCWarps + 1;  // epilogue warp: combines a unit's consumer states
constexpr int kQThreads = (kCWarps + 2) * 32;

template <int D>
struct TmaCfg {
    static constexpr int NCH = D * 2 / 128;            // 128-byte column chunks per row
    static constexpr int BOX_BYTES = kBoxRows * 128;   // one TMA box = 2 KB
    static constexpr int UNIT_BYTES = NCH * BOX_BYTES;  // one box across all column chunks
    static constexpr int KV_BYTES = kTileBoxes * UNIT_BYTES;
    static constexpr int STAGE_BYTES = 2 * KV_BYTES;
    static constexpr int NT = D / 16;                  // k-steps (QK) and m-tiles (PV)
    static constexpr int WO_LD = D + 4;
    static constexpr int QB_BYTES = 8 * D * 4;         // the unit's q rows (f32, G <= 8)
    static constexpr size_t TILES = (size_t)kStages * STAGE_BYTES;
    static constexpr size_t QB = TILES;
    static constexpr size_t HDR = QB + (size_t)kStages * QB_BYTES;
    static constexpr size_t BAR = HDR + kStages * sizeof(TileHdr);
    static constexpr size_t SINFO = BAR + (2 * kStages + 2) * sizeof(uint64_t);
    static constexpr size_t WO = SINFO + 32;
    static constexpr size_t WM = WO + (size_t)kCWarps * 8 * WO_LD * sizeof(float);
    static constexpr size_t WL = WM + kCWarps * 8 * sizeof(float);
    static constexpr size_t TOTAL = WL + kCWarps * 8 * sizeof(float) + 1024;  // + align slack
};

constexpr int kMergeThreads = 128;  // the narrowest unit-merge CTA (launch_unit_merge picks 128 / 256 / 512)
// Fold the partials at slots [base, base + nun) of head h into (o, lse): the
// max of the slot LSEs, then each thread owns one float4 column of a fixed
// subset of the slots (eight slots' loads in flight), the subsets combined in
// a fixed order: deterministic.  All kMergeThreads threads.
template <int NT>
__device__ void merge_slots(int G, int D, int h, int base, int nun, const float* __restrict__ part_o,
                            const float* __restrict__ part_lse, float* __restrict__ o_dst,
                            float* __restrict__ lse_dst) {
    const int t = threadIdx.x;
    const int VP = D / 4;                   // float4 columns of the head
    const int S = NT / VP;       // slot subsets (D <= 512)
    __shared__ float s_wm[NT / 32];
    __shared__ float4 s_acc[NT];
    __shared__ float s_den[NT];
    float m = -INFINITY;
    for (int i = t; i < nun; i += NT) m = fmaxf(m, __ldg(part_lse + (int64_t)(base + i) * G + h));
    m = warp_max(m);
    if ((t & 31) == 0) s_wm[t >> 5] = m;
    __syncthreads();
    float M = s_wm[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) M = fmaxf(M, s_wm[w]);
    const int v = t % VP, sub = t / VP;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float den = 0.f;
    if (sub < S) {
        constexpr int kIn = 8;
        for (int i0 = sub; i0 < nun; i0 += S * kIn) {
            float4 x[kIn];
            float l[kIn];
#pragma unroll
            for (int j = 0; j < kIn; ++j) {
                const int i = i0 + j * S;
                const int64_t slot = (int64_t)(base + i) * G + h;
                l[j] = i < nun ? __ldg(part_lse + slot) : -INFINITY;
                x[j] = i < nun ? __ldg(reinterpret_cast<const float4*>(part_o + slot * D) + v)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int j = 0; j < kIn; ++j) {
                if (l[j] == -INFINITY) continue;
                const float w = __expf(l[j] - M);
                den += w;
                acc.x += w * x[j].x;
                acc.y += w * x[j].y;
                acc.z += w * x[j].z;
                acc.w += w * x[j].w;
            }
        }
    }
    s_acc[t] = acc;
    s_den[t] = den;
    __syncthreads();
    if (sub != 0) return;
    for (int k = 1; k < S; ++k) {
        const float4 a = s_acc[k * VP + v];
        acc.x += a.x;
        acc.y += a.y;
        acc.z += a.z;
        acc.w += a.w;
        den += s_den[k * VP + v];
    }
    const float inv = den > 0.f ? 1.f / den : 0.f;
    *reinterpret_cast<float4*>(o_dst + v * 4) = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    if (v == 0 && lse_dst) *lse_dst = den > 0.f ? M + __logf(den) : -INFINITY;
}

// Merge of the unit partials of every multi-unit group (attention.cpp:89-104
// across the units, in unit order): one 128-thread CTA per (b, g, head),
// launched behind the attention kernel (PDL) -- small CTAs, so every group's
// heads merge at once even with thousands of groups (C4).
template <int NT>
__global__ void __launch_bounds__(NT) k_merge_units(int Hkv, int G, int D,
                                                              const int32_t* __restrict__ bg_count,
                                                              const int32_t* __restrict__ ubase,
                                                              const float* __restrict__ part_o,
                                                              const float* __restrict__ part_lse,
                                                              float* __restrict__ o, float* __restrict__ lse) {
    pdl_wait();
    pdl_trigger();
    const int bg = blockIdx.x, h = blockIdx.y;
    const int total = __ldg(bg_count + bg);
    const int nun = total > 0 ? (total + kUnitBoxes - 1) / kUnitBoxes : 1;
    if (nun <= 1) return;  // written final by the attention kernel
    const int b = bg / Hkv, g = bg % Hkv;
    const int64_t hd = (int64_t)b * Hkv * G + (int64_t)g * G + h;
    merge_slots<NT>(G, D, h, __ldg(ubase + bg), nun, part_o, part_lse, o + hd * D, lse ? lse + hd : nullptr);
}

#ifdef FX_TRACE  // profiling build only: per-CTA start/end time, units, tiles
__device__ long long g_trace[12 * 2048];
__device__ long long g_gtrace[8 * 2048];  // generic kernel: per-CTA phase times
__device__ __forceinline__ long long globaltimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// Warp roles: 0..3 consumers (MMA), 4 producer (claims units, TMA), 5
// epilogue.  No griddepcontrol.wait: the kernel reads only the worklist's
// boxes (ordered by the acquire of the unit words), q and K/V; it becomes
// resident once every selection CTA has started, and those were launched
// after the scorer passed its wait on k_prepare (appended rows, zeroed
// counters), so every earlier write of the step is visible.
template <int D>
__global__ void __launch_bounds__(kQThreads, 1) k_attend_tma(const __grid_constant__ KvMaps maps,
                                                      const QView p) {
    if (threadIdx.x == kProducer * 32) {
        tma_prefetch_desc(&maps.box[0]);
        tma_prefetch_desc(&maps.box[1]);
    }
    pdl_trigger();
    using C = TmaCfg<D>;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    TileHdr* hdr = reinterpret_cast<TileHdr*>(smem + C::HDR);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR);
    uint64_t* empty = full + kStages;
    uint64_t* sfull = empty + kStages;  // staging (wO / wm / wl) holds a finished unit
    uint64_t* sempty = sfull + 1;       // ... and is free again
    int* sinfo = reinterpret_cast<int*>(smem + C::SINFO);  // bg, u, c, nun, flags
    float* wO = reinterpret_cast<float*>(smem + C::WO);
    float* wm = reinterpret_cast<float*>(smem + C::WM);
    float* wl = reinterpret_cast<float*>(smem + C::WL);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, kCWarps);
        }
        mbar_init(sfull, kCWarps);
        mbar_init(sempty, 1);
        fence_mbar_init();
    }
    __syncthreads();
#ifdef FX_TRACE
    if (tid == 0) {
        g_trace[blockIdx.x * 12 + 0] = globaltimer();
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_trace[blockIdx.x * 12 + 11] = smid;
    }
#endif

    if (warp == kProducer) {
        // ------------------------------ producer ------------------------------
        // Units are claimed one ahead: while unit `cur` streams, the next
        // claim's flag word, box count and box descriptors are fetched.
        constexpr int UPL = kUnitBoxes / 32;  // box descriptors per lane
        struct Unit {
            int u, bg, c, total;
            Box wb[UPL];  // this lane's box descriptors (boxes lane, lane + 32, ...)
        };
        int st = 0;
        uint32_t ph = 0;
#ifdef FX_TRACE
        long long p_wait = 0;
#endif
        // 1 = fetched, 0 = not published yet (block == false), -1 = queue drained
        auto fetch = [&](int u, bool block, Unit& f) -> int {
            uint64_t wd = 0;
            int state = 0;
            if (lane == 0) {
                while (true) {
                    wd = ld_acquire_gpu_u64(p.uq.words + u);
                    if ((uint32_t)(wd >> 32) == p.uq.epoch) {
                        state = 1;
                        break;
                    }
                    if (ld_acquire_gpu_s32(p.uq.ctl + 1) == p.n_bg && u >= ld_relaxed_gpu_s32(p.uq.ctl + 0)) {
                        state = -1;
                        break;
                    }
                    if (!block) break;
                    __nanosleep(64);
                }
            }
            __syncwarp();  // lane 0's acquire orders the other lanes' box loads
            state = __shfl_sync(0xffffffffu, state, 0);
            if (state != 1) return state;
            const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)wd, 0);
            f.u = u;
            f.bg = (int)(lo >> kUnitIdxBits);
            f.c = (int)(lo & ((1u << kUnitIdxBits) - 1u));
            f.total = __ldcg(p.bg_count + f.bg);
            const int x0 = f.c * kUnitBoxes, x1 = min(x0 + kUnitBoxes, f.total);
#pragma unroll
            for (int k = 0; k < UPL; ++k) {
                f.wb[k] = Box{0, 0, 0};
                if (x0 + lane + 32 * k < x1) {
                    const int2 r = __ldcg(reinterpret_cast<const int2*>(p.boxes + (int64_t)f.bg * p.box_stride + x0 +
                                                                       lane + 32 * k));
                    f.wb[k].row = r.x;
                    f.wb[k].n = (uint16_t)(r.y & 0xffff);
                    f.wb[k].mask = (uint16_t)((uint32_t)r.y >> 16);
                }
            }
            return 1;
        };
        auto claim = [&]() {
            int u = 0;
            if (lane == 0) u = atomicAdd(p.uq.ctl + 2, 1);
            return __shfl_sync(0xffffffffu, u, 0);
        };
        static_assert(kUnitBoxes % 32 == 0 && kTileBoxes <= 32 && 32 % kTileBoxes == 0,
                      "whole descriptor sets per lane; a tile's boxes in one set");
        Unit cur, nxt;
#ifdef FX_TRACE
        long long pw0 = globaltimer();
#endif
        int have = fetch(claim(), true, cur);
#ifdef FX_TRACE
        p_wait += globaltimer() - pw0;
#endif
        while (have == 1) {
            const int un = claim();
            int nstate = 0;
            const int nun = cur.total > 0 ? (cur.total + kUnitBoxes - 1) / kUnitBoxes : 1;
            const int x0 = cur.c * kUnitBoxes, x1 = min(x0 + kUnitBoxes, cur.total);
            const int b = cur.bg / p.Hkv, g = cur.bg % p.Hkv;
            const float* qsrc = p.q + ((int64_t)b * p.Hkv * p.G + (int64_t)g * p.G) * D;
            const int64_t base = (int64_t)cur.bg * p.l_cap;
            int x = x0;
            bool first = true;
            do {
                const int nb = max(0, min(kTileBoxes, x1 - x));
                Box bx[kTileBoxes];
                // the tile's descriptor set (warp-uniform: tiles are 8-aligned in the unit)
                Box ws = cur.wb[0];
#pragma unroll
                for (int k = 1; k < UPL; ++k)
                    if (((x - x0) >> 5) == k) ws = cur.wb[k];
#pragma unroll
                for (int i = 0; i < kTileBoxes; ++i) {
                    const int src = (x - x0 + i) & 31;
                    bx[i].row = __shfl_sync(0xffffffffu, ws.row, src);
                    const uint32_t nm = __shfl_sync(0xffffffffu, (uint32_t)ws.n | ((uint32_t)ws.mask << 16), src);
                    bx[i].n = (uint16_t)(nm & 0xffffu);
                    bx[i].mask = (uint16_t)(nm >> 16);
                }
                if (lane == 0) {
                    mbar_wait(empty + st, ph ^ 1u);
                    TileHdr& H = hdr[st];
                    const bool last = x + nb >= x1;
                    H.bg = cur.bg;
                    H.nb = nb;
                    H.u = cur.u;
                    H.c = cur.c;
                    H.nun = nun;
                    H.flags = (first ? F_FIRST : 0) | (last ? F_LAST | (nun == 1 ? F_SOLE : 0) : 0);
#pragma unroll
                    for (int i = 0; i < kTileBoxes; ++i) H.box[i] = bx[i];
                    unsigned char* kt = smem + (size_t)st * C::STAGE_BYTES;
                    unsigned char* vt = kt + C::KV_BYTES;
                    const uint32_t qbytes = first ? (uint32_t)(p.G * D * 4) : 0u;
                    mbar_arrive_expect_tx(full + st, (uint32_t)(nb * 2 * C::NCH * C::BOX_BYTES) + qbytes);
                    if (first) bulk_g2s(smem + C::QB + (size_t)st * C::QB_BYTES, qsrc, qbytes, full + st);
                    for (int i = 0; i < nb; ++i) {
                        const int row0 = (int)(base + bx[i].row);
                        tma_load_3d(kt + i * C::UNIT_BYTES, &maps.box[0], full + st, 0, row0, 0);
                        tma_load_3d(vt + i * C::UNIT_BYTES, &maps.box[1], full + st, 0, row0, 0);
                    }
                }
                __syncwarp();
                first = false;
                x += nb;
                if (++st == kStages) {
                    st = 0;
                    ph ^= 1u;
                }
                // the next unit's descriptors, while this unit's tiles are in flight
                if (nstate == 0) nstate = fetch(un, false, nxt);
            } while (x < x1);
#ifdef FX_TRACE
            pw0 = globaltimer();
#endif
            if (nstate == 0) nstate = fetch(un, true, nxt);
#ifdef FX_TRACE
            p_wait += globaltimer() - pw0;
#endif
            have = nstate;
            cur = nxt;
        }
        if (lane == 0) {
            mbar_wait(empty + st, ph ^ 1u);
#ifdef FX_TRACE
            g_trace[blockIdx.x * 12 + 7] = p_wait;
#endif
            hdr[st].flags = F_END;
            mbar_arrive(full + st);
        }
        return;
    }

    if (warp == kEpi) {
        // ------------------------------ epilogue ------------------------------
        uint32_t sph = 0;
        const int G = p.G;
        while (true) {
            mbar_wait(sfull, sph);
            const int bg = sinfo[0], u = sinfo[1], flags = sinfo[4];
            if (flags & F_END) break;
            const bool sole = flags & F_SOLE;
            const int64_t head0 = sole ? (int64_t)(bg / p.Hkv) * p.Hkv * G + (int64_t)(bg % p.Hkv) * G
                                       : (int64_t)u * G;
            float* dst_o = sole ? p.o : p.part_o;
            float* dst_l = sole ? p.lse : p.part_lse;
            // the four consumer warps' states of the unit -> one (o, lse): lane
            // h < G forms head h's warp weights f_w / den once (into wl), then
            // every lane combines float4 columns
            if (lane < G) {
                float M = -INFINITY;
#pragma unroll
                for (int w = 0; w < kCWarps; ++w) M = fmaxf(M, wm[w * 8 + lane]);
                float hf[kCWarps], den = 0.f;
#pragma unroll
                for (int w = 0; w < kCWarps; ++w) {
                    const float mw = wm[w * 8 + lane];
                    hf[w] = (M == -INFINITY || mw == -INFINITY) ? 0.f : exp2f(mw - M);
                    den += hf[w] * wl[w * 8 + lane];
                }
                const float inv = den > 0.f ? 1.f / den : 0.f;
#pragma unroll
                for (int w = 0; w < kCWarps; ++w) wl[w * 8 + lane] = hf[w] * inv;
                if (dst_l) dst_l[head0 + lane] = den > 0.f ? (M + log2f(den)) * kLn2 : -INFINITY;
            }
            __syncwarp();
            for (int e = lane; e < G * D / 4; e += 32) {
                const int h = e * 4 / D, d = e * 4 % D;
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int w = 0; w < kCWarps; ++w) {
                    const float f = wl[w * 8 + h];
                    const float4 x = *reinterpret_cast<const float4*>(wO + ((size_t)w * 8 + h) * C::WO_LD + d);
                    acc.x += f * x.x;
                    acc.y += f * x.y;
                    acc.z += f * x.z;
                    acc.w += f * x.w;
                }
                float* dst = dst_o + (head0 + h) * D + d;
                dst[0] = acc.x;
                dst[1] = acc.y;
                dst[2] = acc.z;
                dst[3] = acc.w;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(sempty);
            sph ^= 1u;
        }
#ifdef FX_TRACE
        if (lane == 0) g_trace[blockIdx.x * 12 + 8] = globaltimer();
#endif
        return;
    }

    // ------------------------------- consumers -------------------------------
    const int G = p.G;
    const float sl2 = rsqrtf((float)D) * kLog2e;
    const int tok0 = lane >> 2, h0 = 2 * (lane & 3);
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    float O[C::NT][4];
    uint32_t qh[C::NT][2], ql[C::NT][2];
#pragma unroll
    for (int i = 0; i < C::NT; ++i) O[i][0] = O[i][1] = O[i][2] = O[i][3] = 0.f;
    int st = 0;
    uint32_t ph = 0, sph = 0;
#ifdef FX_TRACE
    int units = 0, tiles = 0;
    long long t_wait = 0, tw0 = 0;
#endif
    while (true) {
#ifdef FX_TRACE
        tw0 = globaltimer();
#endif
        mbar_wait(full + st, ph);
#ifdef FX_TRACE
        t_wait += globaltimer() - tw0;
#endif
        const int flags = hdr[st].flags;
        if (flags & F_END) {
#ifdef FX_TRACE
            if (tid == 0) {
                g_trace[blockIdx.x * 12 + 1] = globaltimer();
                g_trace[blockIdx.x * 12 + 2] = units;
                g_trace[blockIdx.x * 12 + 3] = tiles;
                g_trace[blockIdx.x * 12 + 4] = t_wait;
            }
#endif
            break;
        }
#ifdef FX_TRACE
        ++tiles;
        units += (flags & F_FIRST) ? 1 : 0;
#endif
        // everything the unit's end needs from the header is read before this
        // warp releases the stage (the producer then refills hdr[st])
        const int bg = hdr[st].bg, nb = hdr[st].nb;
        const int u = hdr[st].u, c = hdr[st].c, nun = hdr[st].nun;
        const int i0 = warp * kBPW;  // this warp's boxes: i0, i0 + 1
        const Box bxa = hdr[st].box[i0];
        const Box bxb = hdr[st].box[i0 + 1];
        if (flags & F_FIRST) {
            // the unit's q rows arrived with this stage: split into bf16 hi + lo
            const float* qs = reinterpret_cast<const float*>(smem + C::QB + (size_t)st * C::QB_BYTES);
            const int hq = lane >> 2;
#pragma unroll
            for (int j = 0; j < C::NT; ++j) {
                const int d0 = 16 * j + 2 * (lane & 3);
                float2 x0 = make_float2(0.f, 0.f), x1 = make_float2(0.f, 0.f);
                if (hq < G) {
                    x0 = *reinterpret_cast<const float2*>(qs + hq * D + d0);
                    x1 = *reinterpret_cast<const float2*>(qs + hq * D + d0 + 8);
                }
                const float a0 = __bfloat162float(__float2bfloat16_rn(x0.x));
                const float a1 = __bfloat162float(__float2bfloat16_rn(x0.y));
                const float a2 = __bfloat162float(__float2bfloat16_rn(x1.x));
                const float a3 = __bfloat162float(__float2bfloat16_rn(x1.y));
                qh[j][0] = pack_bf16(a0, a1);
                qh[j][1] = pack_bf16(a2, a3);
                ql[j][0] = pack_bf16(x0.x - a0, x0.y - a1);
                ql[j][1] = pack_bf16(x1.x - a2, x1.y - a3);
            }
            m0 = m1 = -INFINITY;
            l0 = l1 = 0.f;
#pragma unroll
            for (int i = 0; i < C::NT; ++i) O[i][0] = O[i][1] = O[i][2] = O[i][3] = 0.f;
        }
#ifdef FX_ATTEND_NO_MATH  // profiling variant: data delivery only
        if (false) {
#else
        if (i0 < nb) {
#endif
            // two boxes (32 tokens) per warp: independent MMA chains interleave
            const bool two = i0 + 1 < nb;  // warp-uniform
            constexpr uint32_t csa = C::BOX_BYTES, csb = C::BOX_BYTES;  // chunk stride in a box
            const uint32_t ka = smem_u32(smem + (size_t)st * C::STAGE_BYTES) + i0 * C::UNIT_BYTES;
            const uint32_t kb2 = ka + C::UNIT_BYTES;
            float sha[4] = {0.f, 0.f, 0.f, 0.f}, sla[4] = {0.f, 0.f, 0.f, 0.f};
            float shb[4] = {0.f, 0.f, 0.f, 0.f}, slb[4] = {0.f, 0.f, 0.f, 0.f};
            {
                const int r = (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
                for (int j = 0; j < C::NT; ++j) {
                    const int u = ((j & 3) << 1) + (lane >> 4);
                    const uint32_t off = r * 128 + ((u ^ (r & 7)) << 4);
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4(ka + (j >> 2) * csa + off, a0, a1, a2, a3);
                    mma_bf16_16816(sha, a0, a1, a2, a3, qh[j][0], qh[j][1]);
                    mma_bf16_16816(sla, a0, a1, a2, a3, ql[j][0], ql[j][1]);
                    if (two) {
                        ldsm_x4(kb2 + (j >> 2) * csb + off, a0, a1, a2, a3);
                        mma_bf16_16816(shb, a0, a1, a2, a3, qh[j][0], qh[j][1]);
                        mma_bf16_16816(slb, a0, a1, a2, a3, ql[j][0], ql[j][1]);
                    }
                }
            }
            // V fragments into registers now, so the stage goes back to the
            // producer before the softmax and the PV products (it refills
            // the ring a few hundred cycles earlier every tile)
            uint32_t vfa[C::NT][4], vfb[C::NT][4];
            {
                const uint32_t va = ka + C::KV_BYTES, vb2 = kb2 + C::KV_BYTES;
                const int mi = lane >> 3;
                const int r = (lane & 7) + (mi >> 1) * 8;
#pragma unroll
                for (int i = 0; i < C::NT; ++i) {
                    const int u = ((i & 3) << 1) + (mi & 1);
                    const uint32_t off = r * 128 + ((u ^ (r & 7)) << 4);
                    ldsm_x4_t(va + (i >> 2) * csa + off, vfa[i][0], vfa[i][1], vfa[i][2], vfa[i][3]);
                    if (two) ldsm_x4_t(vb2 + (i >> 2) * csb + off, vfb[i][0], vfb[i][1], vfb[i][2], vfb[i][3]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + st);
            // scores (log2 domain), masked by token validity and head selection
            float s[2][4];
            {
                const Box bxs[2] = {bxa, bxb};
                const float* hiv[2] = {sha, shb};
                const float* lov[2] = {sla, slb};
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const bool live = q == 0 || two;
                    const bool v0 = live && tok0 < bxs[q].n, v1 = live && tok0 + 8 < bxs[q].n;
                    const bool e0 = (bxs[q].mask >> h0) & 1, e1 = (bxs[q].mask >> (h0 + 1)) & 1;
                    s[q][0] = (v0 && e0) ? (hiv[q][0] + lov[q][0]) * sl2 : -INFINITY;
                    s[q][1] = (v0 && e1) ? (hiv[q][1] + lov[q][1]) * sl2 : -INFINITY;
                    s[q][2] = (v1 && e0) ? (hiv[q][2] + lov[q][2]) * sl2 : -INFINITY;
                    s[q][3] = (v1 && e1) ? (hiv[q][3] + lov[q][3]) * sl2 : -INFINITY;
                }
            }
            float c0 = fmaxf(fmaxf(s[0][0], s[0][2]), fmaxf(s[1][0], s[1][2]));
            float c1 = fmaxf(fmaxf(s[0][1], s[0][3]), fmaxf(s[1][1], s[1][3]));
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                c0 = fmaxf(c0, __shfl_xor_sync(0xffffffffu, c0, o));
                c1 = fmaxf(c1, __shfl_xor_sync(0xffffffffu, c1, o));
            }
            const float n0 = fmaxf(m0, c0), n1 = fmaxf(m1, c1);
            const float b0 = n0 == -INFINITY ? 0.f : n0, b1 = n1 == -INFINITY ? 0.f : n1;
            const float al0 = n0 == -INFINITY ? 1.f : exp2f(m0 - n0);
            const float al1 = n1 == -INFINITY ? 1.f : exp2f(m1 - n1);
            uint32_t x[2][2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                x[q][0] = pack_bf16(exp2f(s[q][0] - b0), exp2f(s[q][1] - b1));
                x[q][1] = pack_bf16(exp2f(s[q][2] - b0), exp2f(s[q][3] - b1));
            }
            l0 = l0 * al0 + ((bf16lo_to_f(x[0][0]) + bf16lo_to_f(x[0][1])) +
                             (bf16lo_to_f(x[1][0]) + bf16lo_to_f(x[1][1])));
            l1 = l1 * al1 + ((bf16hi_to_f(x[0][0]) + bf16hi_to_f(x[0][1])) +
                             (bf16hi_to_f(x[1][0]) + bf16hi_to_f(x[1][1])));
            m0 = n0;
            m1 = n1;
            const uint32_t pa0 = movmatrix_t(x[0][0]), pa1 = movmatrix_t(x[0][1]);
            const uint32_t pb0 = movmatrix_t(x[1][0]), pb1 = movmatrix_t(x[1][1]);
#pragma unroll
            for (int i = 0; i < C::NT; ++i) {
                O[i][0] *= al0;
                O[i][1] *= al1;
                O[i][2] *= al0;
                O[i][3] *= al1;
                mma_bf16_16816(O[i], vfa[i][0], vfa[i][1], vfa[i][2], vfa[i][3], pa0, pa1);
                if (two) mma_bf16_16816(O[i], vfb[i][0], vfb[i][1], vfb[i][2], vfb[i][3], pb0, pb1);
            }
        } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + st);
        }
        if (flags & F_LAST) {
            // ---- unit end: hand this warp's state to the epilogue warp ----
            float t0 = l0, t1 = l1;
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                t0 += __shfl_xor_sync(0xffffffffu, t0, o);
                t1 += __shfl_xor_sync(0xffffffffu, t1, o);
            }
            mbar_wait(sempty, sph ^ 1u);
            if (lane < 4) {
                wm[warp * 8 + h0] = m0;
                wm[warp * 8 + h0 + 1] = m1;
                wl[warp * 8 + h0] = t0;
                wl[warp * 8 + h0 + 1] = t1;
            }
            float* wo = wO + (size_t)warp * 8 * C::WO_LD;
#pragma unroll
            for (int i = 0; i < C::NT; ++i) {
                const int d0 = 16 * i + tok0;
                wo[h0 * C::WO_LD + d0] = O[i][0];
                wo[(h0 + 1) * C::WO_LD + d0] = O[i][1];
                wo[h0 * C::WO_LD + d0 + 8] = O[i][2];
                wo[(h0 + 1) * C::WO_LD + d0 + 8] = O[i][3];
            }
            if (warp == 0 && lane == 0) {
                sinfo[0] = bg;
                sinfo[1] = u;
                sinfo[2] = c;
                sinfo[3] = nun;
                sinfo[4] = flags;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(sfull);
            sph ^= 1u;
        }
        if (++st == kStages) {
            st = 0;
            ph ^= 1u;
        }
    }
    // no more units: release the epilogue warp
    mbar_wait(sempty, sph ^ 1u);
    if (warp == 0 && lane == 0) sinfo[4] = F_END;
    __syncwarp();
    if (lane == 0) mbar_arrive(sfull);
}

// ---------------------------------------------------------------------------
// generic kernel (any dtype, CUDA cores)
// ---------------------------------------------------------------------------
// DC / GC > 0: head dim / group size fixed at compile time (the f32 decode
// path of config C1): index arithmetic folds, the loops unroll.
template <int DT, int DC = 0, int GC = 0>
__global__ void __launch_bounds__(kGen, 8) k_attend_generic(const View p) {
#ifdef FX_TRACE
#define GT_MARK(i) if (threadIdx.x == 0 && blockIdx.x < 2048) g_gtrace[blockIdx.x * 8 + (i)] = globaltimer()
#else
#define GT_MARK(i)
#endif
    GT_MARK(0);
    pdl_wait();
    pdl_trigger();
    GT_MARK(1);
    using T = typename Elem<DT>::T;
    extern __shared__ float gsm[];
    const int t = threadIdx.x;
    const int G = GC > 0 ? GC : p.G, D = DC > 0 ? DC : p.D;
    // dynamic smem: Ks[16][D+1] | Vs[16][D] | qs[G][D] | sc[16][G] | mst,lst,alp[G]
    float* Ksm = gsm;
    float* Vsm = Ksm + kBoxRows * (D + 1);
    float* qsm = Vsm + kBoxRows * D;
    float* scm = qsm + G * D;
    float* mst = scm + kBoxRows * G;
    float* lst = mst + G;
    float* alp = lst + G;
#define Ks(r, d) Ksm[(r) * (D + 1) + (d)]
#define Vs(r, d) Vsm[(r) * D + (d)]
#define qs(h, d) qsm[(h) * D + (d)]
#define sc(r, h) scm[(r) * G + (h)]
    __shared__ int32_t s_start[kMaxPrefix + 1];
    __shared__ int s_wtmp[kGen / 32];
    const int32_t* starts = run_starts(p, s_start, s_wtmp, t, kGen);
    GT_MARK(2);
    const int grid = gridDim.x, cta = blockIdx.x;
    const int64_t NB = starts[p.n_bg];
    const int64_t r0 = NB * cta / grid, r1 = NB * (cta + 1) / grid;
    if (r0 >= r1) return;
    const float scale = rsqrtf((float)D);
    float acc[kGenMaxG][2];
    int bg = find_bg(starts, p.n_bg, r0);
    int64_t s_bg = starts[bg], e_bg = starts[bg + 1];
    bool fresh = true;
    // The next box's K / V elements are loaded into registers while this box
    // is computed (the loads of a box are the latency that dominates here).
    // (D <= 128; wider heads load each box synchronously)
    constexpr int EPT = kBoxRows * 128 / kGen;  // elements per thread at D = 128
    const bool pf = D <= 128;
    float nk[EPT], nv[EPT];
    auto box_of = [&](int64_t xx, int bgx, int64_t sbg) { return p.boxes[(int64_t)bgx * p.box_stride + (xx - sbg)]; };
    auto load_box = [&](const Box& bx, int bgx) {
        if (!pf) return;
        const T* kb = static_cast<const T*>(p.k) + (int64_t)bgx * p.l_cap * D;
        const T* vb = static_cast<const T*>(p.v) + (int64_t)bgx * p.l_cap * D;
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int e = t + u * kGen;
            nk[u] = nv[u] = 0.f;
            if (e < kBoxRows * D) {
                const int r = e / D, d = e % D;
                if (r < bx.n) {
                    const int64_t row = p.idx ? (int64_t)p.idx[bx.row + r] : (int64_t)bx.row + r;
                    nk[u] = tofl(kb[row * D + d]);
                    nv[u] = tofl(vb[row * D + d]);
                }
            }
        }
    };
    // (box x, group) of the next real box after x in this range, or -1
    auto next_real = [&](int64_t xx, int bgx, int64_t ebg, int64_t& nx, int& nbg, int64_t& nsbg) {
        nx = xx + 1;
        nbg = bgx;
        int64_t e2 = ebg;
        nsbg = starts[bgx];
        while (nx < r1 && nx >= e2 - p.pad) {
            nx = e2;
            if (nx >= r1) break;
            ++nbg;
            nsbg = starts[nbg];
            e2 = starts[nbg + 1];
        }
        return nx < r1;
    };
    // QK: TPP threads per (token, head) pair split the dot product
    const int pairs = kBoxRows * G;
    const int TPP = pairs >= kGen ? 1 : pairs * 2 >= kGen ? 2 : pairs * 4 >= kGen ? 4 : 8;
    const int DPT = D / TPP;  // contiguous dims per thread of a pair (D % 8 == 0 on this path)
    {   // first real box of the range
        int64_t x0 = r0;
        int b0 = bg;
        int64_t s0 = s_bg, e0 = e_bg;
        while (x0 < r1 && x0 >= e0 - p.pad) {
            x0 = e0;
            if (x0 >= r1) break;
            ++b0;
            s0 = starts[b0];
            e0 = starts[b0 + 1];
        }
        if (x0 < r1) load_box(box_of(x0, b0, s0), b0);
    }
    for (int64_t x = r0; x < r1; ++x) {
        while (x >= e_bg - p.pad) {  // range starts in (or reaches) virtual boxes
            x = e_bg;
            if (x >= r1) goto done;
            ++bg;
            s_bg = starts[bg];
            e_bg = starts[bg + 1];
            fresh = true;
        }
        if (fresh) {
            const int b = bg / p.Hkv, g = bg % p.Hkv;
            const float* qp = p.q + ((int64_t)b * p.Hkv * G + (int64_t)g * G) * D;
            for (int e = t; e < G * D; e += kGen) qs(e / D, e % D) = qp[e];
            if (t < G) {
                mst[t] = -INFINITY;
                lst[t] = 0.f;
            }
#pragma unroll
            for (int h = 0; h < kGenMaxG; ++h) acc[h][0] = acc[h][1] = 0.f;
            fresh = false;
        }
        const Box bx = box_of(x, bg, s_bg);
        if (pf) {
#pragma unroll
            for (int u = 0; u < EPT; ++u) {
                const int e = t + u * kGen;
                if (e < kBoxRows * D) {
                    Ks(e / D, e % D) = nk[u];
                    Vs(e / D, e % D) = nv[u];
                }
            }
        } else {
            const T* kb = static_cast<const T*>(p.k) + (int64_t)bg * p.l_cap * D;
            const T* vb = static_cast<const T*>(p.v) + (int64_t)bg * p.l_cap * D;
            for (int e = t; e < kBoxRows * D; e += kGen) {
                const int r = e / D, d = e % D;
                float kv = 0.f, vv = 0.f;
                if (r < bx.n) {
                    const int64_t row = p.idx ? (int64_t)p.idx[bx.row + r] : (int64_t)bx.row + r;
                    kv = tofl(kb[row * D + d]);
                    vv = tofl(vb[row * D + d]);
                }
                Ks(r, d) = kv;
                Vs(r, d) = vv;
            }
        }
        {   // the next real box starts loading now
            int64_t nx, nsbg;
            int nbg;
            if (next_real(x, bg, e_bg, nx, nbg, nsbg)) load_box(box_of(nx, nbg, nsbg), nbg);
        }
        __syncthreads();
        if (x == r0) GT_MARK(3);
        for (int pi = t / TPP; pi < pairs; pi += kGen / TPP) {
            const int tok = pi / G, h = pi % G, sub = t % TPP;
            float a = 0.f;
            if (tok < bx.n && ((bx.mask >> h) & 1)) {
                if (D % 8 == 0) {  // contiguous slice, four independent chains
                    float a4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
                    for (int j = 0; j < DPT; ++j) {
                        const int d = sub * DPT + j;
                        a4[j & 3] = fmaf(qs(h, d), Ks(tok, d), a4[j & 3]);
                    }
                    a = (a4[0] + a4[1]) + (a4[2] + a4[3]);
                } else {
                    for (int d = sub; d < D; d += TPP) a = fmaf(qs(h, d), Ks(tok, d), a);
                }
            }
            for (int o = TPP / 2; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (sub == 0) sc(tok, h) = (tok < bx.n && ((bx.mask >> h) & 1)) ? a * scale : -INFINITY;
        }
        __syncthreads();
        if (t < G) {
            float mx = mst[t];
            for (int tok = 0; tok < kBoxRows; ++tok) mx = fmaxf(mx, sc(tok, t));
            alp[t] = mx == -INFINITY ? 1.f : expf(mst[t] - mx);
            lst[t] *= alp[t];
            mst[t] = mx;
        }
        __syncthreads();
        for (int pi = t; pi < pairs; pi += kGen) {  // one exp per (token, head)
            const int tok = pi / G, h = pi % G;
            const float base = mst[h] == -INFINITY ? 0.f : mst[h];
            sc(tok, h) = expf(sc(tok, h) - base);
        }
        __syncthreads();
        if (t < G) {
            float sum = 0.f;
            for (int tok = 0; tok < kBoxRows; ++tok) sum += sc(tok, t);
            lst[t] += sum;
        }
#pragma unroll
        for (int dd = 0; dd < 2; ++dd) {
            const int d = t + dd * kGen;
            if (d < D) {
#pragma unroll
                for (int h = 0; h < kGenMaxG; ++h) {
                    if (h < G) {
                        float a = acc[h][dd] * alp[h];
                        for (int tok = 0; tok < kBoxRows; ++tok) a = fmaf(sc(tok, h), Vs(tok, d), a);
                        acc[h][dd] = a;
                    }
                }
            }
        }
        __syncthreads();
        if (x + 1 == r1 || x + 1 == e_bg - p.pad) {
            // a run wholly inside this CTA is final; else a partial for k_merge_runs
            const bool sole = s_bg >= r0 && e_bg - p.pad <= r1;
            const int64_t head0 = sole ? (int64_t)(bg / p.Hkv) * p.Hkv * G + (int64_t)(bg % p.Hkv) * G
                                       : (int64_t)(cta + bg) * G;
            float* dst_o = sole ? p.o : p.part_o;
            float* dst_l = sole ? p.lse : p.part_lse;
#pragma unroll
            for (int dd = 0; dd < 2; ++dd) {
                const int d = t + dd * kGen;
                if (d < D) {
#pragma unroll
                    for (int h = 0; h < kGenMaxG; ++h)
                        if (h < G) dst_o[(head0 + h) * D + d] = lst[h] > 0.f ? acc[h][dd] / lst[h] : 0.f;
                }
            }
            if (t < G && dst_l) dst_l[head0 + t] = lst[t] > 0.f ? mst[t] + logf(lst[t]) : -INFINITY;
            __syncthreads();
            if (x + 1 < r1) {
                x = e_bg - 1;  // skip the run's virtual boxes
                ++bg;
                s_bg = starts[bg];
                e_bg = starts[bg + 1];
                fresh = true;
            }
        }
    }
done:
    __syncthreads();
    write_empty_runs(p, starts, r0, r1, t, kGen);
    GT_MARK(5);
    // runs cut by a range end left partials: k_merge_runs follows
}

// ---------------------------------------------------------------------------
// f32 kernel with per-warp box streams (contiguous boxes, the decode path of
// config C1: f32 KV, D 64 / 128, G in {4, 7, 8})
// ---------------------------------------------------------------------------
// Every run (b, g) is cut into chunks of kFChunk consecutive boxes from its
// start; chunk k of the batch (runs in order) goes to warp k % (grid * kFW)
// of one CTA per SM, through a private ring of 1-D bulk copies (the K and V
// rows of a box are contiguous), so a box costs no CTA barrier and the warp's
// stream continues across its chunks.  Per box: QK with lane = (row, half of
// the dims), the row softmax by shuffles (exp2 domain), PV with lane = D/32
// dims.  A chunk's (o, lse) is a partial in chunk slot k (final when the run
// has one chunk); k_merge_chunks folds a run's chunks in chunk order.  The
// cut points depend only on the run, so a result does not depend on the other
// runs of the batch (the drop-in arena's batch sizes).
constexpr int kFW = 6;       // warps per CTA
constexpr int kFStages = 2;  // boxes in flight per warp
constexpr int kFChunk = 4;   // boxes per chunk

// Chunk prefix of the runs in smem (n_bg <= kMaxPrefix): cstart[bg] = first
// chunk of run bg, cstart[n_bg] = the total.  All threads; ends in a barrier.
__device__ const int32_t* chunk_starts(const int32_t* bg_count, int n_bg, int32_t* cs, int* wtmp, int t, int nt) {
    const int lane = t & 31, warp = t >> 5, nw = nt >> 5;
    int carry = 0;
    for (int c0 = 0; c0 < n_bg; c0 += nt) {
        const int i = c0 + t;
        const int v = i < n_bg ? (__ldcg(bg_count + i) + kFChunk - 1) / kFChunk : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wtmp[warp] = x;
        __syncthreads();
        int off = carry, tot = 0;
        for (int w = 0; w < nw; ++w) {
            if (w < warp) off += wtmp[w];
            tot += wtmp[w];
        }
        if (i < n_bg) cs[i] = off + x - v;
        __syncthreads();
        carry += tot;
    }
    if (t == 0) cs[n_bg] = carry;
    __syncthreads();
    return cs;
}

template <int D>
struct F32wCfg {
    static constexpr int BOXF = kBoxRows * D;  // floats of one box of K (or V)
    static constexpr size_t BAR = 0;
    static constexpr size_t RING = 128;
    static constexpr size_t QS = RING + (size_t)kFW * kFStages * 2 * BOXF * 4;
    static size_t total(int G) { return QS + (size_t)kFW * G * D * 4; }
};

template <int D, int G>
__global__ void __launch_bounds__(kFW * 32, 1) k_attend_f32w(const View p) {
    GT_MARK(0);
    pdl_wait();
    pdl_trigger();
    GT_MARK(1);
    using C = F32wCfg<D>;
    constexpr int DL = D / 32;  // PV: dims per lane
    constexpr int Q4 = D / 8;   // QK: float4s per half row
    extern __shared__ __align__(128) unsigned char fsm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(fsm + C::BAR);
    __shared__ int32_t s_cs[kMaxPrefix + 1];
    __shared__ int s_wtmp[kFW];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (t < kFW * kFStages) mbar_init(bars + t, 1);
    fence_mbar_init();
    const int32_t* cs = chunk_starts(p.bg_count, p.n_bg, s_cs, s_wtmp, t, kFW * 32);  // + barrier
    GT_MARK(2);
    const int NC = cs[p.n_bg];
    const int W = gridDim.x * kFW;            // warps of the grid
    const int w0 = blockIdx.x * kFW + warp;   // this warp's chunks: w0, w0 + W, ...
    const float sl2 = rsqrtf((float)D) * kLog2e;
    uint64_t* wbar = bars + warp * kFStages;
    float* wring = reinterpret_cast<float*>(fsm + C::RING) + (size_t)warp * kFStages * 2 * C::BOXF;
    float* wq = reinterpret_cast<float*>(fsm + C::QS) + (size_t)warp * G * D;
    // a cursor over this warp's boxes: chunk k, its run bg, box x of [x0, x1)
    struct Cur {
        int k, bg, x, x1;
    };
    auto chunk_at = [&](int k, Cur& c) -> bool {
        c.k = k;
        if (k >= NC) return false;
        int lo = 0, hi = p.n_bg - 1;  // last run whose first chunk is <= k
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (cs[mid] <= k) lo = mid;
            else hi = mid - 1;
        }
        c.bg = lo;
        c.x = (k - cs[lo]) * kFChunk;
        c.x1 = min(c.x + kFChunk, __ldcg(p.bg_count + lo));
        return true;
    };
    auto advance = [&](Cur& c) -> bool {  // next box of this warp's stream
        if (++c.x < c.x1) return true;
        return chunk_at(c.k + W, c);
    };
    auto issue = [&](const Cur& c, uint32_t slot) {  // lane 0
        const Box bx = p.boxes[(int64_t)c.bg * p.box_stride + c.x];
        const int st = (int)(slot % kFStages);
        float* kt = wring + (size_t)st * 2 * C::BOXF;
        const uint32_t bytes = (uint32_t)bx.n * D * 4;
        const int64_t row = (int64_t)c.bg * p.l_cap + bx.row;
        fence_proxy_async();  // this warp's earlier reads of the slot before the async writes
        mbar_arrive_expect_tx(wbar + st, 2 * bytes);
        bulk_g2s(kt, static_cast<const float*>(p.k) + row * D, bytes, wbar + st);
        bulk_g2s(kt + C::BOXF, static_cast<const float*>(p.v) + row * D, bytes, wbar + st);
    };
    Cur cur, pre;
    bool have = chunk_at(w0, cur);
    pre = cur;
    bool pre_ok = have;
    uint32_t issued = 0;  // (lane 0) boxes issued into the ring so far
    if (lane == 0)
        for (; pre_ok && issued < (uint32_t)kFStages; ++issued) {
            issue(pre, issued);
            pre_ok = advance(pre);
        }
    const int r = lane >> 1, hf = lane & 1;
    uint32_t slot = 0;
    bool marked = false;
    while (have) {
        // ---- one chunk: q of its group, then its boxes ----
        const int bg = cur.bg, k = cur.k;
        {
            const int bb = bg / p.Hkv, g = bg % p.Hkv;
            const float4* qp = reinterpret_cast<const float4*>(p.q + ((int64_t)bb * p.Hkv * G + (int64_t)g * G) * D);
            __syncwarp();
            for (int e = lane; e < G * D / 4; e += 32) reinterpret_cast<float4*>(wq)[e] = qp[e];
            __syncwarp();
        }
        float m[G], l[G], acc[G][DL];
#pragma unroll
        for (int h = 0; h < G; ++h) {
            m[h] = -INFINITY;
            l[h] = 0.f;
#pragma unroll
            for (int kk = 0; kk < DL; ++kk) acc[h][kk] = 0.f;
        }
        bool more = true;
        while (more) {
            const Box bx = p.boxes[(int64_t)bg * p.box_stride + cur.x];
            const int st = (int)(slot % kFStages);
            mbar_wait(wbar + st, (slot / kFStages) & 1u);
            if (!marked) {
                if (warp == 0) GT_MARK(3);
                marked = true;
            }
            const float* kt = wring + (size_t)st * 2 * C::BOXF;
            const float* vt = kt + C::BOXF;
            // QK: lane (row r, half hf) over D/2 dims, float4 reads rotated by lane
            float sc[G];
#pragma unroll
            for (int h = 0; h < G; ++h) sc[h] = 0.f;
            const bool rv = r < bx.n;  // rows past the box's end hold stale bytes: never read
            if (rv) {
                const float4* krow = reinterpret_cast<const float4*>(kt + r * D + hf * (D / 2));
                const float4* qrow = reinterpret_cast<const float4*>(wq + hf * (D / 2));
#pragma unroll
                for (int j = 0; j < Q4; ++j) {
                    const int jj = (j + lane) & (Q4 - 1);
                    const float4 k4 = krow[jj];
#pragma unroll
                    for (int h = 0; h < G; ++h) {
                        const float4 q4 = qrow[h * (D / 4) + jj];
                        sc[h] = fmaf(q4.x, k4.x, sc[h]);
                        sc[h] = fmaf(q4.y, k4.y, sc[h]);
                        sc[h] = fmaf(q4.z, k4.z, sc[h]);
                        sc[h] = fmaf(q4.w, k4.w, sc[h]);
                    }
                }
            }
            float pr[G];
#pragma unroll
            for (int h = 0; h < G; ++h) {
                float x = sc[h] + __shfl_xor_sync(0xffffffffu, sc[h], 1);
                x = (rv && ((bx.mask >> h) & 1)) ? x * sl2 : -INFINITY;
                // row softmax (16 rows: lanes 2r and 2r + 1 hold the same value)
                float mx = x;
#pragma unroll
                for (int o = 2; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                const float nm = fmaxf(m[h], mx);
                const float base = nm == -INFINITY ? 0.f : nm;
                const float al = nm == -INFINITY ? 1.f : exp2f(m[h] - nm);
                pr[h] = exp2f(x - base);
                float sum = pr[h];
#pragma unroll
                for (int o = 2; o < 32; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                l[h] = l[h] * al + sum;
                m[h] = nm;
#pragma unroll
                for (int kk = 0; kk < DL; ++kk) acc[h][kk] *= al;
            }
            // PV: lane owns dims [lane * DL, lane * DL + DL)
#pragma unroll 4
            for (int rr = 0; rr < kBoxRows; ++rr) {
                if (rr >= bx.n) break;  // (warp-uniform)
                float v[DL];
                if constexpr (DL == 4) {
                    const float4 v4 = reinterpret_cast<const float4*>(vt + rr * D)[lane];
                    v[0] = v4.x, v[1] = v4.y, v[2] = v4.z, v[3] = v4.w;
                } else {
                    const float2 v2 = reinterpret_cast<const float2*>(vt + rr * D)[lane];
                    v[0] = v2.x, v[1] = v2.y;
                }
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    const float ph = __shfl_sync(0xffffffffu, pr[h], 2 * rr);
#pragma unroll
                    for (int kk = 0; kk < DL; ++kk) acc[h][kk] = fmaf(ph, v[kk], acc[h][kk]);
                }
            }
            __syncwarp();  // every lane is done with the slot
            ++slot;
            if (lane == 0 && pre_ok) {  // refill the slot with the stream's next box
                issue(pre, issued++);
                pre_ok = advance(pre);
            }
            more = ++cur.x < cur.x1;
        }
        // ---- the chunk's (o, lse): final when its run has one chunk ----
        const bool sole = cs[bg + 1] - cs[bg] == 1;
        const int64_t head0 = sole ? (int64_t)(bg / p.Hkv) * p.Hkv * G + (int64_t)(bg % p.Hkv) * G
                                   : (int64_t)k * G;
        float* dst_o = sole ? p.o : p.part_o;
        float* dst_l = sole ? p.lse : p.part_lse;
#pragma unroll
        for (int h = 0; h < G; ++h) {
            const float inv = l[h] > 0.f ? 1.f / l[h] : 0.f;
            if constexpr (DL == 4)
                reinterpret_cast<float4*>(dst_o + (head0 + h) * D)[lane] =
                    make_float4(acc[h][0] * inv, acc[h][1] * inv, acc[h][2] * inv, acc[h][3] * inv);
            else
                reinterpret_cast<float2*>(dst_o + (head0 + h) * D)[lane] = make_float2(acc[h][0] * inv, acc[h][1] * inv);
            if (lane == 0 && dst_l) dst_l[head0 + h] = l[h] > 0.f ? (m[h] + log2f(l[h])) * kLn2 : -INFINITY;
        }
        have = chunk_at(k + W, cur);
    }
    GT_MARK(5);
}

// Merge of a run's chunk partials (k_attend_f32w), in chunk order: one
// 512-thread CTA per (b, g, head) (a batch-1 layer has few runs of many
// chunks: 16 slot subsets, one round of loads in flight); a run with no boxes
// gets the merge identity, a one-chunk run was written final.
constexpr int kMergeChunkThreads = 512;
__global__ void __launch_bounds__(kMergeChunkThreads) k_merge_chunks(int n_bg, int G, int D,
                                                               const int32_t* __restrict__ bg_count,
                                                               const float* __restrict__ part_o,
                                                               const float* __restrict__ part_lse,
                                                               float* __restrict__ o, float* __restrict__ lse) {
    pdl_wait();
    pdl_trigger();
    __shared__ int32_t s_cs[kMaxPrefix + 1];
    __shared__ int s_wtmp[kMergeChunkThreads / 32];
    const int bg = blockIdx.x, h = blockIdx.y, t = threadIdx.x;
    const int32_t* cs = chunk_starts(bg_count, n_bg, s_cs, s_wtmp, t, kMergeChunkThreads);
    const int base = cs[bg], nun = cs[bg + 1] - cs[bg];
    if (nun == 1) return;  // written final by the attention kernel
    const int64_t hd = (int64_t)bg * G + h;  // (b, g, h) = b * Hkv * G + g * G + h
    if (nun == 0) {
        for (int d = t; d < D; d += kMergeChunkThreads) o[hd * D + d] = 0.f;
        if (t == 0 && lse) lse[hd] = -INFINITY;
        return;
    }
    merge_slots<kMergeChunkThreads>(G, D, h, base, nun, part_o, part_lse, o + hd * D, lse ? lse + hd : nullptr);
}

// Merge of the partials of the generic kernel's runs cut by CTA range ends
// (attention.cpp:89-104 across the contributing CTAs): one 256-thread CTA per
// (b, g, head), launched behind it (PDL).  The contributors' LSEs first, then
// each thread folds one float4 column over a fixed subset of the contributors
// (eight loads in flight), subsets combined in a fixed order: deterministic.
constexpr int kMergeRunThreads = 256;
constexpr int kMaxMergeList = 2048;  // contributors of one run (>= the generic grid, 8 per SM)
__global__ void __launch_bounds__(kMergeRunThreads) k_merge_runs(const View p, int grid) {
    pdl_wait();
    pdl_trigger();
    __shared__ int32_t s_start[kMaxPrefix + 1];
    __shared__ int s_wtmp[kMergeRunThreads / 32];
    __shared__ float s_wm[kMergeRunThreads / 32];
    __shared__ float4 s_acc[kMergeRunThreads];
    __shared__ float s_den[kMergeRunThreads];
    const int t = threadIdx.x, bg = blockIdx.x, h = blockIdx.y, G = p.G, D = p.D;
    const int32_t* starts = run_starts(p, s_start, s_wtmp, t, kMergeRunThreads);
    const int64_t NB = starts[p.n_bg];
    const int64_t rs = starts[bg], re = starts[bg + 1] - p.pad;
    if (re <= rs) return;  // no real boxes: write_empty_runs wrote the identity
    const int cf = cta_of(rs, NB, grid), cl = cta_of(re - 1, NB, grid);
    if (cf == cl) return;  // wholly inside one CTA: written final
    // the CTAs of [cf, cl] with a non-empty range left a partial: compact them
    // in CTA (= box) order, so the fold below depends only on the run's boxes
    // and partials, not on how many other runs share the grid
    __shared__ int s_list[kMaxMergeList];
    __shared__ int s_n;
    if (t == 0) s_n = 0;
    __syncthreads();
    for (int c0 = cf; c0 <= cl; c0 += kMergeRunThreads) {
        const int c = c0 + t;
        const bool ne = c <= cl && cta_nonempty(c, NB, grid);
        const unsigned bal = __ballot_sync(0xffffffffu, ne);
        if ((t & 31) == 0) s_wtmp[t >> 5] = __popc(bal);
        __syncthreads();
        int off = s_n;
        for (int w = 0; w < (t >> 5); ++w) off += s_wtmp[w];
        if (ne) {
            const int pos = off + __popc(bal & ((1u << (t & 31)) - 1u));
            if (pos < kMaxMergeList) s_list[pos] = c;
        }
        __syncthreads();
        if (t == 0)
            for (int w = 0; w < kMergeRunThreads / 32; ++w) s_n += s_wtmp[w];
        __syncthreads();
    }
    const int n = min(s_n, kMaxMergeList);
    float m = -INFINITY;
    for (int i = t; i < n; i += kMergeRunThreads) m = fmaxf(m, __ldg(p.part_lse + (int64_t)(s_list[i] + bg) * G + h));
    m = warp_max(m);
    if ((t & 31) == 0) s_wm[t >> 5] = m;
    __syncthreads();
    float M = s_wm[0];
#pragma unroll
    for (int w = 1; w < kMergeRunThreads / 32; ++w) M = fmaxf(M, s_wm[w]);
    const int b = bg / p.Hkv, g = bg % p.Hkv;
    const int64_t hd = (int64_t)b * p.Hkv * G + (int64_t)g * G + h;
    const bool vec = D % 4 == 0;
    const int VP = vec ? D / 4 : D;              // columns of the head
    const int S = max(1, kMergeRunThreads / VP);  // contributor subsets
    for (int c0 = 0; c0 < VP; c0 += kMergeRunThreads / S) {
        const int v = c0 + t % (kMergeRunThreads / S), sub = t / (kMergeRunThreads / S);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        float den = 0.f;
        if (v < VP && sub < S) {
            constexpr int kIn = 8;
            for (int i0 = sub; i0 < n; i0 += S * kIn) {
                float4 x[kIn];
                float l[kIn];
#pragma unroll
                for (int j = 0; j < kIn; ++j) {
                    const int i = i0 + j * S;
                    const bool live = i < n;
                    const int64_t slot = (int64_t)((live ? s_list[i] : cf) + bg) * G + h;
                    l[j] = live ? __ldg(p.part_lse + slot) : -INFINITY;
                    x[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (live) {
                        if (vec) x[j] = __ldg(reinterpret_cast<const float4*>(p.part_o + slot * D) + v);
                        else x[j].x = __ldg(p.part_o + slot * D + v);
                    }
                }
#pragma unroll
                for (int j = 0; j < kIn; ++j) {
                    if (l[j] == -INFINITY) continue;
                    const float w = __expf(l[j] - M);
                    den += w;
                    acc.x += w * x[j].x;
                    acc.y += w * x[j].y;
                    acc.z += w * x[j].z;
                    acc.w += w * x[j].w;
                }
            }
        }
        s_acc[t] = acc;
        s_den[t] = den;
        __syncthreads();
        if (sub == 0 && v < VP) {
            for (int k = 1; k < S; ++k) {
                const float4 a = s_acc[k * (kMergeRunThreads / S) + t % (kMergeRunThreads / S)];
                acc.x += a.x;
                acc.y += a.y;
                acc.z += a.z;
                acc.w += a.w;
                den += s_den[k * (kMergeRunThreads / S) + t % (kMergeRunThreads / S)];
            }
            const float inv = den > 0.f ? 1.f / den : 0.f;
            if (vec) {
                *reinterpret_cast<float4*>(p.o + hd * D + v * 4) =
                    make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
            } else {
                p.o[hd * D + v] = acc.x * inv;
            }
            if (v == 0 && p.lse) p.lse[hd] = den > 0.f ? M + __logf(den) : -INFINITY;
        }
        __syncthreads();
    }
}

#undef Ks
#undef Vs
#undef qs
#undef sc

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------
__global__ void k_index_boxes(int64_t n, Box* boxes, int32_t* bg_start, int32_t* bg_count,
                              int32_t* bg_done) {
    const int64_t nb = (n + kBoxRows - 1) / kBoxRows;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nb) {
        Box b;
        b.row = (int32_t)(j * kBoxRows);
        b.n = (uint16_t)min((int64_t)kBoxRows, n - j * kBoxRows);
        b.mask = 1;
        boxes[j] = b;
    }
    if (j == 0) {
        bg_start[0] = 0;
        bg_start[1] = (int32_t)nb;
        bg_count[0] = (int32_t)nb;
        bg_done[0] = 0;
    }
}

__global__ void k_merge_partials(int n, int dim, const float* __restrict__ op,
                                 const float* __restrict__ lp, float* __restrict__ o,
                                 float* __restrict__ lse) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    float M = -INFINITY;
    for (int i = 0; i < n; ++i) M = fmaxf(M, lp[i]);
    if (d < dim) {
        if (M == -INFINITY) {
            o[d] = 0.f;
        } else {
            float num = 0.f, den = 0.f;
            for (int i = 0; i < n; ++i) {
                if (lp[i] == -INFINITY) continue;
                const float w = expf(lp[i] - M);
                num += w * op[(int64_t)i * dim + d];
                den += w;
            }
            o[d] = num / den;
            if (d == 0 && lse) lse[0] = M + logf(den);
        }
    }
    if (d == 0 && lse && M == -INFINITY) lse[0] = -INFINITY;
}

template <typename T>
__global__ void k_append(int64_t n_bg, int D, int64_t l_cap, int64_t row, T* k, T* v,
                         const float* kn, const float* vn) {
    pdl_wait();  // launched early behind the attention kernel (PDL); writes after it completes
    pdl_trigger();
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_bg * D) return;
    const int64_t bg = e / D, d = e % D;
    k[(bg * l_cap + row) * D + d] = (T)kn[e];
    v[(bg * l_cap + row) * D + d] = (T)vn[e];
}

template <typename T>
__global__ void k_convert(const float* src, T* dst, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = (T)src[i];
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
View make_view(const AttendArgs& a) {
    View v;
    v.n_bg = a.L.batch * a.L.kv_heads;
    v.Hkv = a.L.kv_heads;
    v.G = a.L.group_size;
    v.D = a.L.head_dim;
    v.l_cap = a.L.l_cap;
    v.k = a.k;
    v.v = a.v;
    v.q = a.q;
    v.idx = a.idx;
    v.boxes = a.boxes;
    v.box_stride = a.box_stride;
    v.bg_start = a.bg_start;
    v.bg_count = a.bg_count;
    v.pad = a.pad;
    v.part_o = a.part_o;
    v.part_lse = a.part_lse;
    v.bg_done = a.bg_done;
    v.o = a.o;
    v.lse = a.lse;
    return v;
}

template <int D>
void launch_tma(const AttendArgs& a, int grid, cudaStream_t s) {
    FX_REQUIRE(a.uq.words != nullptr && a.uq.ctl != nullptr && a.uq.ubase != nullptr && a.uq.epoch != 0,
               FX_ERR_STATE,
               "no-context: the TMA attention kernel needs the worklist's unit queue");
    QView v;
    v.n_bg = a.L.batch * a.L.kv_heads;
    v.Hkv = a.L.kv_heads;
    v.G = a.L.group_size;
    v.l_cap = a.L.l_cap;
    v.q = a.q;
    v.boxes = a.boxes;
    v.box_stride = a.box_stride;
    v.bg_count = a.bg_count;
    v.uq = a.uq;
    v.part_o = a.part_o;
    v.part_lse = a.part_lse;
    v.o = a.o;
    v.lse = a.lse;
    const int64_t rows = (int64_t)v.n_bg * a.L.l_cap;
    KvMaps maps;
    maps.box[0] = make_row_map(a.k, D, rows, kBoxRows);
    maps.box[1] = make_row_map(a.v, D, rows, kBoxRows);
    const size_t smem = TmaCfg<D>::TOTAL;
    FX_CUDA(cudaFuncSetAttribute(k_attend_tma<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch_pdl(k_attend_tma<D>, grid, kQThreads, smem, s, maps, v);
    FX_CUDA(cudaGetLastError());
}

}  // namespace

bool f32w_supported(const fx_layout& L, bool has_idx) {
    return !has_idx && L.dtype == FX_F32 && (L.head_dim == 128 || L.head_dim == 64) &&
           (L.group_size == 4 || L.group_size == 7 || L.group_size == 8) &&
           L.batch * L.kv_heads <= kMaxPrefix;
}


typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        FX_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
        FX_REQUIRE(ptr != nullptr && q == cudaDriverEntryPointSuccess, FX_ERR_CUDA,
                   "cuda-error: cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
    return fn;
}

// [rows][D] bf16 viewed as 3-D {64 columns, rows, D/64 chunks} (strides: row
// D*2 bytes, chunk 128 bytes); box = {64, box_rows, D/64}; 128-byte swizzle.
// (K/V rows here; metadata rows [min | max] = D' = 2 * head_dim in fx_score.cu.)
CUtensorMap make_row_map(const void* base, int D, int64_t rows, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(D / 64)};
    const cuuint64_t strides[2] = {(cuuint64_t)D * 2, 128};
    const cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)(D / 64)};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base),
                                   dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    FX_REQUIRE(r == CUDA_SUCCESS, FX_ERR_CUDA, "cuda-error: cuTensorMapEncodeTiled failed");
    return m;
}

int64_t chunk_capacity(int64_t n_bg, int64_t box_stride) {
    return n_bg * cdiv(std::max<int64_t>(box_stride, 1), kFChunk);
}

int64_t unit_capacity(int64_t n_bg, int64_t box_stride) {
    // every group's units at the worst case, plus the claims that run past the
    // tail (at most two per CTA)
    return n_bg * cdiv(std::max<int64_t>(box_stride, 1), kUnitBoxes) + 4096;
}

bool attend_uses_tma(const fx_layout& L, bool has_idx) {
    return !has_idx && L.dtype == FX_BF16 && (L.head_dim == 64 || L.head_dim == 128) &&
           L.group_size <= 8;
}

int attend_grid(const fx_layout& L, bool has_idx, int num_sms) {
    return attend_uses_tma(L, has_idx) || f32w_supported(L, has_idx) ? num_sms : num_sms * 8;
}

int launch_attend(const AttendArgs& a, int grid, bool allow_tma, cudaStream_t s) {
    FX_REQUIRE(a.L.group_size >= 1 && a.L.group_size <= kGenMaxG, FX_ERR_INVALID,
               "bad-shape: group_size must be in [1, 16]");
    FX_REQUIRE(a.L.head_dim >= 1 && a.L.head_dim <= kGenMaxD, FX_ERR_INVALID,
               "bad-shape: head_dim must be in [1, 256]");
    int n = 1;
    if (allow_tma && attend_uses_tma(a.L, a.idx != nullptr)) {
        if (a.L.head_dim == 128) launch_tma<128>(a, grid, s);
        else launch_tma<64>(a, grid, s);
        n = 1;  // launch_unit_merge follows
    } else {
        const View v = make_view(a);
        const int D = a.L.head_dim, G = a.L.group_size;
        const size_t smem = sizeof(float) * ((size_t)kBoxRows * (D + 1) + (size_t)kBoxRows * D +
                                             (size_t)G * D + (size_t)kBoxRows * G + 3 * G);
        if (a.L.dtype == FX_BF16) {
            FX_CUDA(cudaFuncSetAttribute(k_attend_generic<FX_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            launch_pdl(k_attend_generic<FX_BF16>, grid, kGen, smem, s, v);
        } else if (f32w_supported(a.L, a.idx != nullptr)) {
            using KernFn = void (*)(View);
            KernFn kern = nullptr;
            size_t fs = 0;
            if (D == 128) {
                fs = F32wCfg<128>::total(G);
                kern = G == 4 ? k_attend_f32w<128, 4> : G == 7 ? k_attend_f32w<128, 7> : k_attend_f32w<128, 8>;
            } else {
                fs = F32wCfg<64>::total(G);
                kern = G == 4 ? k_attend_f32w<64, 4> : G == 7 ? k_attend_f32w<64, 7> : k_attend_f32w<64, 8>;
            }
            FX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fs));
            launch_pdl(kern, grid, kFW * 32, fs, s, v);
        } else {
            auto kern = k_attend_generic<FX_F32>;
            if (D == 128 && G == 4) kern = k_attend_generic<FX_F32, 128, 4>;
            else if (D == 128 && G == 7) kern = k_attend_generic<FX_F32, 128, 7>;
            else if (D == 128 && G == 8) kern = k_attend_generic<FX_F32, 128, 8>;
            else if (D == 64 && G == 4) kern = k_attend_generic<FX_F32, 64, 4>;
            FX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            launch_pdl(kern, grid, kGen, smem, s, v);
        }
    }
    FX_CUDA(cudaGetLastError());
    return n;
}

int launch_unit_merge(const AttendArgs& a, int grid, bool allow_tma, cudaStream_t s) {
    if (!(allow_tma && attend_uses_tma(a.L, a.idx != nullptr)) && f32w_supported(a.L, a.idx != nullptr)) {
        const int n_bg = a.L.batch * a.L.kv_heads;  // f32 warp streams: chunk partials
        launch_pdl(k_merge_chunks, dim3((unsigned)n_bg, (unsigned)a.L.group_size), kMergeChunkThreads, 0, s, n_bg,
                   a.L.group_size, a.L.head_dim, (const int32_t*)a.bg_count, (const float*)a.part_o,
                   (const float*)a.part_lse, a.o, a.lse);
        FX_CUDA(cudaGetLastError());
        return 1;
    }
    if (!allow_tma || !attend_uses_tma(a.L, a.idx != nullptr)) {  // generic kernel: cut runs
        FX_REQUIRE(grid <= kMaxMergeList, FX_ERR_INVALID, "bad-shape: attention grid too large for the run merge");
        launch_pdl(k_merge_runs, dim3((unsigned)(a.L.batch * a.L.kv_heads), (unsigned)a.L.group_size),
                   kMergeRunThreads, 0, s, make_view(a), grid);
        FX_CUDA(cudaGetLastError());
        return 1;
    }
    const int n_bg = a.L.batch * a.L.kv_heads;
    // the widest CTA that still holds every (b, g, head) in one wave: a small
    // batch (C3, C5) folds more slots per round of loads (S = NT / (D / 4))
    static int occ[3] = {0, 0, 0};
    if (occ[0] == 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[0], k_merge_units<512>, 512, 0) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[1], k_merge_units<256>, 256, 0) != cudaSuccess) {
            cudaGetLastError();
            occ[0] = occ[1] = 0;
        }
        occ[2] = 1;
    }
    const int64_t ctas = (int64_t)n_bg * a.L.group_size;
    auto go = [&](auto kern, int nt) {
        launch_pdl(kern, dim3((unsigned)n_bg, (unsigned)a.L.group_size), nt, 0, s,
                   a.L.kv_heads, a.L.group_size, a.L.head_dim,
                   (const int32_t*)a.bg_count, (const int32_t*)a.uq.ubase, (const float*)a.part_o,
                   (const float*)a.part_lse, a.o, a.lse);
    };
    if (a.L.head_dim / 4 <= 512 && ctas <= (int64_t)grid * occ[0]) go(k_merge_units<512>, 512);
    else if (a.L.head_dim / 4 <= 256 && ctas <= (int64_t)grid * occ[1]) go(k_merge_units<256>, 256);
    else go(k_merge_units<kMergeThreads>, kMergeThreads);
    FX_CUDA(cudaGetLastError());
    return 1;
}

void launch_index_boxes(int64_t n, Box* boxes, int32_t* bg_start, int32_t* bg_count,
                        int32_t* bg_done, cudaStream_t s) {
    const int64_t nb = std::max<int64_t>(1, cdiv(n, kBoxRows));
    k_index_boxes<<<(unsigned)cdiv(nb, 256), 256, 0, s>>>(n, boxes, bg_start, bg_count, bg_done);
    FX_CUDA(cudaGetLastError());
}

void launch_merge_partials(int n, int dim, const float* o_parts, const float* lse_parts, float* o,
                           float* lse, cudaStream_t s) {
    k_merge_partials<<<(unsigned)cdiv(dim, 128), 128, 0, s>>>(n, dim, o_parts, lse_parts, o, lse);
    FX_CUDA(cudaGetLastError());
}

void launch_append(const fx_layout& L, void* k, void* v, int64_t row, const float* kn,
                   const float* vn, cudaStream_t s) {
    const int64_t n_bg = (int64_t)L.batch * L.kv_heads;
    const unsigned grid = (unsigned)cdiv(n_bg * L.head_dim, 256);
    if (L.dtype == FX_BF16)
        launch_pdl(k_append<__nv_bfloat16>, grid, 256, 0, s, n_bg, L.head_dim, L.l_cap, row,
                   static_cast<__nv_bfloat16*>(k), static_cast<__nv_bfloat16*>(v), kn, vn);
    else
        launch_pdl(k_append<float>, grid, 256, 0, s, n_bg, L.head_dim, L.l_cap, row,
                   static_cast<float*>(k), static_cast<float*>(v), kn, vn);
    FX_CUDA(cudaGetLastError());
}

void launch_convert(const float* src, void* dst, int dtype, size_t n, cudaStream_t s) {
    if (n == 0) return;
    const unsigned grid = (unsigned)((n + 255) / 256);
    if (dtype == FX_BF16) k_convert<__nv_bfloat16><<<grid, 256, 0, s>>>(src, static_cast<__nv_bfloat16*>(dst), n);
    else k_convert<float><<<grid, 256, 0, s>>>(src, static_cast<float*>(dst), n);
    FX_CUDA(cudaGetLastError());
}

}  // namespace fx

#ifdef FX_TRACE
extern "C" FX_API int fx_debug_trace(long long* out, int n) {
    return cudaMemcpyFromSymbol(out, fx::g_trace, sizeof(long long) * n) == cudaSuccess ? 0 : -2;
}
extern "C" FX_API int fx_debug_gtrace(long long* out, int n) {
    return cudaMemcpyFromSymbol(out, fx::g_gtrace, sizeof(long long) * n) == cudaSuccess ? 0 : -2;
}
#endif
