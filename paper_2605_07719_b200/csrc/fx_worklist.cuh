// fx_worklist.cuh -- the worklist body shared by the standalone k_worklist
// (fx_select.cu: given selections, no sparse segment) and the fused tail of
// k_select (fx_topk.cu: the CTA that finishes a group's last head builds that
// group's boxes, so the step has no separate worklist launch).
//
// One group (b, g): the default rows (sink, then local + decoded, the order of
// default_kv_attention, attention.cpp:143-151) and the union of the group's
// per-head block selections become 16-row boxes carrying the mask of the heads
// that attend them; the per-(b, g) box count goes to bg_count.  The selection
// bits may have been written by other CTAs of the same grid, so they are read
// through L2 (__ldcg), never the non-coherent path.
#pragma once

#include "fx_common.cuh"

#ifndef WL_MARK
#define WL_MARK(i)
#endif

namespace fx {

struct WorklistArgs {
    int Hkv, G;
    int64_t l_sink, l_cpu, l_tail;  // l_tail = local + decoded rows
    const int32_t* blk;             // [n_bg] chosen granularity (0 = streaming group)
    const uint32_t* sel_bits;       // [B*H][sel_words]
    int sel_words;
    Box* boxes;                     // [n_bg][box_stride]
    int64_t box_stride;
    int32_t* bg_count;              // [n_bg]
    int32_t* bg_start;              // [n_bg + 1] (published only when n_bg > kMaxRunPrefix)
    int32_t* publish_done;          // completion counter for the publish
    UnitQueue uq;                   // the attention unit queue (uq.words == nullptr: none)
};

// A group's boxes are final: publish its attention units (kUnitBoxes boxes
// each; one empty unit for a group without boxes, whose output is then the
// merge identity) to the unit queue.  All threads of the CTA, after the boxes
// and bg_count are written.  Release: each publishing lane fences after the
// CTA barrier, then stores its epoch-tagged flag words; the group counter is a
// release add after the words (a claimer that sees every group published reads
// the final tail).
__device__ inline void publish_units(const WorklistArgs& w, int bg, int64_t total) {
    if (w.uq.words == nullptr) return;
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const int n = total > 0 ? (int)((total + kUnitBoxes - 1) / kUnitBoxes) : 1;
    int base = 0;
    if (lane == 0) {
        base = atomicAdd(w.uq.ctl + 0, n);
        w.uq.ubase[bg] = base;
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    fence_acq_rel_gpu();
    const uint64_t tag = ((uint64_t)w.uq.epoch << 32) | ((uint64_t)(uint32_t)bg << kUnitIdxBits);
    for (int i = lane; i < n; i += 32) st_relaxed_gpu_u64(w.uq.words + base + i, tag | (uint64_t)i);
    __syncwarp();
    if (lane == 0) red_release_gpu_add(w.uq.ctl + 1, 1);
}

// Exclusive block scan of cnt[0..n) in place; returns the total.  wsum: nt + 1.
__device__ inline int64_t block_exclusive_scan(int32_t* cnt, int n, int64_t* wsum) {
    const int t = threadIdx.x, nt = blockDim.x;
    const int per = (n + nt - 1) / nt;
    const int a = min(n, t * per), e = min(n, a + per);
    int64_t s = 0;
    for (int i = a; i < e; ++i) s += cnt[i];
    wsum[t] = s;
    __syncthreads();
    if (t < 32) {  // warp scan of the nt partial sums
        int64_t run = 0;
        for (int base = 0; base < nt; base += 32) {
            const int i = base + t;
            const int64_t v = i < nt ? wsum[i] : 0;
            int64_t x = v;
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (t >= o) x += y;
            }
            if (i < nt) wsum[i] = run + x - v;
            run += __shfl_sync(0xffffffffu, x, 31);
        }
        if (t == 0) wsum[nt] = run;
    }
    __syncthreads();
    int64_t run = wsum[t];
    for (int i = a; i < e; ++i) {
        const int32_t v = cnt[i];
        cnt[i] = (int32_t)run;
        run += v;
    }
    __syncthreads();
    return wsum[nt];
}

// Boxes of group bg.  Smem: wcnt >= ceil(nblk/32) words, wsum >= blockDim + 1.
// All threads of the CTA.
__device__ inline void worklist_group(const WorklistArgs& w, int bg, int32_t* wcnt, int64_t* wsum) {
    const int b = bg / w.Hkv, g = bg % w.Hkv, G = w.G;
    const int t = threadIdx.x, nt = blockDim.x;
    const int blk = __ldcg(w.blk + bg);
    const uint16_t all = (uint16_t)((1u << G) - 1u);
    Box* out = w.boxes + (int64_t)bg * w.box_stride;
    const int nb_s = (int)cdiv_dev(w.l_sink, kBoxRows);
    const int nb_t = (int)cdiv_dev(w.l_tail, kBoxRows);
    for (int i = t; i < nb_s + nb_t; i += nt) {
        Box bx;
        if (i < nb_s) {
            bx.row = i * kBoxRows;
            bx.n = (uint16_t)min((int64_t)kBoxRows, w.l_sink - (int64_t)i * kBoxRows);
        } else {
            const int r = i - nb_s;
            bx.row = (int32_t)(w.l_sink + w.l_cpu + (int64_t)r * kBoxRows);
            bx.n = (uint16_t)min((int64_t)kBoxRows, w.l_tail - (int64_t)r * kBoxRows);
        }
        bx.mask = all;
        out[i] = bx;
    }
    const int nd = nb_s + nb_t;
    int64_t total = nd;
    if (blk > 0) {
        // thread per selection word: the G head words load together (one L2
        // round trip), the union's box count goes to wcnt; after the scan the
        // same thread emits its word's boxes (its set bits in order).
        const int64_t nblk = cdiv_dev(w.l_cpu, blk);
        const int W = (int)cdiv_dev(nblk, 32);
        const int bpb = blk / kBoxRows;
        const int64_t last = nblk - 1;
        const int nb_last = (int)cdiv_dev(w.l_cpu - last * blk, kBoxRows);
        const uint32_t* hg = w.sel_bits + ((int64_t)b * w.Hkv * G + (int64_t)g * G) * w.sel_words;
        if (W <= nt) {
            // one word per thread: the head words stay in registers from the
            // count to the emit (one L2 round trip), two-level shuffle scan
            const int j = t;
            uint32_t x[16];
            uint32_t u = 0;
#pragma unroll
            for (int h = 0; h < 16; ++h) {
                x[h] = (h < G && j < W) ? __ldcg(hg + (int64_t)h * w.sel_words + j) : 0u;
                u |= x[h];
            }
            int c = __popc(u) * bpb;
            if ((last >> 5) == j && ((u >> (last & 31)) & 1u)) c -= bpb - nb_last;
            WL_MARK(12);
            const int lane = t & 31, warp = t >> 5;
            int inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) wcnt[warp] = inc;
            __syncthreads();
            int base = 0, tot = 0;
            for (int q = 0; q < nt / 32; ++q) {
                const int v = wcnt[q];
                base += q < warp ? v : 0;
                tot += v;
            }
            __syncthreads();  // wcnt is reused by the caller
            total += tot;
            WL_MARK(13);
            int64_t o = nd + base + inc - c;
            while (u) {
                const int l = __ffs(u) - 1;
                u &= u - 1;
                uint32_t m = 0;
#pragma unroll
                for (int h = 0; h < 16; ++h) m |= ((x[h] >> l) & 1u) << h;
                const int r0 = (j * 32 + l) * blk;
                const int len = min(blk, (int)(w.l_cpu - r0));
                const int nb = (len + kBoxRows - 1) >> 4;
                const int row0 = (int)w.l_sink + r0;
                for (int y = 0; y < nb; ++y) {
                    Box bx;
                    bx.row = row0 + y * kBoxRows;
                    bx.n = (uint16_t)min(kBoxRows, len - y * kBoxRows);
                    bx.mask = (uint16_t)m;
                    out[o + y] = bx;
                }
                o += nb;
            }
            WL_MARK(14);
            if (t == 0) w.bg_count[bg] = (int32_t)total;
            publish_units(w, bg, total);
            return;
        }
        for (int j = t; j < W; j += nt) {
            uint32_t u = 0;
            for (int h = 0; h < G; ++h) u |= __ldcg(hg + (int64_t)h * w.sel_words + j);
            int c = __popc(u) * bpb;
            if ((last >> 5) == j && ((u >> (last & 31)) & 1u)) c -= bpb - nb_last;
            wcnt[j] = c;
        }
        WL_MARK(12);
        __syncthreads();
        total += block_exclusive_scan(wcnt, W, wsum);
        WL_MARK(13);
        for (int j = t; j < W; j += nt) {
            uint32_t x[16];
            uint32_t u = 0;
#pragma unroll
            for (int h = 0; h < 16; ++h) {
                x[h] = h < G ? __ldcg(hg + (int64_t)h * w.sel_words + j) : 0u;
                u |= x[h];
            }
            int64_t o = nd + wcnt[j];
            while (u) {
                const int l = __ffs(u) - 1;
                u &= u - 1;
                uint32_t m = 0;  // heads that selected this block
#pragma unroll
                for (int h = 0; h < 16; ++h) m |= ((x[h] >> l) & 1u) << h;
                const int r0 = (j * 32 + l) * blk;  // < 2^31 (checked by the launcher)
                const int len = min(blk, (int)(w.l_cpu - r0));
                const int nb = (len + kBoxRows - 1) >> 4;
                const int row0 = (int)w.l_sink + r0;
                for (int y = 0; y < nb; ++y) {
                    Box bx;
                    bx.row = row0 + y * kBoxRows;
                    bx.n = (uint16_t)min(kBoxRows, len - y * kBoxRows);
                    bx.mask = (uint16_t)m;
                    out[o + y] = bx;
                }
                o += nb;
            }
        }
    }
    WL_MARK(14);
    if (t == 0) w.bg_count[bg] = (int32_t)total;
    publish_units(w, bg, total);
}

// For n_bg > kMaxRunPrefix: the CTA that completes the last group publishes
// the exclusive prefix of (box count + kRunPad) over (b, g) into bg_start.
// All threads of a CTA that has just finished worklist_group(); blockDim <= 1024.
__device__ inline void worklist_publish(const WorklistArgs& w, int n_bg) {
    if (n_bg <= kMaxRunPrefix) return;  // the attention kernels rebuild the run starts from the counts
    if (w.uq.words) return;             // the unit queue needs no global prefix
    __shared__ int s_last;
    __shared__ int wtot[32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nt = blockDim.x;
    __syncthreads();
    if (t == 0) s_last = atomic_add_acq_rel_gpu(w.publish_done, 1) == n_bg - 1;
    __syncthreads();
    if (!s_last) return;
    fence_acq_rel_gpu();
    const int nw = nt / 32;
    for (int i0 = 0, run = 0; i0 < n_bg; i0 += nt) {
        const int i = i0 + t;
        const int v = i < n_bg ? __ldcg(w.bg_count + i) + kRunPad : 0;  // + virtual run cost
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wtot[warp] = x;
        __syncthreads();
        int wo = 0, ctot = 0;
        for (int q = 0; q < nw; ++q) {
            if (q < warp) wo += wtot[q];
            ctot += wtot[q];
        }
        if (i < n_bg) w.bg_start[i] = run + wo + x - v;
        run += ctot;
        __syncthreads();
        if (i0 + nt >= n_bg && t == 0) w.bg_start[n_bg] = run;
    }
}

}  // namespace fx
