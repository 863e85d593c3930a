// fx_capi.cu -- the C-ABI (include/fluxattn_b200.h): context, device scratch,
// and the entry points that sequence the K1..K5 kernels.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include <cuda.h>
#include <nvtx3/nvToolsExt.h>

#include "fx_internal.h"
#include "fx_worklist.cuh"

namespace {
thread_local std::string g_last_error;

// NVTX range over one C-ABI call (header-only NVTX3: a no-op unless a
// profiler injects itself), so nsys / ncu timelines show the API phases.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return FX_OK;
    } catch (const fx::Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::exception& e) {
        g_last_error = std::string("internal: ") + e.what();
        return FX_ERR_STATE;
    }
}

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t n) {
        if (n <= bytes) return;
        // regrowth frees (a device-wide synchronization): grow by half again at
        // least, so sizes that creep up step by step (the decoded rows) regrow rarely
        if (p) n = std::max(n, bytes + bytes / 2);
        if (p) FX_CUDA(cudaFree(p));
        p = nullptr;
        bytes = 0;
        n = (n + 255) & ~size_t(255);
        if (cudaMalloc(&p, n) != cudaSuccess) {
            cudaGetLastError();
            fx::fail(FX_ERR_NOMEM, "out-of-memory: device scratch of " + std::to_string(n) + " bytes");
        }
        bytes = n;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

// Bump allocator over one DevBuf (all regions 256-byte aligned).
struct Carve {
    size_t off = 0;
    template <class T>
    size_t take(size_t n) {
        const size_t o = off;
        off += (n * sizeof(T) + 255) & ~size_t(255);
        return o;
    }
};

void check_layout(const fx_layout* L) {
    FX_REQUIRE(L != nullptr, FX_ERR_INVALID, "bad-shape: null layout");
    FX_REQUIRE(L->batch > 0 && L->kv_heads > 0 && L->group_size > 0 && L->head_dim > 0,
               FX_ERR_INVALID, "bad-shape: non-positive layout dimension");
    FX_REQUIRE(L->dtype == FX_F32 || L->dtype == FX_BF16, FX_ERR_INVALID, "bad-shape: unknown dtype");
    FX_REQUIRE(L->l_sink >= 0 && L->l_cpu >= 0 && L->l_local >= 0, FX_ERR_INVALID,
               "bad-shape: negative segment length");
    FX_REQUIRE(L->l_cap >= L->l_sink + L->l_cpu + L->l_local, FX_ERR_INVALID,
               "bad-shape: l_cap smaller than sink + cpu + local");
    FX_REQUIRE(L->l_cap * L->batch * L->kv_heads < (int64_t)INT32_MAX, FX_ERR_INVALID,
               "bad-shape: more than 2^31 cache rows");
}

int elem_bytes(int dtype) { return dtype == FX_BF16 ? 2 : 4; }
}  // namespace

struct fx_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    uint64_t launches = 0;
    DevBuf step;  // fx_decode_step scratch
    DevBuf api;   // per-query API scratch
    DevBuf label; // fx_label_heads scratch
    DevBuf errw;  // sticky device error word (invalid given block sizes), read by fx_ctx_synchronize
    // attention unit queue flag words (epoch-tagged; zeroed when grown, so a
    // fresh buffer never holds the current epoch)
    DevBuf uq;
    uint32_t uq_epoch = 0;
    // optional per-kernel CUDA-event timing (fx_ctx_set_timing)
    bool timing = false;
    std::vector<cudaEvent_t> pool;
    struct Pending {
        int id;
        cudaEvent_t a, b;
    };
    std::vector<Pending> pending;
    double total_ms[FX_KERNEL_COUNT] = {};
    int64_t count[FX_KERNEL_COUNT] = {};
};

struct fx_model {
    fx_ctx* ctx = nullptr;
    DevBuf buf;
    DevBuf act;  // hidden activations of the tiled layers (grown to the largest batch)
    DevBuf tiles;  // monotonic row-tile counters of the layer-2 kernel (zeroed when allocated)
    const double *w1t, *b1, *w2t, *b2, *w3t, *b3, *mu, *sigma;
    int32_t* row_tiles(int n, cudaStream_t s) {
        const size_t need = (size_t)fx::predict_row_tiles(n) * sizeof(int32_t);
        if (need > tiles.bytes) {
            tiles.ensure(need);
            FX_CUDA(cudaMemsetAsync(tiles.p, 0, tiles.bytes, s));
        }
        return static_cast<int32_t*>(tiles.p);
    }
};

namespace {
cudaEvent_t pool_event(fx_ctx* c) {
    if (!c->pool.empty()) {
        cudaEvent_t e = c->pool.back();
        c->pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    FX_CUDA(cudaEventCreate(&e));
    return e;
}

// Brackets one kernel launch with CUDA events on the ctx stream when timing.
// contexts with event timing on: PDL is off process-wide while any is (fx_internal.h)
std::atomic<int> g_timing_ctxs{0};

struct Timed {
    fx_ctx* c;
    int id;
    cudaEvent_t a = nullptr, b = nullptr;
    Timed(fx_ctx* ctx, int kid) : c(ctx), id(kid) {
        if (!c->timing) return;
        a = pool_event(c);
        b = pool_event(c);
        FX_CUDA(cudaEventRecord(a, c->stream));
    }
    ~Timed() {
        if (!c->timing || !a) return;
        cudaEventRecord(b, c->stream);
        c->pending.push_back({id, a, b});
    }
};

void collect_timing(fx_ctx* c) {
    if (c->pending.empty()) return;
    FX_CUDA(cudaStreamSynchronize(c->stream));
    for (auto& p : c->pending) {
        float ms = 0.f;
        FX_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        c->total_ms[p.id] += ms;
        c->count[p.id] += 1;
        c->pool.push_back(p.a);
        c->pool.push_back(p.b);
    }
    c->pending.clear();
}

struct DeviceGuard {
    explicit DeviceGuard(fx_ctx* c) {
        FX_REQUIRE(c != nullptr, FX_ERR_STATE, "no-context: null fx_ctx");
        FX_CUDA(cudaSetDevice(c->device));
    }
};

struct StepScratch {
    int32_t* blk;
    double* budgets;
    int32_t* kblocks;
    float* approx;
    int64_t approx_stride;
    uint32_t* sel_bits;
    int sel_words;
    uint64_t* cand_keys;
    uint32_t* cand_ids;
    fx::Box* boxes;
    int64_t box_stride;
    int32_t* bg_count;
    int32_t* bg_start;
    int32_t* bg_done;  // [2 n_bg + 5]: attend counters | publish counter | select counters | unit queue
    int32_t* ubase;    // [n_bg] first unit of each group
    float* part_o;
    float* part_lse;
};

// Offsets of the decode-step scratch regions (one layout for the allocation
// and for the public size query fx_step_scratch_bytes).
struct StepOffsets {
    size_t blk, bud, kb, apx, bits, ck, ci, box, cnt, st, dn, ub, po, pl, total;
    int64_t approx_stride, box_stride;
    int words;
};

StepOffsets step_offsets(const fx_layout& L, int grid) {
    const int64_t n_bg = (int64_t)L.batch * L.kv_heads;
    const int64_t heads = n_bg * L.group_size;
    const int64_t nblk16 = std::max<int64_t>(1, fx::level_blocks(L.l_cpu, 16));
    const int64_t tail_max = L.l_cap - L.l_sink - L.l_cpu;
    StepOffsets o;
    o.words = (int)fx::cdiv(nblk16, 32);
    o.approx_stride = (nblk16 + 3) & ~int64_t(3);
    o.box_stride = fx::cdiv(L.l_sink, fx::kBoxRows) + fx::cdiv(tail_max, fx::kBoxRows) + nblk16 + 2;
    Carve c;
    o.blk = c.take<int32_t>(n_bg);
    o.bud = c.take<double>(heads);
    o.kb = c.take<int32_t>(heads);
    o.apx = c.take<float>(heads * o.approx_stride);
    o.bits = c.take<uint32_t>(heads * o.words);
    // the band lists use the approx row stride (nblk16 rounded up to 4)
    o.ck = c.take<uint64_t>(heads * o.approx_stride);
    o.ci = c.take<uint32_t>(heads * o.approx_stride);
    o.box = c.take<fx::Box>(n_bg * o.box_stride);
    o.cnt = c.take<int32_t>(n_bg);
    o.st = c.take<int32_t>(n_bg + 1);
    o.dn = c.take<int32_t>(2 * n_bg + 5);
    o.ub = c.take<int32_t>(n_bg);
    // partial slots: the generic kernel's (grid + n_bg), the TMA kernel's units
    // (the f32 warp-stream kernel's chunk slots only when that kernel runs)
    const int64_t slots = std::max<int64_t>({grid + n_bg, fx::unit_capacity(n_bg, o.box_stride),
                                             fx::f32w_supported(L, false) ? fx::chunk_capacity(n_bg, o.box_stride)
                                                                          : int64_t(0)});
    o.po = c.take<float>(slots * L.group_size * L.head_dim);
    o.pl = c.take<float>(slots * L.group_size);
    o.total = c.off;
    return o;
}

StepScratch carve_step(fx_ctx* ctx, const fx_layout& L, int grid, bool alloc) {
    const StepOffsets o = step_offsets(L, grid);
    if (alloc) ctx->step.ensure(o.total);
    char* b = static_cast<char*>(ctx->step.p);
    StepScratch s;
    s.blk = reinterpret_cast<int32_t*>(b + o.blk);
    s.budgets = reinterpret_cast<double*>(b + o.bud);
    s.kblocks = reinterpret_cast<int32_t*>(b + o.kb);
    s.approx = reinterpret_cast<float*>(b + o.apx);
    s.approx_stride = o.approx_stride;
    s.sel_bits = reinterpret_cast<uint32_t*>(b + o.bits);
    s.sel_words = o.words;
    s.cand_keys = reinterpret_cast<uint64_t*>(b + o.ck);
    s.cand_ids = reinterpret_cast<uint32_t*>(b + o.ci);
    s.boxes = reinterpret_cast<fx::Box*>(b + o.box);
    s.box_stride = o.box_stride;
    s.bg_count = reinterpret_cast<int32_t*>(b + o.cnt);
    s.bg_start = reinterpret_cast<int32_t*>(b + o.st);
    s.bg_done = reinterpret_cast<int32_t*>(b + o.dn);
    s.ubase = reinterpret_cast<int32_t*>(b + o.ub);
    s.part_o = reinterpret_cast<float*>(b + o.po);
    s.part_lse = reinterpret_cast<float*>(b + o.pl);
    return s;
}

int64_t next_pow2(int64_t x) {
    int64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}
}  // namespace

namespace {

// Validation + plan + score/select shared by fx_decode_step and
// fx_cp_candidates.  Returns the kernels launched; fills `s.sel_bits` (or
// points it at the caller's / given selection).
struct Planned {
    int32_t* blk;
    double* budgets;
    int32_t* kblocks;
    int launches;
    bool fused;  // the worklist ran inside k_select
};
// wl != nullptr: fuse the worklist into the selection kernel (Planned.fused).
// ap != nullptr: the plan kernel first appends one decoded row per (b, g).
Planned plan_and_select(fx_ctx* ctx, const fx_layout& L, const fx_step_args* a, StepScratch& s,
                        bool need_meta_for_select, const fx::WorklistArgs* wl = nullptr,
                        const fx::AppendArgs* ap = nullptr) {
    FX_REQUIRE(a->l_new >= 0 && L.l_sink + L.l_cpu + L.l_local + a->l_new + (ap ? 1 : 0) <= L.l_cap,
               FX_ERR_INVALID, "bad-shape: decoded rows exceed l_cap");
    FX_REQUIRE(a->plan_mode >= FX_PLAN_PROPS && a->plan_mode <= FX_PLAN_GIVEN, FX_ERR_INVALID,
               "bad-shape: unknown plan mode");
    const bool sparse = L.l_cpu > 0;
    const bool given_sel = a->sel_in != nullptr;
    const int64_t l_plan = a->l_cpu_total > 0 ? a->l_cpu_total : L.l_cpu;
    FX_REQUIRE(l_plan >= L.l_cpu && a->cpu_offset >= 0 && a->cpu_offset % 128 == 0 &&
                   a->cpu_offset + L.l_cpu <= l_plan,
               FX_ERR_INVALID, "bad-shape: shard [cpu_offset, +l_cpu) outside l_cpu_total or unaligned");
    if (sparse && (!given_sel || need_meta_for_select)) {
        for (int i = 0; i < 4; ++i)
            FX_REQUIRE(a->meta[i] != nullptr, FX_ERR_STATE, "no-context: missing block metadata");
        FX_REQUIRE(a->absmax != nullptr, FX_ERR_STATE, "no-context: missing absmax");
    }
    if (a->plan_mode == FX_PLAN_PROPS)
        FX_REQUIRE(a->bgt0 && a->kslope && a->streaming, FX_ERR_STATE,
                   "no-context: plan mode PROPS needs head properties");
    if (a->plan_mode == FX_PLAN_GIVEN)
        FX_REQUIRE(a->plan_blk && a->plan_budgets, FX_ERR_STATE,
                   "no-context: plan mode GIVEN needs blk and budgets");
    if (given_sel) {
        FX_REQUIRE(a->plan_mode == FX_PLAN_GIVEN, FX_ERR_INVALID,
                   "bad-shape: a given selection needs plan mode GIVEN");
        FX_REQUIRE(a->sel_words >= s.sel_words, FX_ERR_INVALID, "bad-shape: sel_words too small");
        s.sel_bits = const_cast<uint32_t*>(a->sel_in);
        s.sel_words = a->sel_words;
    } else if (a->sel_bits) {
        FX_REQUIRE(a->sel_words >= s.sel_words, FX_ERR_INVALID, "bad-shape: sel_words too small");
        s.sel_bits = a->sel_bits;
        s.sel_words = a->sel_words;
    }
    Planned p;
    p.blk = a->plan_blk ? a->plan_blk : s.blk;
    p.budgets = a->plan_budgets ? a->plan_budgets : s.budgets;
    p.kblocks = a->plan_kblocks ? a->plan_kblocks : s.kblocks;
    cudaStream_t st = ctx->stream;
    {
        Timed tm(ctx, FX_KERNEL_PLAN);
        fx::launch_prepare(L, l_plan, a->plan_mode, a->fixed_block_size, a->fixed_budget, a->bgt0,
                           a->kslope, a->streaming, p.blk, p.budgets, a->plan_volume,
                           a->plan_cand_volumes, p.kblocks, s.bg_done, st,
                           ap ? *ap : fx::AppendArgs(), static_cast<int32_t*>(ctx->errw.p));
    }
    p.launches = 1;
    p.fused = false;
    if (sparse && !given_sel) {
        {
            Timed tm(ctx, FX_KERNEL_SCORE);
            fx::launch_approx_scores(L, a->meta, a->q, p.blk, p.kblocks, s.approx, s.approx_stride,
                                     ctx->num_sms, st);
        }
        {
            Timed tm(ctx, FX_KERNEL_SELECT);
            fx::WorklistArgs w{};
            if (wl) {
                w = *wl;
                w.blk = p.blk;
                w.sel_bits = s.sel_bits;
                w.sel_words = s.sel_words;
            }
            fx::launch_select(L, a->meta, a->absmax, a->q, p.blk, p.kblocks, s.approx,
                              s.approx_stride, s.sel_bits, s.sel_words, s.cand_keys, s.cand_ids, st,
                              wl ? &w : nullptr, s.bg_done + (int64_t)L.batch * L.kv_heads + 1);
            p.fused = wl != nullptr;
        }
        p.launches += 2;
    } else if (!sparse) {
        FX_CUDA(cudaMemsetAsync(p.blk, 0, sizeof(int32_t) * L.batch * L.kv_heads, st));
    }
    return p;
}

}  // namespace

namespace fx {
bool pdl_enabled() { return g_timing_ctxs.load(std::memory_order_relaxed) == 0; }
}  // namespace fx

extern "C" {

const char* fx_last_error(void) { return g_last_error.c_str(); }
int fx_abi_version(void) { return FX_ABI_VERSION; }

int fx_ctx_create(int device, fx_ctx** out) {
    return guarded([&] {
        FX_REQUIRE(out != nullptr, FX_ERR_INVALID, "bad-shape: null out pointer");
        int n = 0;
        FX_CUDA(cudaGetDeviceCount(&n));
        FX_REQUIRE(device >= 0 && device < n, FX_ERR_INVALID, "bad-shape: no such CUDA device");
        FX_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        FX_CUDA(cudaGetDeviceProperties(&prop, device));
        FX_REQUIRE(prop.major == 10, FX_ERR_CUDA,
                   "cuda-error: this library is built for sm_100a (B200) only");
        auto* c = new fx_ctx();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        FX_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
        c->stream = c->own;
        c->errw.ensure(sizeof(int32_t));
        FX_CUDA(cudaMemset(c->errw.p, 0, sizeof(int32_t)));
        *out = c;
    });
}

int fx_ctx_destroy(fx_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        collect_timing(ctx);
        for (auto e : ctx->pool) cudaEventDestroy(e);
        ctx->step.release();
        ctx->api.release();
        ctx->label.release();
        ctx->errw.release();
        ctx->uq.release();
        if (ctx->own) cudaStreamDestroy(ctx->own);
        delete ctx;
    });
}

int fx_ctx_set_stream(fx_ctx* ctx, void* stream) {
    return guarded([&] {
        DeviceGuard g(ctx);
        // NULL is the legacy default stream (torch's default stream handle is 0)
        ctx->stream = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    });
}

void* fx_ctx_stream(fx_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int fx_ctx_synchronize(fx_ctx* ctx) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_CUDA(cudaStreamSynchronize(ctx->stream));
        int32_t e = 0;
        FX_CUDA(cudaMemcpy(&e, ctx->errw.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (e) {
            FX_CUDA(cudaMemset(ctx->errw.p, 0, sizeof(int32_t)));
            fx::fail(FX_ERR_INVALID,
                     "invalid-granularity: a given plan held a block size outside {0, 16, 32, 64, 128}; "
                     "those groups attended their resident defaults only");
        }
    });
}

uint64_t fx_ctx_launches(fx_ctx* ctx) { return ctx ? ctx->launches : 0; }

int fx_ctx_set_timing(fx_ctx* ctx, int enable) {
    return guarded([&] {
        DeviceGuard g(ctx);
        collect_timing(ctx);
        const bool on = enable != 0;
        if (on != ctx->timing) g_timing_ctxs += on ? 1 : -1;
        ctx->timing = on;
    });
}

int fx_ctx_kernel_time(fx_ctx* ctx, int32_t kernel, double* total_ms, int64_t* launches) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_REQUIRE(kernel >= 0 && kernel < FX_KERNEL_COUNT, FX_ERR_INVALID, "bad-shape: kernel id");
        collect_timing(ctx);
        if (total_ms) *total_ms = ctx->total_ms[kernel];
        if (launches) *launches = ctx->count[kernel];
    });
}

int fx_ctx_reset_timing(fx_ctx* ctx) {
    return guarded([&] {
        DeviceGuard g(ctx);
        collect_timing(ctx);
        for (int i = 0; i < FX_KERNEL_COUNT; ++i) {
            ctx->total_ms[i] = 0.0;
            ctx->count[i] = 0;
        }
    });
}

int fx_malloc(fx_ctx* ctx, size_t bytes, void** dptr) {
    return guarded([&] {
        DeviceGuard g(ctx);
        if (cudaMalloc(dptr, std::max<size_t>(bytes, 1)) != cudaSuccess) {
            cudaGetLastError();
            fx::fail(FX_ERR_NOMEM, "out-of-memory: fx_malloc");
        }
    });
}

int fx_free(fx_ctx* ctx, void* dptr) {
    return guarded([&] {
        DeviceGuard g(ctx);
        if (dptr) FX_CUDA(cudaFree(dptr));
    });
}

int fx_memcpy_h2d(fx_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    });
}

int fx_memcpy_d2h(fx_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        FX_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int fx_memcpy_d2d(fx_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    });
}

int fx_memset(fx_ctx* ctx, void* dptr, int value, size_t bytes) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_CUDA(cudaMemsetAsync(dptr, value, bytes, ctx->stream));
    });
}

int64_t fx_block_count(int64_t rows, int32_t block_size) {
    return block_size > 0 ? fx::cdiv(rows, block_size) : 0;
}

size_t fx_meta_level_bytes(const fx_layout* lay, int32_t block_size) {
    if (!lay || block_size <= 0) return 0;
    return (size_t)lay->batch * lay->kv_heads * fx::cdiv(lay->l_cpu, block_size) * 2 *
           lay->head_dim * elem_bytes(lay->dtype);
}

size_t fx_step_scratch_bytes(fx_ctx* ctx, const fx_layout* lay) {
    if (!lay) return 0;
    int sms = ctx ? ctx->num_sms : 148;
    if (!ctx) {
        int dev = 0;
        cudaDeviceProp prop;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaGetDeviceProperties(&prop, dev) == cudaSuccess)
            sms = prop.multiProcessorCount;
        else
            cudaGetLastError();
    }
    return step_offsets(*lay, fx::attend_grid(*lay, false, sms)).total;
}

int fx_build_metadata_levels(fx_ctx* ctx, const fx_layout* lay, const void* k, void* m16,
                             void* m32, void* m64, void* m128, float* absmax) {
    return guarded([&] {
        NvtxRange nv("fx_build_metadata_levels");
        DeviceGuard g(ctx);
        check_layout(lay);
        Timed tm(ctx, FX_KERNEL_METADATA);
        fx::launch_meta_levels(*lay, k, m16, m32, m64, m128, absmax, ctx->stream);
        ctx->launches += 1;
    });
}

int fx_build_metadata_means(fx_ctx* ctx, const fx_layout* lay, const void* k, void* const levels[4],
                            float* absmax, float* const means[4]) {
    return guarded([&] {
        NvtxRange nv("fx_build_metadata_means");
        DeviceGuard g(ctx);
        check_layout(lay);
        FX_REQUIRE(levels && means, FX_ERR_INVALID, "bad-shape: null level / mean arrays");
        for (int i = 0; i < 4; ++i)
            FX_REQUIRE(levels[i] && means[i], FX_ERR_INVALID, "bad-shape: every level needs its min/max and mean output");
        Timed tm(ctx, FX_KERNEL_METADATA);
        fx::launch_meta_levels(*lay, k, levels[0], levels[1], levels[2], levels[3], absmax, ctx->stream, means);
        ctx->launches += 1;
    });
}

int fx_build_metadata(fx_ctx* ctx, const void* k, int32_t dtype, int64_t rows, int32_t dim,
                      int32_t block_size, void* meta) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_REQUIRE(block_size > 0, FX_ERR_INVALID, "invalid-granularity: block size must be >= 1");
        FX_REQUIRE(dim > 0 && rows >= 0, FX_ERR_INVALID, "bad-shape: metadata input");
        fx::launch_meta_generic(k, dtype, rows, dim, block_size, meta, ctx->stream);
        ctx->launches += rows > 0 ? 1 : 0;
    });
}

int fx_block_scores(fx_ctx* ctx, const float* q, const void* meta, int32_t dtype, int64_t nblk,
                    int32_t dim, double* scores) {
    return guarded([&] {
        DeviceGuard g(ctx);
        fx::launch_exact_scores(q, meta, dtype, nblk, dim, scores, ctx->stream);
        ctx->launches += nblk > 0 ? 1 : 0;
    });
}

int fx_topk_blocks(fx_ctx* ctx, const float* q, const void* meta, int32_t dtype, int64_t nblk,
                   int32_t dim, int64_t k, uint32_t* blocks_out, int64_t* k_eff,
                   int32_t* clamped) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_REQUIRE(k >= 0 && nblk >= 0, FX_ERR_INVALID, "bad-shape: negative k or block count");
        const int64_t ke = std::min(k, nblk);
        if (k_eff) *k_eff = ke;
        if (clamped) *clamped = k > nblk ? 1 : 0;
        if (ke == 0) return;
        const int64_t cap = next_pow2(nblk);
        Carve c;
        const size_t ok = c.take<uint64_t>(cap), oi = c.take<uint32_t>(cap);
        ctx->api.ensure(c.off);
        char* b = static_cast<char*>(ctx->api.p);
        fx::launch_topk_exact(q, meta, dtype, nblk, dim, ke, blocks_out,
                              reinterpret_cast<uint64_t*>(b + ok), reinterpret_cast<uint32_t*>(b + oi),
                              cap, ctx->stream);
        int lg = 0;
        for (int64_t x = cap; x > 1; x >>= 1) ++lg;
        ctx->launches += 1 + (uint64_t)lg * (lg + 1) / 2;
    });
}

int fx_approx_scores(fx_ctx* ctx, const fx_layout* lay, const void* const meta[4],
                     const float* q, const int32_t* blk, float* out, double* eps_scale) {
    return guarded([&] {
        DeviceGuard g(ctx);
        check_layout(lay);
        const int64_t heads = (int64_t)lay->batch * lay->kv_heads * lay->group_size;
        Carve c;
        const size_t ok = c.take<int32_t>(heads);
        ctx->api.ensure(c.off);
        int32_t* kb = reinterpret_cast<int32_t*>(static_cast<char*>(ctx->api.p) + ok);
        // k = 1 for every head: forces scoring wherever a group has >= 2 blocks
        std::vector<int32_t> ones(heads, 1);
        FX_CUDA(cudaMemcpyAsync(kb, ones.data(), sizeof(int32_t) * heads, cudaMemcpyHostToDevice,
                                ctx->stream));
        fx::launch_approx_scores(*lay, meta, q, blk, kb, out,
                                 std::max<int64_t>(1, fx::level_blocks(lay->l_cpu, 16)), ctx->num_sms,
                                 ctx->stream);
        FX_CUDA(cudaStreamSynchronize(ctx->stream));
        if (eps_scale) *eps_scale = fx::approx_eps_scale(*lay);
        ctx->launches += 1;
    });
}

int fx_plan_groups(fx_ctx* ctx, int32_t n_groups, int32_t group_size, int64_t l_cpu,
                   const double* bgt0, const double* kslope, const int32_t* streaming,
                   int32_t* blk, double* budgets, double* volume, double* cand_volumes,
                   int32_t* kblocks) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_REQUIRE(n_groups >= 0, FX_ERR_INVALID, "bad-shape: negative group count");
        FX_REQUIRE(group_size >= 1, FX_ERR_INVALID, "empty-group: plan_group needs at least one head");
        if (n_groups == 0) return;
        fx_layout L{};
        L.batch = n_groups;
        L.kv_heads = 1;
        L.group_size = group_size;
        L.head_dim = 1;
        L.l_cpu = l_cpu;
        fx::launch_prepare(L, l_cpu, FX_PLAN_PROPS, 0, 0.0, bgt0, kslope, streaming, blk, budgets, volume,
                           cand_volumes, kblocks, nullptr, ctx->stream);
        ctx->launches += 1;
    });
}

int fx_blocks_for_budget(fx_ctx* ctx, int32_t n, const double* budgets, const int32_t* blk,
                         int64_t l_cpu, int32_t* kblocks) {
    return guarded([&] {
        DeviceGuard g(ctx);
        fx::launch_blocks_for_budget(n, budgets, blk, l_cpu, kblocks, ctx->stream);
        ctx->launches += n > 0 ? 1 : 0;
    });
}

int fx_model_create(fx_ctx* ctx, const double* w1, const double* b1, const double* w2,
                    const double* b2, const double* w3, const double* b3, const double* mu,
                    const double* sigma, fx_model** out) {
    return guarded([&] {
        DeviceGuard g(ctx);
        constexpr int F = 41, H1 = 256, H2 = 384, O = 3;
        // marshal to the device layout: transposed weights [in][out]
        std::vector<double> h;
        auto put_t = [&](const double* w, int outs, int ins) {
            for (int i = 0; i < ins; ++i)
                for (int o = 0; o < outs; ++o) h.push_back(w[(size_t)o * ins + i]);
        };
        auto put = [&](const double* x, int n) { h.insert(h.end(), x, x + n); };
        put_t(w1, H1, F);
        put(b1, H1);
        put_t(w2, H2, H1);
        put(b2, H2);
        put_t(w3, O, H2);
        put(b3, O);
        put(mu, F);
        put(sigma, F);
        auto* m = new fx_model();
        m->ctx = ctx;
        m->buf.ensure(h.size() * sizeof(double));
        FX_CUDA(cudaMemcpy(m->buf.p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
        const double* d = static_cast<const double*>(m->buf.p);
        m->w1t = d;
        d += F * H1;
        m->b1 = d;
        d += H1;
        m->w2t = d;
        d += H1 * H2;
        m->b2 = d;
        d += H2;
        m->w3t = d;
        d += H2 * O;
        m->b3 = d;
        d += O;
        m->mu = d;
        d += F;
        m->sigma = d;
        *out = m;
    });
}

int fx_model_destroy(fx_model* m) {
    return guarded([&] {
        if (!m) return;
        cudaSetDevice(m->ctx->device);
        m->buf.release();
        m->act.release();
        m->tiles.release();
        delete m;
    });
}

int fx_predict(fx_ctx* ctx, const fx_model* m, int32_t n, const double* features, double* bgt0,
               double* kslope, int32_t* streaming, double* z) {
    return guarded([&] {
        NvtxRange nv("fx_predict");
        DeviceGuard g(ctx);
        FX_REQUIRE(m != nullptr, FX_ERR_STATE, "no-model: predictor source requires a model");
        auto* mm = const_cast<fx_model*>(m);
        mm->act.ensure(fx::predict_scratch_bytes(n));
        int32_t* tiles = mm->row_tiles(n, ctx->stream);
        fx::launch_predict(n, m->w1t, m->b1, m->w2t, m->b2, m->w3t, m->b3, m->mu, m->sigma,
                           features, bgt0, kslope, streaming, z, mm->act.p, tiles, ctx->stream);
        ctx->launches += n > 0 ? 2 : 0;
    });
}

int fx_decode_step(fx_ctx* ctx, const fx_layout* lay, const fx_step_args* a) {
    return guarded([&] {
        NvtxRange nv("fx_decode_step");
        DeviceGuard g(ctx);
        check_layout(lay);
        FX_REQUIRE(a != nullptr && a->k && a->v && a->q && a->o, FX_ERR_STATE,
                   "no-context: decode step has no executable payload");
        const fx_layout& L = *lay;
        const int grid = fx::attend_grid(L, false, ctx->num_sms);
        StepScratch s = carve_step(ctx, L, grid, true);
        const int n_bg = L.batch * L.kv_heads;
        FX_REQUIRE((a->append_k == nullptr) == (a->append_v == nullptr), FX_ERR_INVALID,
                   "bad-shape: append_k and append_v go together");
        fx::AppendArgs ap;
        if (a->append_k) {
            ap.k = const_cast<void*>(a->k);
            ap.v = const_cast<void*>(a->v);
            ap.kn = a->append_k;
            ap.vn = a->append_v;
            ap.l_cap = L.l_cap;
            ap.row = L.l_sink + L.l_cpu + L.l_local + a->l_new;
            ap.D = L.head_dim;
            ap.bf16 = L.dtype == FX_BF16;
        }
        const int64_t l_new = a->l_new + (a->append_k ? 1 : 0);  // rows attended this step
        // the TMA attention kernel is fed by the worklist's unit queue
        fx::UnitQueue uq;
        if (fx::attend_uses_tma(L, false)) {
            const size_t wbytes = sizeof(uint64_t) * (size_t)fx::unit_capacity(n_bg, s.box_stride);
            if (wbytes > ctx->uq.bytes) {
                ctx->uq.ensure(wbytes);
                FX_CUDA(cudaMemsetAsync(ctx->uq.p, 0, ctx->uq.bytes, ctx->stream));
            }
            if (++ctx->uq_epoch == 0) ctx->uq_epoch = 1;
            uq.words = static_cast<uint64_t*>(ctx->uq.p);
            uq.ctl = s.bg_done + 2 * n_bg + 1;
            uq.ubase = s.ubase;
            uq.epoch = ctx->uq_epoch;
        }
        const fx::WorklistArgs wl{L.kv_heads, L.group_size, L.l_sink, L.l_cpu, L.l_local + l_new,
                                  nullptr, nullptr, 0, s.boxes, s.box_stride, s.bg_count,
                                  s.bg_start, s.bg_done + n_bg, uq};
        static const bool no_fuse = std::getenv("FX_DEBUG_NO_FUSED_WORKLIST") != nullptr;
        const Planned pl = plan_and_select(ctx, L, a, s, false, no_fuse ? nullptr : &wl,
                                           a->append_k ? &ap : nullptr);
        int32_t* blk = pl.blk;
        int n = pl.launches;
        cudaStream_t st = ctx->stream;
        if (!pl.fused) {
            Timed tm(ctx, FX_KERNEL_WORKLIST);
            fx::launch_worklist(L, l_new, blk, s.sel_bits, s.sel_words, s.boxes, s.box_stride,
                                s.bg_count, s.bg_start, s.bg_done, st, uq);
            n += 1;
        }
        fx::AttendArgs aa{};
        aa.L = L;
        aa.k = a->k;
        aa.v = a->v;
        aa.q = a->q;
        aa.idx = nullptr;
        aa.boxes = s.boxes;
        aa.box_stride = s.box_stride;
        aa.bg_start = s.bg_start;
        aa.bg_count = s.bg_count;
        aa.pad = fx::kRunPad;  // the worklist prefix includes kRunPad per run
        aa.part_o = s.part_o;
        aa.part_lse = s.part_lse;
        aa.bg_done = s.bg_done;
        aa.o = a->o;
        aa.lse = a->lse;
        aa.uq = uq;
        {
            Timed tm(ctx, FX_KERNEL_ATTEND);
            n += fx::launch_attend(aa, grid, true, st);
        }
        {
            Timed tm(ctx, FX_KERNEL_MERGE);
            n += fx::launch_unit_merge(aa, grid, true, st);
        }
        ctx->launches += n;
    });
}

int fx_plan_select(fx_ctx* ctx, const fx_layout* lay, const fx_step_args* a) {
    return guarded([&] {
        NvtxRange nv("fx_plan_select");
        DeviceGuard g(ctx);
        check_layout(lay);
        FX_REQUIRE(a != nullptr && a->q && a->sel_bits && a->plan_blk && a->plan_budgets &&
                       a->plan_kblocks, FX_ERR_STATE,
                   "no-context: plan_select needs q, sel_bits and the plan outputs");
        FX_REQUIRE(a->sel_in == nullptr && a->append_k == nullptr, FX_ERR_INVALID,
                   "bad-shape: plan_select takes no given selection or append");
        const fx_layout& L = *lay;
        StepScratch s = carve_step(ctx, L, fx::attend_grid(L, false, ctx->num_sms), true);
        const Planned pl = plan_and_select(ctx, L, a, s, false, nullptr);
        ctx->launches += pl.launches;
    });
}

int fx_sparse_decode(fx_ctx* ctx, const fx_layout* lay, const fx_step_args* a) {
    const int rc = guarded([&] {
        FX_REQUIRE(a != nullptr && a->sel_in != nullptr && a->plan_mode == FX_PLAN_GIVEN,
                   FX_ERR_STATE, "no-context: sparse_decode needs a given plan and selection");
    });
    return rc != FX_OK ? rc : fx_decode_step(ctx, lay, a);
}

int fx_gathered_attention(fx_ctx* ctx, const float* q, const void* k, const void* v,
                          int32_t dtype, int64_t rows, int32_t dim, const uint32_t* idx,
                          int64_t n, float* o, float* lse) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_REQUIRE(dim > 0 && n >= 0, FX_ERR_INVALID, "bad-shape: gathered attention input");
        if (n == 0) {  // merge identity: o = 0, lse = -inf
            fx::launch_merge_partials(0, dim, nullptr, nullptr, o, lse, ctx->stream);
            ctx->launches += 1;
            return;
        }
        fx_layout L{};
        L.batch = 1;
        L.kv_heads = 1;
        L.group_size = 1;
        L.head_dim = dim;
        L.dtype = dtype;
        L.l_cap = rows;
        const int64_t nb = fx::cdiv(n, fx::kBoxRows);
        const int grid = (int)std::min<int64_t>(nb, (int64_t)ctx->num_sms * 4);
        Carve c;
        const size_t ob = c.take<fx::Box>(nb), os = c.take<int32_t>(2), od = c.take<int32_t>(2),
                     oc = c.take<int32_t>(2);
        const size_t oo = c.take<float>((size_t)(grid + 1) * dim), ol = c.take<float>(grid + 1);
        ctx->api.ensure(c.off);
        char* b = static_cast<char*>(ctx->api.p);
        fx::AttendArgs aa{};
        aa.L = L;
        aa.k = k;
        aa.v = v;
        aa.q = q;
        aa.idx = idx;
        aa.boxes = reinterpret_cast<fx::Box*>(b + ob);
        aa.box_stride = nb;
        aa.bg_start = reinterpret_cast<int32_t*>(b + os);
        aa.bg_count = reinterpret_cast<int32_t*>(b + oc);
        aa.part_o = reinterpret_cast<float*>(b + oo);
        aa.part_lse = reinterpret_cast<float*>(b + ol);
        aa.bg_done = reinterpret_cast<int32_t*>(b + od);
        aa.o = o;
        aa.lse = lse;
        fx::launch_index_boxes(n, const_cast<fx::Box*>(aa.boxes), const_cast<int32_t*>(aa.bg_start),
                               const_cast<int32_t*>(aa.bg_count), aa.bg_done, ctx->stream);
        ctx->launches += 1 + fx::launch_attend(aa, grid, false, ctx->stream);
        ctx->launches += fx::launch_unit_merge(aa, grid, false, ctx->stream);
    });
}

int fx_merge_partials(fx_ctx* ctx, int32_t n, int32_t dim, const float* o_parts,
                      const float* lse_parts, float* o, float* lse) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_REQUIRE(n >= 0 && dim > 0, FX_ERR_INVALID, "bad-shape: merge input");
        fx::launch_merge_partials(n, dim, o_parts, lse_parts, o, lse, ctx->stream);
        ctx->launches += 1;
    });
}

int fx_append_kv(fx_ctx* ctx, const fx_layout* lay, void* k, void* v, int64_t row,
                 const float* k_new, const float* v_new) {
    return guarded([&] {
        NvtxRange nv("fx_append_kv");
        DeviceGuard g(ctx);
        check_layout(lay);
        FX_REQUIRE(row >= 0 && row < lay->l_cap, FX_ERR_INVALID, "bad-shape: append row out of range");
        Timed tm(ctx, FX_KERNEL_APPEND);
        fx::launch_append(*lay, k, v, row, k_new, v_new, ctx->stream);
        ctx->launches += 1;
    });
}

int fx_convert(fx_ctx* ctx, const float* src, void* dst, int32_t dtype, size_t n) {
    return guarded([&] {
        DeviceGuard g(ctx);
        fx::launch_convert(src, dst, dtype, n, ctx->stream);
        ctx->launches += n > 0 ? 1 : 0;
    });
}

// ---- output-aware budget oracle (budget_oracle.cpp) ------------------------

int fx_label_heads(fx_ctx* ctx, const fx_layout* lay, const void* k, const void* v, int64_t l_new,
                   const void* const meta[4], const float* q, double tau, int32_t criterion,
                   double* o_full, double* normalizer, double* budgets, int64_t* blocks,
                   double* bgt0, double* kslope, int32_t* streaming) {
    return guarded([&] {
        NvtxRange nv("fx_label_heads");
        DeviceGuard g(ctx);
        check_layout(lay);
        const fx_layout& L = *lay;
        FX_REQUIRE(k && v && q && o_full && normalizer && budgets && bgt0 && kslope && streaming,
                   FX_ERR_STATE, "no-context: label call has no payload");
        FX_REQUIRE(l_new >= 0 && L.l_sink + L.l_cpu + L.l_local + l_new <= L.l_cap, FX_ERR_INVALID,
                   "bad-shape: decoded rows exceed l_cap");
        FX_REQUIRE(L.l_sink + L.l_cpu + L.l_local + l_new > 0, FX_ERR_INVALID,
                   "empty-context: cache has no tokens");
        FX_REQUIRE(criterion == 0 || criterion == 1, FX_ERR_INVALID, "bad-shape: unknown criterion");
        if (L.l_cpu > 0)
            for (int i = 0; i < 4; ++i)
                FX_REQUIRE(meta && meta[i], FX_ERR_STATE, "no-context: missing block metadata");
        const void* mp[4] = {nullptr, nullptr, nullptr, nullptr};
        if (meta)
            for (int i = 0; i < 4; ++i) mp[i] = meta[i];
        ctx->label.ensure(fx::label_scratch_bytes(L, l_new) + 256);
        int32_t* err = reinterpret_cast<int32_t*>(static_cast<char*>(ctx->label.p) +
                                                  fx::label_scratch_bytes(L, l_new));
        fx::launch_label(L, k, v, l_new, q, mp, tau, criterion, ctx->label.p, o_full, normalizer,
                         budgets, blocks, bgt0, kslope, streaming, err, ctx->stream);
        ctx->launches += L.l_cpu > 0 ? 7 : 5;
        int32_t h_err = 0;
        FX_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        FX_CUDA(cudaStreamSynchronize(ctx->stream));
        FX_REQUIRE(h_err == 0, FX_ERR_INVALID, "degenerate-normalizer: all head outputs are zero");
    });
}

// ---- predictor features (features.cpp) -------------------------------------

int fx_prefill_stats(fx_ctx* ctx, const fx_layout* lay, const void* k, const void* v,
                     const void* const meta[4], const float* anchor, double tau, int32_t layer,
                     double* rec) {
    return guarded([&] {
        NvtxRange nv("fx_prefill_stats");
        DeviceGuard g(ctx);
        check_layout(lay);
        const fx_layout& L = *lay;
        FX_REQUIRE(k && v && anchor && rec, FX_ERR_STATE, "no-context: prefill has no payload");
        FX_REQUIRE(L.l_sink + L.l_cpu + L.l_local > 0, FX_ERR_INVALID,
                   "empty-context: cache has no tokens");
        if (L.l_cpu > 0)
            for (int i = 0; i < 4; ++i)
                FX_REQUIRE(meta && meta[i], FX_ERR_STATE, "no-context: missing block metadata");
        const void* mp[4] = {nullptr, nullptr, nullptr, nullptr};
        if (meta)
            for (int i = 0; i < 4; ++i) mp[i] = meta[i];
        const int64_t nh = (int64_t)L.batch * L.kv_heads * L.group_size;
        const size_t lab = fx::label_scratch_bytes(L, 0);
        // label outputs the prefill only consumes internally, then the group accumulators
        const size_t outs = (size_t)nh * L.head_dim * 8 + (size_t)L.batch * 8 + (size_t)nh * 5 * 8 * 2 +
                            (size_t)nh * 8 * 3 + 4096;
        ctx->label.ensure(lab + outs + fx::prefill_group_scratch_bytes(L) + 256);
        char* b = static_cast<char*>(ctx->label.p) + lab;
        auto take = [&](size_t bytes) {
            char* r = b;
            b += (bytes + 255) & ~size_t(255);
            return r;
        };
        double* o_full = reinterpret_cast<double*>(take((size_t)nh * L.head_dim * 8));
        double* nrm = reinterpret_cast<double*>(take((size_t)L.batch * 8));
        double* bud = reinterpret_cast<double*>(take((size_t)nh * 5 * 8));
        int64_t* blocks = reinterpret_cast<int64_t*>(take((size_t)nh * 5 * 8));
        double* b0 = reinterpret_cast<double*>(take((size_t)nh * 8));
        double* ks = reinterpret_cast<double*>(take((size_t)nh * 8));
        int32_t* st = reinterpret_cast<int32_t*>(take((size_t)nh * 4));
        int32_t* err = reinterpret_cast<int32_t*>(take(4));
        void* grp = take(fx::prefill_group_scratch_bytes(L));
        fx::launch_label(L, k, v, 0, anchor, mp, tau, 0, ctx->label.p, o_full, nrm, bud, blocks, b0, ks,
                         st, err, ctx->stream, rec, layer);
        fx::launch_prefill_group(L, k, v, rec, grp, ctx->stream);
        ctx->launches += (L.l_cpu > 0 ? 8 : 6) + 3;
        int32_t h_err = 0;
        FX_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        FX_CUDA(cudaStreamSynchronize(ctx->stream));
        FX_REQUIRE(h_err == 0, FX_ERR_INVALID, "degenerate-normalizer: all head outputs are zero");
    });
}

int fx_decode_features(fx_ctx* ctx, const fx_layout* lay, const void* k, const void* v,
                       int64_t l_new, const float* q, const double* rec, double* features) {
    return guarded([&] {
        NvtxRange nv("fx_decode_features");
        DeviceGuard g(ctx);
        check_layout(lay);
        const fx_layout& L = *lay;
        FX_REQUIRE(k && v && q && rec && features, FX_ERR_STATE, "no-context: features have no payload");
        FX_REQUIRE(l_new >= 0 && L.l_sink + L.l_cpu + L.l_local + l_new <= L.l_cap, FX_ERR_INVALID,
                   "bad-shape: decoded rows exceed l_cap");
        if (fx::feat_fused_supported(L)) {
            ctx->api.ensure(fx::feat_fused_scratch_bytes(L, l_new));
            fx::launch_feat_fused(L, const_cast<void*>(k), const_cast<void*>(v), l_new, q, rec, features,
                                  ctx->api.p, ctx->stream, nullptr, nullptr, nullptr, nullptr, ctx->num_sms);
            ctx->launches += 2;
        } else {
            ctx->api.ensure(fx::decode_features_scratch_bytes(L, l_new));
            fx::launch_decode_features(L, k, v, l_new, q, rec, features, ctx->api.p, ctx->stream);
            ctx->launches += 3;
        }
    });
}

int fx_predict_props(fx_ctx* ctx, const fx_layout* lay, void* k, void* v, int64_t l_new,
                     const float* append_k, const float* append_v, const float* q, const double* rec,
                     const fx_model* m, double* features, double* z, double* bgt0, double* kslope,
                     int32_t* streaming) {
    return guarded([&] {
        NvtxRange nv("fx_predict_props");
        DeviceGuard g(ctx);
        check_layout(lay);
        const fx_layout& L = *lay;
        FX_REQUIRE(m != nullptr, FX_ERR_STATE, "no-model: predictor source requires a model");
        FX_REQUIRE(k && v && q && rec && bgt0 && kslope && streaming, FX_ERR_STATE,
                   "no-context: predictor step has no payload");
        FX_REQUIRE((append_k == nullptr) == (append_v == nullptr), FX_ERR_INVALID,
                   "bad-shape: append_k and append_v go together");
        const int64_t l_eff = l_new + (append_k ? 1 : 0);  // rows attended (the appended one included)
        FX_REQUIRE(l_new >= 0 && L.l_sink + L.l_cpu + L.l_local + l_eff <= L.l_cap, FX_ERR_INVALID,
                   "bad-shape: decoded rows exceed l_cap");
        const int64_t nh = (int64_t)L.batch * L.kv_heads * L.group_size;
        const bool fused = fx::feat_fused_supported(L);
        if (!fused && append_k) {  // the general-shape feature kernels read the cache only
            fx::launch_append(L, k, v, L.l_sink + L.l_cpu + L.l_local + l_new, append_k, append_v, ctx->stream);
            ctx->launches += 1;
        }
        auto* mm = const_cast<fx_model*>(m);
        mm->act.ensure(fx::predict_scratch_bytes((int)nh));
        int32_t* tiles = mm->row_tiles((int)nh, ctx->stream);
        double* a1 = static_cast<double*>(mm->act.p);
        double* a2 = a1 + (size_t)nh * 256;
        if (fused) {  // features -> normalize -> layer 1 inside the merge kernel, then layers 2 and 3
            ctx->api.ensure(fx::feat_fused_scratch_bytes(L, l_eff));
            const double* l1[4] = {m->w1t, m->b1, m->mu, m->sigma};
            fx::launch_feat_fused(L, k, v, l_eff, q, rec, features, ctx->api.p, ctx->stream, append_k, append_v,
                                  l1, a1, ctx->num_sms);
            fx::launch_predict_tail((int)nh, a1, m->w2t, m->b2, m->w3t, m->b3, bgt0, kslope, streaming, z, a2,
                                    tiles, ctx->stream);
            ctx->launches += 3;
        } else {
            const size_t fs = fx::decode_features_scratch_bytes(L, l_eff);
            const size_t fb = features ? 0 : (size_t)nh * 41 * sizeof(double);
            ctx->api.ensure(fs + fb + 256);
            double* f = features ? features
                                 : reinterpret_cast<double*>(static_cast<char*>(ctx->api.p) + ((fs + 255) & ~size_t(255)));
            fx::launch_decode_features(L, k, v, l_eff, q, rec, f, ctx->api.p, ctx->stream);
            fx::launch_predict((int)nh, m->w1t, m->b1, m->w2t, m->b2, m->w3t, m->b3, m->mu, m->sigma, f, bgt0,
                               kslope, streaming, z, mm->act.p, tiles, ctx->stream);
            ctx->launches += 5;
        }
    });
}

// ---- synthetic workload generator (workload.cpp) ---------------------------

void* api_scratch(size_t bytes, void* c) {
    fx_ctx* ctx = static_cast<fx_ctx*>(c);
    ctx->api.ensure(bytes);
    return ctx->api.p;
}

int fx_generate(fx_ctx* ctx, const fx_workload_spec* sp, const fx_layout* lay, const uint64_t* seeds,
                const int32_t* layers, void* k, void* v, float* anchor_q, int32_t steps,
                float* step_q, float* step_new_k, float* step_new_v, int32_t* archetypes) {
    return guarded([&] {
        NvtxRange nv("fx_generate");
        DeviceGuard g(ctx);
        check_layout(lay);
        FX_REQUIRE(sp && seeds && layers && k && v, FX_ERR_STATE, "no-context: generate has no payload");
        const fx_layout& L = *lay;
        // validate_spec (workload.cpp:124-146)
        FX_REQUIRE(sp->context_len > sp->sink_tokens + sp->local_tokens, FX_ERR_INVALID,
                   "infeasible-spec: context shorter than sink+local defaults");
        FX_REQUIRE(sp->heads > 0 && sp->group_size > 0 && sp->heads % sp->group_size == 0, FX_ERR_INVALID,
                   "infeasible-spec: heads must be a multiple of group_size");
        const double fsum = sp->streaming_frac + sp->retrieval_frac + sp->sink_frac + sp->diffuse_frac;
        FX_REQUIRE(std::abs(fsum - 1.0) <= 1e-9, FX_ERR_INVALID,
                   "infeasible-spec: archetype fractions must sum to 1");
        FX_REQUIRE(sp->query_drift >= -1.0 && sp->query_drift <= 1.0, FX_ERR_INVALID,
                   "infeasible-spec: query drift outside [-1, 1]");
        const int64_t l_cpu = (int64_t)sp->context_len - sp->sink_tokens - sp->local_tokens;
        FX_REQUIRE(!(sp->sink_frac > 0.0 && l_cpu < (int64_t)sp->decoy_tokens + sp->decoy_payload_tokens + 256),
                   FX_ERR_INVALID, "infeasible-spec: cpu segment too small for decoy runs");
        FX_REQUIRE(!(sp->retrieval_frac > 0.0 && l_cpu < (int64_t)sp->needles * sp->needle_tokens),
                   FX_ERR_INVALID, "infeasible-spec: cpu segment too small for needles");
        FX_REQUIRE(L.kv_heads == sp->heads / sp->group_size && L.group_size == sp->group_size &&
                       L.head_dim == sp->head_dim && L.l_sink == sp->sink_tokens &&
                       L.l_local == sp->local_tokens && L.l_cpu == l_cpu && L.l_cap >= sp->context_len,
                   FX_ERR_INVALID, "bad-shape: layout does not match the workload spec");
        FX_REQUIRE(steps >= 0, FX_ERR_INVALID, "bad-shape: negative step count");
        fx::generate_workload(L, *sp, seeds, layers, k, v, anchor_q, steps, step_q, step_new_k,
                              step_new_v, archetypes, api_scratch, ctx, ctx->stream);
        ctx->launches += 2;
    });
}

// ---- FXT1 traces (workload.cpp:311-433) -------------------------------------

int fx_trace_info_read(const char* path, fx_trace_info* info) {
    return guarded([&] {
        FX_REQUIRE(info != nullptr, FX_ERR_INVALID, "bad-shape: null info");
        fx::trace_info(path, info);
    });
}

int fx_trace_load(fx_ctx* ctx, const char* path, int32_t layer, const fx_layout* lay, int32_t b,
                  void* k, void* v, float* anchor_q, float* step_q, float* new_k, float* new_v,
                  int32_t* archetypes) {
    return guarded([&] {
        DeviceGuard g(ctx);
        check_layout(lay);
        FX_REQUIRE(k && v, FX_ERR_STATE, "no-context: trace load has no cache");
        fx::trace_load(path, layer, *lay, b, k, v, anchor_q, step_q, new_k, new_v, archetypes,
                       api_scratch, ctx, ctx->stream);
        ctx->launches += lay->dtype == FX_BF16 ? 2 * lay->kv_heads : 0;
    });
}

int fx_trace_save(fx_ctx* ctx, const char* path, const fx_trace_info* info, const fx_layout* lay,
                  const int32_t* entries, const void* k, const void* v, const float* anchor_q,
                  const float* step_q, const float* new_k, const float* new_v,
                  const int32_t* archetypes, const int32_t* needle_count, const uint32_t* needles) {
    return guarded([&] {
        DeviceGuard g(ctx);
        check_layout(lay);
        FX_REQUIRE(info && entries && k && v, FX_ERR_STATE, "no-context: trace save has no payload");
        FX_REQUIRE(info->layers > 0 && info->heads > 0 && info->group_size > 0 &&
                       info->heads % info->group_size == 0 && info->decode_steps >= 0,
                   FX_ERR_INVALID, "bad-shape: implausible trace header");
        FX_REQUIRE(!needle_count || needles, FX_ERR_INVALID, "bad-shape: needle counts without ranges");
        fx::trace_save(path, *info, *lay, entries, k, v, anchor_q, step_q, new_k, new_v, archetypes,
                       needle_count, needles, ctx->stream);
    });
}

// ---- context-parallel decode (C5) ----------------------------------------

int fx_cp_candidates(fx_ctx* ctx, const fx_layout* lay, const fx_step_args* a, int64_t cap,
                     uint64_t* keys, uint32_t* ids, int32_t* count, uint64_t* kth) {
    return guarded([&] {
        NvtxRange nv("fx_cp_candidates");
        DeviceGuard g(ctx);
        check_layout(lay);
        const fx_layout& L = *lay;
        FX_REQUIRE(a != nullptr && a->q && keys && ids && count && kth, FX_ERR_STATE,
                   "no-context: candidate selection has no payload");
        FX_REQUIRE(L.l_cpu > 0, FX_ERR_INVALID, "empty-context: shard has no cpu rows");
        FX_REQUIRE(a->sel_in == nullptr, FX_ERR_INVALID, "bad-shape: candidates select, sel_in must be null");
        FX_REQUIRE(a->append_k == nullptr, FX_ERR_INVALID, "bad-shape: append with the attend phase, not candidates");
        FX_REQUIRE(cap >= fx::level_blocks(L.l_cpu, 16), FX_ERR_INVALID,
                   "bad-shape: cap must hold every block of the shard at granularity 16");
        const int grid = fx::attend_grid(L, false, ctx->num_sms);
        StepScratch s = carve_step(ctx, L, grid, true);
        const Planned pl = plan_and_select(ctx, L, a, s, true);
        fx::launch_cp_candidates(L, a->meta, a->q, pl.blk, pl.kblocks, s.sel_bits, s.sel_words,
                                 a->cpu_offset, cap, keys, ids, count, kth, ctx->stream);
        ctx->launches += pl.launches + 1;
    });
}

int fx_cp_threshold(fx_ctx* ctx, int32_t ranks, int64_t n, int64_t cap, const uint64_t* keys,
                    const uint64_t* kth_all, uint64_t* thresh, int32_t* keep) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_REQUIRE(ranks >= 1 && n >= 0 && cap >= 1, FX_ERR_INVALID, "bad-shape: threshold input");
        fx::launch_cp_threshold(ranks, n, cap, keys, kth_all, thresh, keep, ctx->stream);
        ctx->launches += n > 0 ? 1 : 0;
    });
}

int fx_cp_select(fx_ctx* ctx, const fx_layout* lay, int32_t ranks, int32_t self, int64_t m,
                 const uint64_t* gkeys, const uint32_t* gids, const uint64_t* thresh,
                 const int32_t* kblocks, const int32_t* blk, int64_t cpu_offset, uint32_t* sel_out,
                 int32_t sel_words) {
    return guarded([&] {
        DeviceGuard g(ctx);
        check_layout(lay);
        FX_REQUIRE(ranks >= 1 && self >= 0 && self < ranks && m >= 0, FX_ERR_INVALID,
                   "bad-shape: rank / candidate count");
        FX_REQUIRE(cpu_offset >= 0 && cpu_offset % 128 == 0, FX_ERR_INVALID,
                   "bad-shape: cpu_offset must be a multiple of 128");
        FX_REQUIRE(sel_words >= fx::cdiv(std::max<int64_t>(1, fx::level_blocks(lay->l_cpu, 16)), 32),
                   FX_ERR_INVALID, "bad-shape: sel_words too small");
        fx::launch_cp_select(*lay, ranks, self, m, gkeys, gids, thresh, kblocks, blk, cpu_offset,
                             sel_out, sel_words, ctx->stream);
        ctx->launches += 1;
    });
}

int fx_cp_signal(fx_ctx* ctx, uint64_t* flags, int32_t slot, uint64_t stamp) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_REQUIRE(flags && slot >= 0 && slot < 4, FX_ERR_INVALID, "bad-shape: flag slot");
        fx::launch_cp_signal(flags, slot, stamp, ctx->stream);
        ctx->launches += 1;
    });
}

int fx_cp_select_peer(fx_ctx* ctx, const fx_layout* lay, int32_t ranks, int32_t self,
                      const fx_cp_peer* peers, uint64_t stamp, const int32_t* kblocks,
                      const int32_t* blk, int64_t cpu_offset, uint32_t* sel_out, int32_t sel_words) {
    return guarded([&] {
        NvtxRange nv("fx_cp_select_peer");
        DeviceGuard g(ctx);
        check_layout(lay);
        FX_REQUIRE(peers && kblocks && blk && sel_out, FX_ERR_STATE, "no-context: peer select has no payload");
        FX_REQUIRE(cpu_offset >= 0 && cpu_offset % 128 == 0, FX_ERR_INVALID,
                   "bad-shape: cpu_offset must be a multiple of 128");
        FX_REQUIRE(sel_words >= fx::cdiv(std::max<int64_t>(1, fx::level_blocks(lay->l_cpu, 16)), 32),
                   FX_ERR_INVALID, "bad-shape: sel_words too small");
        fx::launch_cp_select_peer(*lay, ranks, self, peers, stamp, kblocks, blk, cpu_offset, sel_out,
                                  sel_words, ctx->stream);
        ctx->launches += 1;
    });
}

int fx_cp_dist_phase(fx_ctx* ctx, const fx_layout* lay, const fx_step_args* a, int32_t phase,
                     int32_t ranks, int32_t self, const fx_cp_peer* peers, uint64_t stamp,
                     float* approx, int64_t approx_stride) {
    return guarded([&] {
        NvtxRange nv("fx_cp_dist_phase");
        DeviceGuard g(ctx);
        check_layout(lay);
        const fx_layout& L = *lay;
        FX_REQUIRE(a && a->q && a->plan_blk && a->plan_budgets && a->plan_kblocks && a->sel_bits && peers &&
                       approx,
                   FX_ERR_STATE, "no-context: distributed selection has no payload");
        FX_REQUIRE(phase >= 0 && phase <= 3, FX_ERR_INVALID, "bad-shape: unknown phase");
        FX_REQUIRE(L.l_cpu > 0, FX_ERR_INVALID, "empty-context: shard has no cpu rows");
        FX_REQUIRE(approx_stride >= fx::level_blocks(L.l_cpu, 16), FX_ERR_INVALID,
                   "bad-shape: approx_stride below the shard's block count");
        const int64_t l_plan = a->l_cpu_total > 0 ? a->l_cpu_total : L.l_cpu;
        FX_REQUIRE(a->cpu_offset >= 0 && a->cpu_offset % 128 == 0 && a->cpu_offset + L.l_cpu <= l_plan,
                   FX_ERR_INVALID, "bad-shape: shard [cpu_offset, +l_cpu) outside l_cpu_total or unaligned");
        if (phase == 0) {
            for (int i = 0; i < 4; ++i)
                FX_REQUIRE(a->meta[i] != nullptr, FX_ERR_STATE, "no-context: missing block metadata");
            FX_REQUIRE(a->absmax != nullptr, FX_ERR_STATE, "no-context: missing absmax");
            const int grid = fx::attend_grid(L, false, ctx->num_sms);
            StepScratch s = carve_step(ctx, L, grid, true);
            fx::launch_prepare(L, l_plan, a->plan_mode, a->fixed_block_size, a->fixed_budget, a->bgt0,
                               a->kslope, a->streaming, a->plan_blk, a->plan_budgets, a->plan_volume,
                               a->plan_cand_volumes, a->plan_kblocks, s.bg_done, ctx->stream,
                               fx::AppendArgs(), static_cast<int32_t*>(ctx->errw.p));
            fx::launch_approx_scores(L, a->meta, a->q, a->plan_blk, a->plan_kblocks, approx, approx_stride,
                                     ctx->num_sms, ctx->stream, /*rank_all=*/true);
            ctx->launches += 2;
        }
        fx::launch_cp_dist_phase(L, phase, ranks, self, peers, stamp, approx, approx_stride, a->q, a->absmax,
                                 a->meta, a->plan_blk, a->plan_kblocks, l_plan, a->cpu_offset, a->sel_bits,
                                 a->sel_words, ctx->stream);
        ctx->launches += 1;
    });
}

int fx_cp_combine_peer(fx_ctx* ctx, int32_t ranks, int64_t n, int32_t dim, const fx_cp_peer* peers,
                       uint64_t stamp, float* o, float* lse) {
    return guarded([&] {
        NvtxRange nv("fx_cp_combine_peer");
        DeviceGuard g(ctx);
        FX_REQUIRE(peers && o && n >= 0 && dim > 0, FX_ERR_INVALID, "bad-shape: peer combine input");
        fx::launch_cp_combine_peer(ranks, n, dim, peers, stamp, o, lse, ctx->stream);
        ctx->launches += n > 0 ? 1 : 0;
    });
}

int fx_ipc_handle(const void* dptr, unsigned char handle[64], int64_t* offset) {
    return guarded([&] {
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        // the handle names the whole allocation: export its base and the offset
        // of dptr inside it (caching allocators hand out sub-ranges)
        typedef CUresult (*RangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
        static RangeFn range = nullptr;
        if (!range) {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            FX_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
            FX_REQUIRE(fn && q == cudaDriverEntryPointSuccess, FX_ERR_CUDA,
                       "cuda-error: cuMemGetAddressRange unavailable");
            range = reinterpret_cast<RangeFn>(fn);
        }
        CUdeviceptr base = 0;
        size_t size = 0;
        FX_REQUIRE(range(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) == CUDA_SUCCESS, FX_ERR_CUDA,
                   "cuda-error: not a device allocation");
        cudaIpcMemHandle_t h;
        FX_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
        std::memcpy(handle, &h, 64);
        if (offset) *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(dptr) - base);
    });
}

int fx_ipc_open(fx_ctx* ctx, const unsigned char handle[64], void** dptr) {
    return guarded([&] {
        DeviceGuard g(ctx);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, 64);
        FX_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

int fx_ipc_close(fx_ctx* ctx, void* dptr) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_CUDA(cudaIpcCloseMemHandle(dptr));
    });
}

int fx_cp_combine(fx_ctx* ctx, int32_t ranks, int64_t n, int32_t dim, const float* o_parts,
                  const float* lse_parts, float* o, float* lse) {
    return guarded([&] {
        DeviceGuard g(ctx);
        FX_REQUIRE(ranks >= 1 && n >= 0 && dim > 0, FX_ERR_INVALID, "bad-shape: combine input");
        fx::launch_cp_combine(ranks, n, dim, o_parts, lse_parts, o, lse, ctx->stream);
        ctx->launches += n > 0 ? 1 : 0;
    });
}

}  // extern "C"
