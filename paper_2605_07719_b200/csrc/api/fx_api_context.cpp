// Per-thread C-ABI context of the C++ drop-in.
#include <atomic>
#include <cstdlib>

#include "fluxattn/b200.hpp"
#include "fx_api_arena.hpp"

namespace fluxattn::b200 {
namespace {
std::atomic<int> g_device{-1};

// One per host thread: the C-ABI context and the device-resident caches made
// through it (released before the context).
struct ThreadCtx {
    fx_ctx* ctx = nullptr;
    int device = -1;
    std::map<ArenaShape, std::unique_ptr<Arena>> arenas;
    void* staging = nullptr;
    std::size_t staging_bytes = 0;
    ~ThreadCtx() {
        try {
            arenas.clear();
            if (ctx && staging) fx_free(ctx, staging);
        } catch (...) {
        }
        if (ctx) fx_ctx_destroy(ctx);
    }
};
thread_local ThreadCtx t_ctx;

int device_index() {
    int d = g_device.load();
    if (d < 0) {
        const char* env = std::getenv("FLUXATTN_DEVICE");
        d = env ? std::atoi(env) : 0;
    }
    return d;
}
}  // namespace

fx_ctx* context() {
    const int d = device_index();
    if (!t_ctx.ctx || t_ctx.device != d) {
        t_ctx.arenas.clear();
        if (t_ctx.ctx && t_ctx.staging) fx_free(t_ctx.ctx, t_ctx.staging);
        t_ctx.staging = nullptr;
        t_ctx.staging_bytes = 0;
        if (t_ctx.ctx) fx_ctx_destroy(t_ctx.ctx);
        t_ctx.ctx = nullptr;
        check(fx_ctx_create(d, &t_ctx.ctx));
        t_ctx.device = d;
    }
    return t_ctx.ctx;
}

void set_device(int device) { g_device.store(device); }

std::map<ArenaShape, std::unique_ptr<Arena>>& thread_arenas() { return t_ctx.arenas; }

float* thread_staging(std::size_t bytes) {
    if (bytes > t_ctx.staging_bytes) {
        if (t_ctx.staging) check(fx_free(context(), t_ctx.staging));
        t_ctx.staging = nullptr;
        t_ctx.staging_bytes = 0;
        check(fx_malloc(context(), bytes, &t_ctx.staging));
        t_ctx.staging_bytes = bytes;
    }
    return static_cast<float*>(t_ctx.staging);
}

}  // namespace fluxattn::b200
