// Per-thread C-ABI context of the C++ drop-in.
#include <atomic>
#include <cstdlib>

#include "fluxattn/b200.hpp"

namespace fluxattn::b200 {
namespace {
std::atomic<int> g_device{-1};

struct ThreadCtx {
    fx_ctx* ctx = nullptr;
    int device = -1;
    ~ThreadCtx() {
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
        if (t_ctx.ctx) fx_ctx_destroy(t_ctx.ctx);
        t_ctx.ctx = nullptr;
        check(fx_ctx_create(d, &t_ctx.ctx));
        t_ctx.device = d;
    }
    return t_ctx.ctx;
}

void set_device(int device) { g_device.store(device); }

}  // namespace fluxattn::b200
