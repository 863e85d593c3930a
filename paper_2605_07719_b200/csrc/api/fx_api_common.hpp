// Internal helpers of the C++ drop-in: device buffers through the C-ABI.
#pragma once

#include <cstring>
#include <span>
#include <vector>

#include "fluxattn/b200.hpp"

namespace fluxattn::b200 {

// Device allocation owned by the calling thread's context.
class DevMem {
public:
    explicit DevMem(std::size_t bytes) : n_(bytes) { check(fx_malloc(context(), bytes ? bytes : 1, &p_)); }
    template <class T>
    explicit DevMem(std::span<const T> host) : DevMem(host.size_bytes()) {
        if (!host.empty()) check(fx_memcpy_h2d(context(), p_, host.data(), host.size_bytes()));
    }
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    ~DevMem() {
        if (p_) fx_free(context(), p_);
    }
    void* get() const { return p_; }
    template <class T>
    T* as() const {
        return static_cast<T*>(p_);
    }
    template <class T>
    std::vector<T> download(std::size_t count) const {
        std::vector<T> out(count);
        if (count) check(fx_memcpy_d2h(context(), out.data(), p_, count * sizeof(T)));
        return out;
    }

private:
    void* p_ = nullptr;
    std::size_t n_ = 0;
};

}  // namespace fluxattn::b200
