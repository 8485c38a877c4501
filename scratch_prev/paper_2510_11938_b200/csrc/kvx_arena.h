// kvx_arena.h -- per-device caching allocator for transition state.
//
// A refactor grants, uses and releases a handle per transition; the engine
// does this at every granularity switch.  cudaMalloc/cudaFree (cudaFree
// synchronises the device) and pinned cudaMallocHost/cudaFreeHost would
// otherwise dominate a short transition's end-to-end time, so handles draw
// their device buffers, pinned staging and events from this cache and give
// them back on kvx_destroy (after their stream drained).  Size classes are
// powers of two >= 256 B.  Pools (the KV itself) are NOT cached here: they
// are long-lived and owned by the serving engine.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

namespace kvx {

inline size_t size_class(size_t bytes) {
    size_t c = 256;
    while (c < bytes) c <<= 1;
    return c;
}

class Arena {
public:
    static Arena& of(int device) {
        static std::mutex mu;
        static std::map<int, Arena*> all;
        std::lock_guard<std::mutex> lk(mu);
        auto it = all.find(device);
        if (it == all.end()) it = all.emplace(device, new Arena()).first;  // process lifetime
        return *it->second;
    }

    cudaError_t dev_alloc(void** p, size_t bytes) {
        const size_t c = size_class(bytes);
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto& v = dev_[c];
            if (!v.empty()) {
                *p = v.back();
                v.pop_back();
                return cudaSuccess;
            }
        }
        return cudaMalloc(p, c);
    }
    void dev_free(void* p, size_t bytes) {
        if (!p) return;
        std::lock_guard<std::mutex> lk(mu_);
        dev_[size_class(bytes)].push_back(p);
    }
    cudaError_t host_alloc(void** p, size_t bytes) {
        const size_t c = size_class(bytes);
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto& v = host_[c];
            if (!v.empty()) {
                *p = v.back();
                v.pop_back();
                return cudaSuccess;
            }
        }
        return cudaMallocHost(p, c);
    }
    void host_free(void* p, size_t bytes) {
        if (!p) return;
        std::lock_guard<std::mutex> lk(mu_);
        host_[size_class(bytes)].push_back(p);
    }
    cudaError_t event(cudaEvent_t* e, bool timing) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto& v = timing ? ev_t_ : ev_n_;
            if (!v.empty()) {
                *e = v.back();
                v.pop_back();
                return cudaSuccess;
            }
        }
        return timing ? cudaEventCreate(e) : cudaEventCreateWithFlags(e, cudaEventDisableTiming);
    }
    void event_free(cudaEvent_t e, bool timing) {
        if (!e) return;
        std::lock_guard<std::mutex> lk(mu_);
        (timing ? ev_t_ : ev_n_).push_back(e);
    }

private:
    std::mutex mu_;
    std::unordered_map<size_t, std::vector<void*>> dev_, host_;
    std::vector<cudaEvent_t> ev_t_, ev_n_;
};

}  // namespace kvx
