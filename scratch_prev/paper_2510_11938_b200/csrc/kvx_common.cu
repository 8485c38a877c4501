// kvx_common.cu -- library-wide state: the thread-local error message, the
// launch counter, version / device queries and the hooks kvx_ctl.cpp uses.
#include "kvx_common.h"

#include <mutex>
#include <set>

namespace kvx_host {
std::string& last_error() {
    thread_local std::string msg;
    return msg;
}
std::atomic<uint64_t>& launches() {
    static std::atomic<uint64_t> n{0};
    return n;
}
int ensure_loaded(int device) {
    static std::mutex mu;
    static std::set<int> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count(device)) return KVX_OK;
    DeviceGuard dg(device);
    if (!dg.ok) return fail(KVX_ECUDA, "cudaSetDevice failed");
    for (auto fn : {preload_transition_kernels, preload_pool_kernels, preload_extras_kernels}) {
        const cudaError_t e = fn();
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(KVX_ECUDA, std::string("kernel preload: ") + cudaGetErrorString(e));
        }
    }
    done.insert(device);
    return KVX_OK;
}
}  // namespace kvx_host

using namespace kvx_host;

extern "C" {

const char* kvx_last_error(void) { return last_error().c_str(); }
int kvx_abi_version(void) { return KVX_ABI_VERSION; }
uint64_t kvx_launch_count(void) { return launches().load(); }

int kvx_preload(int32_t device) { return ensure_loaded(device); }

int kvx_device_count(int32_t* out) {
    if (!out) return fail(KVX_EINVAL, "out is null");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *out = 0;
        return fail(KVX_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    }
    *out = n;
    return KVX_OK;
}

}  // extern "C"

// ----------------------------------------------- hooks for kvx_ctl.cpp
namespace kvx {
CtlState& ctl_of(kvx_transition* t) { return t->ctl; }
const CtlState& ctl_of(const kvx_transition* t) { return t->ctl; }
uint64_t epoch_of(const kvx_transition* t) { return t->epoch; }
int set_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace kvx
