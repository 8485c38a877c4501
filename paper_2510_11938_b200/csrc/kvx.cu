// kvx.cu -- host side of the C-ABI (include/kvx.h): pools, transitions,
// waves, commit/abort.  Device code lives in kvx_kernels.cuh.
//
// One handle == one transition of one pipeline instance on one local GPU
// (RefactorCtx, /root/reference/proj/include/pipesim/engine.hpp:149-158).
// In a multi-GPU transition every rank opens its own handle over the same
// plans; each moves the layers whose OLD stage lives on its GPU and pushes
// them into the destination pools (local, or a peer's through NVLink P2P).
// The destination block rule is deterministic, so every rank derives the same
// destination block table without exchanging it.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kvx.h"
#include "kvx_arena.h"
#include "kvx_internal.h"
#include "kvx_kernels.cuh"

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define KVX_CUDA(call)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(KVX_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
    } while (0)

#define KVX_LAUNCHED()                                                                    \
    do {                                                                                  \
        g_launches.fetch_add(1, std::memory_order_relaxed);                               \
        cudaError_t e_ = cudaGetLastError();                                              \
        if (e_ != cudaSuccess)                                                            \
            return fail(KVX_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
    } while (0)

// Restores the caller's current device (torch keeps its own notion of it).
struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

bool geometry_ok(const kvx_geometry* g, std::string* why) {
    if (!g) return *why = "geometry is null", false;
    if (g->num_layers < 1 || g->num_kv_heads < 1 || g->head_dim < 1 || g->elem_bytes < 1 ||
        g->block_tokens < 1)
        return *why = "geometry fields must be positive", false;
    const uint64_t tb = (uint64_t)g->num_kv_heads * g->head_dim * g->elem_bytes;
    if (tb % 16 != 0) return *why = "token_bytes must be a multiple of 16", false;
    return true;
}

uint64_t token_bytes(const kvx_geometry& g) {
    return (uint64_t)g.num_kv_heads * (uint64_t)g.head_dim * (uint64_t)g.elem_bytes;
}
uint64_t block_bytes(const kvx_geometry& g) { return 2ull * (uint64_t)g.block_tokens * token_bytes(g); }

int64_t cdiv64(int64_t a, int64_t b) { return (a + b - 1) / b; }

int stage_of_layer(const std::vector<int32_t>& b, int32_t layer) {  // modelgraph.cpp:55-62
    int s = 0;
    for (int32_t cut : b) {
        if (layer < cut) break;
        ++s;
    }
    return s;
}
int stage_begin(const std::vector<int32_t>& b, int s) { return s == 0 ? 0 : b[(size_t)s - 1]; }

bool plan_ok(const kvx_plan& p, int32_t L, std::string* why, std::vector<int32_t>* out) {
    if (p.num_stages < 1 || p.num_stages > L) return *why = "num_stages out of range", false;
    out->assign(p.boundaries, p.boundaries + (p.num_stages - 1));
    int32_t prev = 0;
    for (int32_t b : *out) {
        if (b <= prev || b >= L) return *why = "boundaries must be strictly increasing in (0, L)", false;
        prev = b;
    }
    if (!p.pools) return *why = "plan pools array is null", false;
    return true;
}

}  // namespace

namespace {
struct PieceRelease {  // returns a call's descriptor buffers to the arena once the stream passed them
    int device;
    void* d;
    void* h;
    size_t bytes;
};
void CUDART_CB release_pieces(void* arg) {
    auto* r = static_cast<PieceRelease*>(arg);
    kvx::Arena& A = kvx::Arena::of(r->device);
    A.dev_free(r->d, r->bytes);
    A.host_free(r->h, r->bytes);
    delete r;
}
}  // namespace

// ---------------------------------------------------------- bulk variants
// (ring depth, chunk bytes) of the TMA bulk mover; selectable with
// KVX_BULK_CFG=<index> for tuning, index 0 is the default.
namespace {
using BulkFn = void (*)(const kvx::Seg*, int32_t, const kvx::LayerPtr*, int32_t, uint64_t, uint64_t, int32_t,
                        int32_t, int32_t);
struct BulkVariant {
    int stages;
    uint32_t chunk;
    BulkFn fn;
};
const BulkVariant kBulkVariants[] = {
    {6, 32768, kvx::kvx_bulk_kernel<6, 32768>},  {4, 49152, kvx::kvx_bulk_kernel<4, 49152>},
    {3, 65536, kvx::kvx_bulk_kernel<3, 65536>},  {12, 16384, kvx::kvx_bulk_kernel<12, 16384>},
    {3, 32768, kvx::kvx_bulk_kernel<3, 32768>},  {8, 16384, kvx::kvx_bulk_kernel<8, 16384>},
    {2, 65536, kvx::kvx_bulk_kernel<2, 65536>},  {4, 16384, kvx::kvx_bulk_kernel<4, 16384>},
};
constexpr int kNumBulkVariants = sizeof(kBulkVariants) / sizeof(kBulkVariants[0]);
}  // namespace

// ------------------------------------------------------------------ types
struct kvx_pool {
    int32_t device = -1;
    bool imported = false;
    bool wrapped = false;  // caller-owned memory
    char* base = nullptr;
    uint64_t bytes = 0;
    kvx_geometry g{};
    int32_t num_layers = 0;
    int32_t num_blocks = 0;
};

// Device-resident block manager: a free-id stack on the GPU, its top mirrored
// on the host so every capacity decision is synchronous and deterministic.
struct kvx_blockmgr {
    int32_t device = -1;
    int32_t capacity = 0;
    int32_t top = 0;          // free blocks (host mirror of the device stack top)
    int32_t* d_stack = nullptr;
};

struct kvx_transition {
    kvx_geometry g{};
    int32_t device = -1;
    cudaStream_t stream = nullptr;
    bool own_stream = true;
    int num_sms = 0;
    int move_ctas_per_sm = 1;
    int bulk_ctas[16] = {};  // resident CTAs per SM of each bulk variant
    int bulk_variant = -1;   // -1: chosen per wave from the average run size
    bool use_bulk = false;   // TMA bulk mover for local destinations
    bool peer_bulk = false;  // ... and for peer (NVLink) destinations
    std::vector<int32_t> old_b, new_b;
    std::vector<kvx_pool*> old_pools, new_pools;
    int32_t max_requests = 0, max_blocks = 0, dst_num_blocks = 0;
    kvx_blockmgr* bm = nullptr;  // destination block manager (NULL: bump rule)
    uint64_t epoch = 0;
    enum State { kActive, kCommitPending, kCommitted, kAborted } state = kActive;

    // device state
    int32_t* d_src_bt = nullptr;
    int32_t* d_dst_bt = nullptr;
    int64_t* d_synced_hi = nullptr;
    kvx::LayerPtr* d_layers = nullptr;
    int32_t n_local_layers = 0;
    int32_t n_peer_layers = 0;  // layers [0, n_peer_layers) of d_layers push to a peer
    bool has_peer_dst = false;
    // wave staging: pinned host ring of 2 + device buffer
    char* h_wave[2] = {nullptr, nullptr};
    cudaEvent_t h_wave_free[2] = {nullptr, nullptr};
    int wave_slot = 0;
    char* d_wave = nullptr;
    kvx::Seg* d_segs = nullptr;
    int64_t seg_cap = 0;
    // commit scratch
    uint8_t* d_live = nullptr;
    int32_t* d_commit_i32 = nullptr;  // row_ptr | blocks | free_list
    int64_t commit_i32_cap = 0;
    size_t bt_bytes = 0, wave_bytes = 0, layers_bytes = 0;
    int64_t* d_commit_out = nullptr;
    // pinned landing zone of an async commit: [int64 x4 | row_ptr | blocks | free]
    char* h_commit = nullptr;
    size_t h_commit_bytes = 0;
    cudaEvent_t ev_commit = nullptr;
    int32_t pend_n_live = 0;
    int64_t pend_nb_live = 0, pend_nb_free = 0;
    // timing
    cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
    bool timing_open = false;
    // one (start, end) event pair per move-kernel launch of this handle
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> move_ev;
    std::vector<uint64_t> move_bytes;

    // activation handoff pieces (grown on demand, freed at destroy)
    kvx::Piece* d_pieces = nullptr;
    kvx::Piece* h_pieces = nullptr;
    int64_t piece_cap = 0;
    cudaEvent_t pieces_free = nullptr;

    // host mirror of the destination rule (capacity checks are synchronous)
    std::vector<int64_t> synced_hi;
    std::vector<int32_t> src_bt;  // host copy: every wave's source blocks must be backed
    int32_t alloc = 0;
    uint64_t bytes_moved = 0;       // by this handle (local-source layers)
    uint64_t bytes_all_layers = 0;  // reference-accounted, all layers

    kvx::CtlState ctl;  // control-plane mirror (kvx_ctl.cpp)
};

extern "C" {

const char* kvx_last_error(void) { return g_last_error.c_str(); }
int kvx_abi_version(void) { return KVX_ABI_VERSION; }
uint64_t kvx_launch_count(void) { return g_launches.load(); }

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

// ------------------------------------------------------------------ pools
int kvx_pool_create(int32_t device, const kvx_geometry* g, int32_t num_layers, int32_t num_blocks,
                    kvx_pool** out) {
    std::string why;
    if (!out) return fail(KVX_EINVAL, "out is null");
    *out = nullptr;
    if (!geometry_ok(g, &why)) return fail(KVX_EINVAL, why);
    if (num_layers < 1 || num_blocks < 1) return fail(KVX_EINVAL, "num_layers/num_blocks must be >= 1");
    DeviceGuard dg(device);
    if (!dg.ok) return fail(KVX_ECUDA, "cudaSetDevice failed for pool device");
    auto* p = new kvx_pool;
    p->device = device;
    p->g = *g;
    p->num_layers = num_layers;
    p->num_blocks = num_blocks;
    p->bytes = (uint64_t)num_layers * (uint64_t)num_blocks * block_bytes(*g);
    cudaError_t e = cudaMalloc(&p->base, p->bytes);
    if (e != cudaSuccess) {
        delete p;
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? KVX_ENOSPC : KVX_ECUDA,
                    std::string("pool cudaMalloc: ") + cudaGetErrorString(e));
    }
    *out = p;
    return KVX_OK;
}

int kvx_pool_wrap(int32_t device, void* ptr, uint64_t bytes, const kvx_geometry* g, int32_t num_layers,
                  int32_t num_blocks, kvx_pool** out) {
    std::string why;
    if (!out) return fail(KVX_EINVAL, "out is null");
    *out = nullptr;
    if (!geometry_ok(g, &why)) return fail(KVX_EINVAL, why);
    if (!ptr || (reinterpret_cast<uintptr_t>(ptr) & 15)) return fail(KVX_EINVAL, "ptr must be 16-byte aligned");
    if (num_layers < 1 || num_blocks < 1) return fail(KVX_EINVAL, "num_layers/num_blocks must be >= 1");
    const uint64_t need = (uint64_t)num_layers * (uint64_t)num_blocks * block_bytes(*g);
    if (bytes < need) return fail(KVX_EINVAL, "wrapped buffer smaller than the pool");
    auto* p = new kvx_pool;
    p->device = device;
    p->wrapped = true;
    p->base = static_cast<char*>(ptr);
    p->g = *g;
    p->num_layers = num_layers;
    p->num_blocks = num_blocks;
    p->bytes = need;
    *out = p;
    return KVX_OK;
}

int kvx_pool_export(const kvx_pool* p, uint8_t handle[KVX_IPC_HANDLE_BYTES]) {
    if (!p || !handle || p->imported) return fail(KVX_EINVAL, "export needs a local pool");
    static_assert(sizeof(cudaIpcMemHandle_t) == KVX_IPC_HANDLE_BYTES, "ipc handle size");
    DeviceGuard dg(p->device);
    cudaIpcMemHandle_t h;
    KVX_CUDA(cudaIpcGetMemHandle(&h, p->base));
    std::memcpy(handle, &h, sizeof(h));
    return KVX_OK;
}

int kvx_pool_import(int32_t device, const uint8_t handle[KVX_IPC_HANDLE_BYTES],
                    const kvx_geometry* g, int32_t num_layers, int32_t num_blocks, kvx_pool** out) {
    std::string why;
    if (!out || !handle) return fail(KVX_EINVAL, "null argument");
    *out = nullptr;
    if (!geometry_ok(g, &why)) return fail(KVX_EINVAL, why);
    DeviceGuard dg(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* ptr = nullptr;
    KVX_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    auto* p = new kvx_pool;
    p->device = device;
    p->imported = true;
    p->base = static_cast<char*>(ptr);
    p->g = *g;
    p->num_layers = num_layers;
    p->num_blocks = num_blocks;
    p->bytes = (uint64_t)num_layers * (uint64_t)num_blocks * block_bytes(*g);
    *out = p;
    return KVX_OK;
}

int kvx_pool_info(const kvx_pool* p, void** dptr, uint64_t* bytes, int32_t* device,
                  int32_t* imported) {
    if (!p) return fail(KVX_EINVAL, "pool is null");
    if (dptr) *dptr = p->base;
    if (bytes) *bytes = p->bytes;
    if (device) *device = p->device;
    if (imported) *imported = p->imported ? 1 : 0;
    return KVX_OK;
}

int kvx_pool_destroy(kvx_pool* p) {
    if (!p) return KVX_OK;
    DeviceGuard dg(p->device);
    cudaError_t e = p->wrapped ? cudaSuccess : p->imported ? cudaIpcCloseMemHandle(p->base) : cudaFree(p->base);
    delete p;
    if (e != cudaSuccess) return fail(KVX_ECUDA, std::string("pool free: ") + cudaGetErrorString(e));
    return KVX_OK;
}

int kvx_pool_zero(kvx_pool* p) {
    if (!p) return fail(KVX_EINVAL, "pool is null");
    DeviceGuard dg(p->device);
    KVX_CUDA(cudaMemset(p->base, 0, p->bytes));
    KVX_CUDA(cudaDeviceSynchronize());
    return KVX_OK;
}

int kvx_pool_read(const kvx_pool* p, uint64_t offset, uint64_t bytes, void* host) {
    if (!p || !host || offset + bytes > p->bytes) return fail(KVX_EINVAL, "read out of range");
    DeviceGuard dg(p->device);
    KVX_CUDA(cudaMemcpy(host, p->base + offset, bytes, cudaMemcpyDeviceToHost));
    return KVX_OK;
}

int kvx_pool_write(kvx_pool* p, uint64_t offset, uint64_t bytes, const void* host) {
    if (!p || !host || offset + bytes > p->bytes) return fail(KVX_EINVAL, "write out of range");
    DeviceGuard dg(p->device);
    KVX_CUDA(cudaMemcpy(p->base + offset, host, bytes, cudaMemcpyHostToDevice));
    return KVX_OK;
}

int kvx_pool_fill_pattern(kvx_pool* p, uint64_t seed, int32_t first_layer, int32_t n,
                          const int32_t* req, const int64_t* tokens, const int32_t* bt,
                          int32_t max_requests, int32_t max_blocks) {
    if (!p || p->imported) return fail(KVX_EINVAL, "fill needs a local pool");
    if (n < 0 || (n > 0 && (!req || !tokens || !bt))) return fail(KVX_EINVAL, "null arrays");
    if (n == 0) return KVX_OK;
    int64_t max_tok = 0;
    for (int32_t i = 0; i < n; ++i) {
        if (req[i] < 0 || req[i] >= max_requests) return fail(KVX_EINVAL, "req out of range");
        if (tokens[i] < 0 || cdiv64(tokens[i], p->g.block_tokens) > max_blocks)
            return fail(KVX_EINVAL, "tokens exceed max_blocks");
        max_tok = std::max(max_tok, tokens[i]);
        for (int64_t b = 0; b < cdiv64(tokens[i], p->g.block_tokens); ++b) {
            const int32_t id = bt[(int64_t)req[i] * max_blocks + b];
            if (id < 0 || id >= p->num_blocks) return fail(KVX_EINVAL, "block id out of pool range");
        }
    }
    if (max_tok == 0) return KVX_OK;
    DeviceGuard dg(p->device);
    kvx::Arena& A = kvx::Arena::of(p->device);
    const size_t bt_bytes = sizeof(int32_t) * (size_t)max_requests * (size_t)max_blocks;
    struct Scratch {  // released on every return path
        kvx::Arena& a;
        void *req = nullptr, *tok = nullptr, *bt = nullptr;
        size_t nreq, ntok, nbt;
        ~Scratch() {
            a.dev_free(req, nreq);
            a.dev_free(tok, ntok);
            a.dev_free(bt, nbt);
        }
    } sc{A, nullptr, nullptr, nullptr, sizeof(int32_t) * n, sizeof(int64_t) * n, bt_bytes};
    KVX_CUDA(A.dev_alloc(&sc.req, sc.nreq));
    KVX_CUDA(A.dev_alloc(&sc.tok, sc.ntok));
    KVX_CUDA(A.dev_alloc(&sc.bt, sc.nbt));
    KVX_CUDA(cudaMemcpy(sc.req, req, sc.nreq, cudaMemcpyHostToDevice));
    KVX_CUDA(cudaMemcpy(sc.tok, tokens, sc.ntok, cudaMemcpyHostToDevice));
    KVX_CUDA(cudaMemcpy(sc.bt, bt, sc.nbt, cudaMemcpyHostToDevice));
    dim3 grid((unsigned)n, (unsigned)cdiv64(max_tok, p->g.block_tokens));
    kvx::kvx_fill_kernel<<<grid, 256>>>(p->base, p->num_blocks, first_layer, p->num_layers,
                                        static_cast<const int32_t*>(sc.req), static_cast<const int64_t*>(sc.tok),
                                        static_cast<const int32_t*>(sc.bt), max_blocks, p->g.block_tokens,
                                        token_bytes(p->g), seed);
    KVX_LAUNCHED();
    KVX_CUDA(cudaDeviceSynchronize());
    return KVX_OK;
}

int kvx_pool_append_pattern(kvx_pool* p, void* stream, uint64_t seed, int32_t first_layer, int32_t n,
                            const int32_t* req, const int64_t* from, const int64_t* to, const int32_t* bt,
                            int32_t max_requests, int32_t max_blocks) {
    if (!p || p->imported) return fail(KVX_EINVAL, "append needs a local pool");
    if (n < 0 || (n > 0 && (!req || !from || !to || !bt))) return fail(KVX_EINVAL, "null arrays");
    int64_t max_tok = 0;
    for (int32_t i = 0; i < n; ++i) {
        if (req[i] < 0 || req[i] >= max_requests || from[i] < 0 || to[i] < from[i])
            return fail(KVX_EINVAL, "bad append entry");
        if (cdiv64(to[i], p->g.block_tokens) > max_blocks) return fail(KVX_EINVAL, "tokens exceed max_blocks");
        for (int64_t b = from[i] / p->g.block_tokens; b < cdiv64(to[i], p->g.block_tokens); ++b) {
            const int32_t id = bt[(int64_t)req[i] * max_blocks + b];
            if (id < 0 || id >= p->num_blocks) return fail(KVX_EINVAL, "block id out of pool range");
        }
        max_tok = std::max(max_tok, to[i]);
    }
    if (n == 0 || max_tok == 0) return KVX_OK;
    DeviceGuard dg(p->device);
    kvx::Arena& A = kvx::Arena::of(p->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // one scratch region [req | from | to | bt], freed after the stream passes it
    const size_t o_from = ((sizeof(int32_t) * (size_t)n) + 15) & ~size_t(15);
    const size_t o_to = o_from + sizeof(int64_t) * (size_t)n;
    const size_t o_bt = o_to + sizeof(int64_t) * (size_t)n;
    const size_t bytes = o_bt + sizeof(int32_t) * (size_t)max_requests * (size_t)max_blocks;
    void *d = nullptr, *h = nullptr;
    KVX_CUDA(A.dev_alloc(&d, bytes));
    KVX_CUDA(A.host_alloc(&h, bytes));
    char* hc = static_cast<char*>(h);
    std::memcpy(hc, req, sizeof(int32_t) * (size_t)n);
    std::memcpy(hc + o_from, from, sizeof(int64_t) * (size_t)n);
    std::memcpy(hc + o_to, to, sizeof(int64_t) * (size_t)n);
    std::memcpy(hc + o_bt, bt, bytes - o_bt);
    KVX_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
    char* dc = static_cast<char*>(d);
    dim3 grid((unsigned)n, (unsigned)cdiv64(max_tok, p->g.block_tokens));
    kvx::kvx_fill_kernel<<<grid, 256, 0, st>>>(p->base, p->num_blocks, first_layer, p->num_layers,
                                               reinterpret_cast<const int32_t*>(dc),
                                               reinterpret_cast<const int64_t*>(dc + o_to),
                                               reinterpret_cast<const int32_t*>(dc + o_bt), max_blocks,
                                               p->g.block_tokens, token_bytes(p->g), seed,
                                               reinterpret_cast<const int64_t*>(dc + o_from));
    KVX_LAUNCHED();
    KVX_CUDA(cudaLaunchHostFunc(st, release_pieces, new PieceRelease{p->device, d, h, bytes}));
    return KVX_OK;
}

// ------------------------------------------------------------- transition
int kvx_begin(const kvx_transition_desc* d, kvx_transition** out) {
    std::string why;
    if (!out || !d) return fail(KVX_EINVAL, "null argument");
    *out = nullptr;
    if (!geometry_ok(&d->geometry, &why)) return fail(KVX_EINVAL, why);
    const kvx_geometry& g = d->geometry;
    std::vector<int32_t> ob, nb;
    if (!plan_ok(d->old_plan, g.num_layers, &why, &ob)) return fail(KVX_EINVAL, "old plan: " + why);
    if (!plan_ok(d->new_plan, g.num_layers, &why, &nb)) return fail(KVX_EINVAL, "new plan: " + why);
    if (d->max_requests < 1 || d->max_blocks < 1 || d->dst_num_blocks < 1)
        return fail(KVX_EINVAL, "max_requests/max_blocks/dst_num_blocks must be >= 1");
    if (!d->src_block_table) return fail(KVX_EINVAL, "src_block_table is null");
    for (int k = 0; k < d->new_plan.num_stages; ++k) {
        const kvx_pool* p = d->new_plan.pools[k];
        if (!p) {
            if (d->pull) continue;  // pull: only the local new pools are written here
            return fail(KVX_EINVAL, "every new-stage pool is required");
        }
        const int32_t layers = (k + 1 < d->new_plan.num_stages ? nb[(size_t)k] : g.num_layers) -
                               stage_begin(nb, k);
        if (p->num_layers != layers) return fail(KVX_EINVAL, "new pool layer count != stage layer range");
        if (p->num_blocks < d->dst_num_blocks) return fail(KVX_EINVAL, "new pool smaller than dst_num_blocks");
        if (!p->imported && p->device != d->device) return fail(KVX_EINVAL, "local new pool on another device");
        if (p->imported && p->device != d->device) return fail(KVX_EINVAL, "imported pool mapped for another device");
        if (p->g.num_kv_heads != g.num_kv_heads || p->g.head_dim != g.head_dim ||
            p->g.elem_bytes != g.elem_bytes || p->g.block_tokens != g.block_tokens)
            return fail(KVX_EINVAL, "new pool geometry mismatch");
    }
    for (int k = 0; k < d->old_plan.num_stages; ++k) {
        const kvx_pool* p = d->old_plan.pools[k];
        if (!p) continue;
        const int32_t layers = (k + 1 < d->old_plan.num_stages ? ob[(size_t)k] : g.num_layers) -
                               stage_begin(ob, k);
        if (p->num_layers != layers) return fail(KVX_EINVAL, "old pool layer count != stage layer range");
        if (p->g.num_kv_heads != g.num_kv_heads || p->g.head_dim != g.head_dim ||
            p->g.elem_bytes != g.elem_bytes || p->g.block_tokens != g.block_tokens)
            return fail(KVX_EINVAL, "old pool geometry mismatch");
    }
    if (d->dst_blockmgr) {
        const auto* bm = static_cast<const kvx_blockmgr*>(d->dst_blockmgr);
        if (bm->device != d->device) return fail(KVX_EINVAL, "block manager lives on another device");
        if (bm->capacity > d->dst_num_blocks) return fail(KVX_EINVAL, "block manager larger than the new pools");
    }
    // Validate the source table against the pools it will be read through.
    const size_t cells = (size_t)d->max_requests * (size_t)d->max_blocks;
    int32_t min_old_blocks = INT32_MAX;
    for (int k = 0; k < d->old_plan.num_stages; ++k)
        if (d->old_plan.pools[k]) min_old_blocks = std::min(min_old_blocks, d->old_plan.pools[k]->num_blocks);
    for (size_t c = 0; c < cells; ++c) {
        const int32_t v = d->src_block_table[c];
        if (v >= min_old_blocks) return fail(KVX_EINVAL, "src_block_table id beyond an old pool");
    }

    DeviceGuard dg(d->device);
    if (!dg.ok) return fail(KVX_ECUDA, "cudaSetDevice failed");
    auto* t = new kvx_transition;
    t->g = g;
    t->device = d->device;
    t->old_b = ob;
    t->new_b = nb;
    t->old_pools.assign(d->old_plan.pools, d->old_plan.pools + d->old_plan.num_stages);
    t->new_pools.assign(d->new_plan.pools, d->new_plan.pools + d->new_plan.num_stages);
    t->max_requests = d->max_requests;
    t->max_blocks = d->max_blocks;
    t->dst_num_blocks = d->dst_num_blocks;
    t->bm = static_cast<kvx_blockmgr*>(d->dst_blockmgr);
    t->epoch = d->epoch;
    t->synced_hi.assign((size_t)d->max_requests, 0);
    t->src_bt.assign(d->src_block_table, d->src_block_table + cells);
    t->ctl.init(d->max_requests, d->max_sync_rounds,
                d->kv_bytes_per_token > 0.0 ? d->kv_bytes_per_token
                                            : (double)g.num_layers * (double)block_bytes(g) /
                                                  (double)g.block_tokens);
    auto bail = [&](int code) {
        kvx_destroy(t);
        return code;
    };
    if (cudaDeviceGetAttribute(&t->num_sms, cudaDevAttrMultiProcessorCount, d->device) != cudaSuccess)
        return bail(fail(KVX_ECUDA, "query SM count"));
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kvx::kvx_move_kernel, kvx::kMoveThreads, 0) !=
        cudaSuccess)
        return bail(fail(KVX_ECUDA, "occupancy query"));
    t->move_ctas_per_sm = std::max(1, occ);
    {
        // -1 = per wave: 3 x 64 KiB ring for slab-sized runs (>= 64 KiB on
        // average, e.g. full 320 KiB 13B blocks), 6 x 32 KiB otherwise
        // (token-sized delta / final waves).  KVX_BULK_CFG pins one variant.
        const char* cfg = getenv("KVX_BULK_CFG");
        t->bulk_variant = cfg ? std::max(0, std::min(kNumBulkVariants - 1, atoi(cfg))) : -1;
        for (int v = 0; v < kNumBulkVariants; ++v) {
            const BulkVariant& bv = kBulkVariants[v];
            const int smem = bv.stages * (int)bv.chunk;
            if (cudaFuncSetAttribute(bv.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bv.fn, kvx::kBulkThreads, smem) != cudaSuccess)
                return bail(fail(KVX_ECUDA, "bulk kernel attributes"));
            t->bulk_ctas[v] = std::max(1, occ);
        }
        // Bulk (TMA engine) mover by default, for local and peer (NVLink)
        // destinations alike; KVX_PEER_BULK=0 keeps the LSU mover for peer
        // pushes, KVX_MOVE_IMPL=lsu everywhere.
        const char* impl = getenv("KVX_MOVE_IMPL");
        t->use_bulk = !(impl && std::string(impl) == "lsu");
        const char* pb = getenv("KVX_PEER_BULK");
        t->peer_bulk = t->use_bulk && !(pb && std::string(pb) == "0");
    }

    if (d->stream) {
        t->stream = static_cast<cudaStream_t>(d->stream);
        t->own_stream = false;
    } else if (cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking) != cudaSuccess) {
        return bail(fail(KVX_ECUDA, "stream create"));
    }
    kvx::Arena& A = kvx::Arena::of(d->device);
    if (A.event(&t->ev_begin, true) != cudaSuccess || A.event(&t->ev_end, true) != cudaSuccess)
        return bail(fail(KVX_ECUDA, "event create"));
    const size_t bt_bytes = sizeof(int32_t) * cells;
    const size_t wave_bytes = (size_t)d->max_requests * (sizeof(int32_t) + 2 * sizeof(int64_t)) + 64;
    t->bt_bytes = bt_bytes;
    t->wave_bytes = wave_bytes;
    if (A.dev_alloc((void**)&t->d_src_bt, bt_bytes) != cudaSuccess ||
        A.dev_alloc((void**)&t->d_dst_bt, bt_bytes) != cudaSuccess ||
        A.dev_alloc((void**)&t->d_synced_hi, sizeof(int64_t) * (size_t)d->max_requests) != cudaSuccess ||
        A.dev_alloc((void**)&t->d_wave, wave_bytes) != cudaSuccess ||
        A.dev_alloc((void**)&t->d_live, (size_t)d->max_requests) != cudaSuccess ||
        A.dev_alloc((void**)&t->d_commit_out, 4 * sizeof(int64_t)) != cudaSuccess)
        return bail(fail(KVX_ENOSPC, "transition state allocation failed"));
    for (int s = 0; s < 2; ++s)
        if (A.host_alloc((void**)&t->h_wave[s], wave_bytes) != cudaSuccess ||
            A.event(&t->h_wave_free[s], false) != cudaSuccess)
            return bail(fail(KVX_ECUDA, "pinned staging allocation failed"));
    if (cudaMemcpyAsync(t->d_src_bt, d->src_block_table, bt_bytes, cudaMemcpyHostToDevice, t->stream) !=
            cudaSuccess ||
        cudaMemsetAsync(t->d_dst_bt, 0xff, bt_bytes, t->stream) != cudaSuccess ||
        cudaMemsetAsync(t->d_synced_hi, 0, sizeof(int64_t) * (size_t)d->max_requests, t->stream) !=
            cudaSuccess)
        return bail(fail(KVX_ECUDA, "transition state init"));

    // Worst-case wave and commit buffers up front, so no allocation happens
    // between the grant and the commit (a wave has at most max_blocks
    // segments per request; commit needs row_ptr + live blocks + free list).
    {
        t->seg_cap = (int64_t)(kvx::size_class(sizeof(kvx::Seg) * cells) / sizeof(kvx::Seg));
        t->commit_i32_cap = (int64_t)(d->max_requests + 1) + 2 * (int64_t)cells;
        t->h_commit_bytes = 32 + sizeof(int32_t) * (size_t)t->commit_i32_cap;
        if (A.dev_alloc((void**)&t->d_segs, sizeof(kvx::Seg) * (size_t)t->seg_cap) != cudaSuccess ||
            A.dev_alloc((void**)&t->d_commit_i32, sizeof(int32_t) * (size_t)t->commit_i32_cap) != cudaSuccess ||
            A.host_alloc((void**)&t->h_commit, t->h_commit_bytes) != cudaSuccess ||
            A.event(&t->ev_commit, false) != cudaSuccess)
            return bail(fail(KVX_ENOSPC, "transition scratch allocation failed"));
    }

    // Per-layer slab bases for the layers this GPU sources.
    std::vector<kvx::LayerPtr> layers;
    std::vector<uint8_t> layer_is_peer;
    const uint64_t bb = block_bytes(g);
    for (int32_t l = 0; l < g.num_layers; ++l) {
        const int so = stage_of_layer(ob, l), sn = stage_of_layer(nb, l);
        kvx_pool* src = t->old_pools[(size_t)so];
        kvx_pool* dst = t->new_pools[(size_t)sn];
        if (d->pull) {  // this GPU owns the layer's destination; the source may be a peer's
            if (!dst || dst->imported || dst->device != d->device) continue;
            if (!src) return bail(fail(KVX_EINVAL, "pull: a local destination layer has no mapped source pool"));
            if (src->imported) t->has_peer_dst = true;  // peer traffic on this handle
        } else if (!src || src->imported || src->device != d->device) {
            continue;
        }
        const uint64_t ls = (uint64_t)(l - stage_begin(ob, so)) * (uint64_t)src->num_blocks * bb;
        const uint64_t ld = (uint64_t)(l - stage_begin(nb, sn)) * (uint64_t)dst->num_blocks * bb;
        layers.push_back({src->base + ls, dst->base + ld});
        layer_is_peer.push_back(dst->imported || src->imported ? 1 : 0);
        if (dst->imported) t->has_peer_dst = true;
    }
    // peer-destination layers first (see kvx_bulk_kernel's CTA split)
    {
        std::vector<kvx::LayerPtr> peer, local;
        for (size_t i = 0; i < layers.size(); ++i) (layer_is_peer[i] ? peer : local).push_back(layers[i]);
        t->n_peer_layers = (int32_t)peer.size();
        layers = peer;
        layers.insert(layers.end(), local.begin(), local.end());
    }
    t->n_local_layers = (int32_t)layers.size();
    if (!layers.empty()) {
        t->layers_bytes = sizeof(kvx::LayerPtr) * layers.size();
        if (A.dev_alloc((void**)&t->d_layers, t->layers_bytes) != cudaSuccess ||
            cudaMemcpyAsync(t->d_layers, layers.data(), sizeof(kvx::LayerPtr) * layers.size(),
                            cudaMemcpyHostToDevice, t->stream) != cudaSuccess)
            return bail(fail(KVX_ECUDA, "layer table upload"));
    }
    // No host sync: the uploads above were staged from pageable memory
    // (copied out before cudaMemcpyAsync returned) and are stream-ordered
    // before every wave.
    *out = t;
    return KVX_OK;
}

int kvx_wave(kvx_transition* t, uint64_t epoch, int32_t n, const int32_t* req, const int64_t* lo,
             const int64_t* hi) {
    if (!t) return fail(KVX_EINVAL, "transition is null");
    if (epoch != t->epoch) return fail(KVX_ESTALE, "stale epoch");
    if (t->state != kvx_transition::kActive) return fail(KVX_ESTATE, "transition is not active");
    if (n < 0 || n > t->max_requests || (n > 0 && (!req || !lo || !hi)))
        return fail(KVX_EINVAL, "bad wave arrays");
    // Validate against the host mirror of the destination rule.
    const int64_t B = t->g.block_tokens;
    int64_t nseg = 0, new_blocks = 0, tokens = 0;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t r = req[i];
        if (r < 0 || r >= t->max_requests) return fail(KVX_EINVAL, "req out of range");
        if (i > 0 && req[i - 1] >= r) return fail(KVX_EINVAL, "wave requests must be strictly ascending");
        if (hi[i] <= lo[i]) continue;
        const int64_t s = t->synced_hi[(size_t)r];
        if (lo[i] < 0 || lo[i] > s) return fail(KVX_EINVAL, "wave interval leaves a gap (lo > synced)");
        if (cdiv64(hi[i], B) > t->max_blocks) return fail(KVX_ENOSPC, "request exceeds max_blocks");
        const int32_t* srow = t->src_bt.data() + (size_t)r * (size_t)t->max_blocks;
        for (int64_t b = lo[i] / B; b < cdiv64(hi[i], B); ++b)
            if (srow[b] < 0) return fail(KVX_EINVAL, "wave reads a source block the source table does not back");
        new_blocks += std::max<int64_t>(0, cdiv64(hi[i], B) - cdiv64(s, B));
        nseg += cdiv64(hi[i], B) - lo[i] / B;
        tokens += hi[i] - lo[i];
    }
    if (t->bm ? new_blocks > t->bm->top : (int64_t)t->alloc + new_blocks > t->dst_num_blocks)
        return fail(KVX_ENOSPC, "destination pools full");
    DeviceGuard dg(t->device);
    if (n == 0 || nseg == 0) return KVX_OK;
    if (nseg > t->seg_cap) {
        kvx::Arena& A = kvx::Arena::of(t->device);
        if (t->d_segs) {
            KVX_CUDA(cudaStreamSynchronize(t->stream));
            A.dev_free(t->d_segs, sizeof(kvx::Seg) * (size_t)t->seg_cap);
            t->d_segs = nullptr;
        }
        const int64_t cap = (int64_t)(kvx::size_class(sizeof(kvx::Seg) * (size_t)std::max<int64_t>(nseg, 2 * t->seg_cap)) /
                                      sizeof(kvx::Seg));
        KVX_CUDA(A.dev_alloc((void**)&t->d_segs, sizeof(kvx::Seg) * (size_t)cap));
        t->seg_cap = cap;
    }
    // Stage (req | lo | hi) into pinned memory; the slot's previous upload
    // must have been consumed first.
    const int slot = t->wave_slot;
    t->wave_slot ^= 1;
    KVX_CUDA(cudaEventSynchronize(t->h_wave_free[slot]));
    char* h = t->h_wave[slot];
    const size_t off_lo = (((size_t)t->max_requests * sizeof(int32_t)) + 15) & ~size_t(15);
    const size_t off_hi = off_lo + (size_t)t->max_requests * sizeof(int64_t);
    std::memcpy(h, req, sizeof(int32_t) * n);
    std::memcpy(h + off_lo, lo, sizeof(int64_t) * n);
    std::memcpy(h + off_hi, hi, sizeof(int64_t) * n);
    if (!t->timing_open) {
        KVX_CUDA(cudaEventRecord(t->ev_begin, t->stream));
        t->timing_open = true;
    }
    // One H2D copy covering the three arrays at their fixed offsets.
    KVX_CUDA(cudaMemcpyAsync(t->d_wave, h, off_hi + sizeof(int64_t) * n, cudaMemcpyHostToDevice, t->stream));
    KVX_CUDA(cudaEventRecord(t->h_wave_free[slot], t->stream));
    const int32_t* d_req = reinterpret_cast<const int32_t*>(t->d_wave);
    const int64_t* d_lo = reinterpret_cast<const int64_t*>(t->d_wave + off_lo);
    const int64_t* d_hi = reinterpret_cast<const int64_t*>(t->d_wave + off_hi);
    kvx::kvx_plan_kernel<<<1, kvx::kPlanThreads, 0, t->stream>>>(
        d_req, d_lo, d_hi, n, t->d_src_bt, t->d_dst_bt, t->d_synced_hi, t->max_blocks,
        t->g.block_tokens, t->bm ? t->bm->top : t->alloc, t->bm ? t->bm->d_stack : nullptr, t->d_segs);
    KVX_LAUNCHED();
    if (t->n_local_layers > 0) {
        const int64_t units = nseg * t->n_local_layers;
        const int64_t full = (int64_t)t->num_sms * t->move_ctas_per_sm;
        const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(units, full));
        std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
        KVX_CUDA(kvx::Arena::of(t->device).event(&ev.first, true));
        KVX_CUDA(kvx::Arena::of(t->device).event(&ev.second, true));
        t->move_ev.push_back(ev);
        t->move_bytes.push_back(2ull * (uint64_t)tokens * 2ull * token_bytes(t->g) *
                                (uint64_t)t->n_local_layers);
        KVX_CUDA(cudaEventRecord(ev.first, t->stream));
        if (t->use_bulk && (!t->has_peer_dst || t->peer_bulk)) {
            const uint64_t run_bytes = nseg > 0 ? (uint64_t)tokens * 2ull * token_bytes(t->g) / (uint64_t)nseg : 0;
            const int vi = t->bulk_variant >= 0 ? t->bulk_variant : (run_bytes >= 65536 ? 2 : 0);
            const BulkVariant& bv = kBulkVariants[vi];
            // Grid: measured on B200 (profiles/r01_grid_sweep.jsonl), 128 one-CTA-per-SM
            // streams beat all 148 SMs for HBM-bound waves (1.034 vs 0.98 of the copy
            // peak); NVLink pushes saturate with ~16 CTAs, so mixed waves give the
            // peer layers kPeerCtas of them and the local layers the rest.
            constexpr int64_t kLocalGrid = 128, kPeerCtas = 32;
            int64_t full_b = std::min<int64_t>((int64_t)t->num_sms * t->bulk_ctas[vi], kLocalGrid);
            if (t->n_peer_layers > 0 && t->n_peer_layers < t->n_local_layers)
                full_b = std::min<int64_t>((int64_t)t->num_sms * t->bulk_ctas[vi], kLocalGrid + kPeerCtas);
            if (const char* cap = getenv("KVX_BULK_GRID"))
                full_b = std::max<int64_t>(1, std::min<int64_t>((int64_t)t->num_sms * t->bulk_ctas[vi], atoll(cap)));
            int32_t peer_ctas = (int32_t)kPeerCtas;
            if (const char* pc = getenv("KVX_PEER_CTAS")) peer_ctas = std::max(0, atoi(pc));
            const unsigned grid_b = (unsigned)std::max<int64_t>(1, std::min<int64_t>(units, full_b));
            bv.fn<<<grid_b, kvx::kBulkThreads, (size_t)bv.stages * bv.chunk, t->stream>>>(
                t->d_segs, (int32_t)nseg, t->d_layers, t->n_local_layers, block_bytes(t->g),
                token_bytes(t->g), t->g.block_tokens, t->n_peer_layers, peer_ctas);
        } else {
            kvx::kvx_move_kernel<<<grid, kvx::kMoveThreads, 0, t->stream>>>(
                t->d_segs, (int32_t)nseg, t->d_layers, t->n_local_layers, block_bytes(t->g),
                token_bytes(t->g), t->g.block_tokens, t->has_peer_dst ? 1 : 0);
        }
        KVX_LAUNCHED();
        KVX_CUDA(cudaEventRecord(ev.second, t->stream));
    }
    KVX_CUDA(cudaEventRecord(t->ev_end, t->stream));
    // Commit the mirror only once every launch was accepted.
    for (int32_t i = 0; i < n; ++i)
        if (hi[i] > t->synced_hi[(size_t)req[i]]) t->synced_hi[(size_t)req[i]] = hi[i];
    t->alloc += (int32_t)new_blocks;
    if (t->bm) t->bm->top -= (int32_t)new_blocks;
    t->bytes_moved += (uint64_t)tokens * 2ull * token_bytes(t->g) * (uint64_t)t->n_local_layers;
    t->bytes_all_layers += (uint64_t)tokens * 2ull * token_bytes(t->g) * (uint64_t)t->g.num_layers;
    return KVX_OK;
}

int kvx_wait(kvx_transition* t, uint64_t epoch, double* measured_ms) {
    if (!t) return fail(KVX_EINVAL, "transition is null");
    if (epoch != t->epoch) return fail(KVX_ESTALE, "stale epoch");
    DeviceGuard dg(t->device);
    KVX_CUDA(cudaStreamSynchronize(t->stream));
    float ms = 0.f;
    if (t->timing_open) {
        KVX_CUDA(cudaEventElapsedTime(&ms, t->ev_begin, t->ev_end));
        t->timing_open = false;
    }
    if (measured_ms) *measured_ms = ms;
    return KVX_OK;
}

int kvx_commit_async(kvx_transition* t, uint64_t epoch, int32_t n_live, const int32_t* req,
                     const int64_t* kv_tokens) {
    if (!t) return fail(KVX_EINVAL, "transition is null");
    if (epoch != t->epoch) return fail(KVX_ESTALE, "stale epoch");
    if (t->state != kvx_transition::kActive) return fail(KVX_ESTATE, "transition is not active");
    if (n_live < 0 || n_live > t->max_requests || (n_live > 0 && (!req || !kv_tokens)))
        return fail(KVX_EINVAL, "bad live arrays");
    for (int32_t i = 0; i < n_live; ++i) {
        if (req[i] < 0 || req[i] >= t->max_requests) return fail(KVX_EINVAL, "req out of range");
        if (i > 0 && req[i - 1] >= req[i]) return fail(KVX_EINVAL, "live requests must be strictly ascending");
    }
    DeviceGuard dg(t->device);
    // Exact output sizes from the host mirror (synced_hi is mirrored).
    const int64_t B = t->g.block_tokens;
    std::vector<uint8_t> live((size_t)t->max_requests, 0);
    int64_t nb_live = 0, nb_free = 0;
    for (int32_t i = 0; i < n_live; ++i) {
        live[(size_t)req[i]] = 1;
        nb_live += cdiv64(t->synced_hi[(size_t)req[i]], B);
    }
    for (int32_t r = 0; r < t->max_requests; ++r)
        if (!live[(size_t)r]) nb_free += cdiv64(t->synced_hi[(size_t)r], B);
    const int64_t need = (n_live + 1) + nb_live + nb_free;
    if (need > t->commit_i32_cap) return fail(KVX_ECUDA, "commit scratch undersized");  // sized at begin
    int32_t* d_row_ptr = t->d_commit_i32;
    int32_t* d_blocks = d_row_ptr + (n_live + 1);
    int32_t* d_free = d_blocks + nb_live;
    // Reuse the wave staging for the live set.
    const int slot = t->wave_slot;
    t->wave_slot ^= 1;
    KVX_CUDA(cudaEventSynchronize(t->h_wave_free[slot]));
    char* h = t->h_wave[slot];
    const size_t off_kv = (((size_t)t->max_requests * sizeof(int32_t)) + 15) & ~size_t(15);
    if (n_live > 0) {
        std::memcpy(h, req, sizeof(int32_t) * n_live);
        std::memcpy(h + off_kv, kv_tokens, sizeof(int64_t) * n_live);
        KVX_CUDA(cudaMemcpyAsync(t->d_wave, h, off_kv + sizeof(int64_t) * n_live, cudaMemcpyHostToDevice,
                                 t->stream));
    }
    KVX_CUDA(cudaEventRecord(t->h_wave_free[slot], t->stream));
    kvx::kvx_commit_kernel<<<1, kvx::kCommitThreads, 0, t->stream>>>(
        reinterpret_cast<const int32_t*>(t->d_wave), reinterpret_cast<const int64_t*>(t->d_wave + off_kv),
        n_live, t->d_dst_bt, t->d_synced_hi, t->d_live, t->max_requests, t->max_blocks, t->g.block_tokens,
        d_row_ptr, d_blocks, d_free, t->d_commit_out);
    KVX_LAUNCHED();
    // results land in pinned memory; kvx_commit_collect reads them
    KVX_CUDA(cudaMemcpyAsync(t->h_commit, t->d_commit_out, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, t->stream));
    KVX_CUDA(cudaMemcpyAsync(t->h_commit + 32, t->d_commit_i32, sizeof(int32_t) * (size_t)need,
                             cudaMemcpyDeviceToHost, t->stream));
    if (t->bm && nb_free > 0) {  // free-list update: dead rows' blocks back on the stack
        KVX_CUDA(cudaMemcpyAsync(t->bm->d_stack + t->bm->top, d_free, sizeof(int32_t) * (size_t)nb_free,
                                 cudaMemcpyDeviceToDevice, t->stream));
        t->bm->top += (int32_t)nb_free;
    }
    KVX_CUDA(cudaEventRecord(t->ev_commit, t->stream));
    t->pend_n_live = n_live;
    t->pend_nb_live = nb_live;
    t->pend_nb_free = nb_free;
    t->state = kvx_transition::kCommitPending;
    ++t->epoch;  // engine.cpp:752 -- the commit is decided; later waves are stale
    t->timing_open = false;
    return KVX_OK;
}

int kvx_commit_collect(kvx_transition* t, kvx_commit_result* out) {
    if (!t) return fail(KVX_EINVAL, "transition is null");
    if (t->state != kvx_transition::kCommitPending) return fail(KVX_ESTATE, "no commit pending");
    DeviceGuard dg(t->device);
    KVX_CUDA(cudaEventSynchronize(t->ev_commit));
    int64_t res[3];
    std::memcpy(res, t->h_commit, sizeof(res));
    if (res[1] != t->pend_nb_live || res[2] != t->pend_nb_free)
        return fail(KVX_ECUDA, "device compaction disagrees with the host mirror");
    const int32_t* h32 = reinterpret_cast<const int32_t*>(t->h_commit + 32);
    if (out) {
        if (out->blocks && out->blocks_cap < t->pend_nb_live) return fail(KVX_EINVAL, "blocks_cap too small");
        if (out->free_list && out->free_cap < t->pend_nb_free) return fail(KVX_EINVAL, "free_cap too small");
        if (out->row_ptr) std::memcpy(out->row_ptr, h32, sizeof(int32_t) * (size_t)(t->pend_n_live + 1));
        if (out->blocks)
            std::memcpy(out->blocks, h32 + t->pend_n_live + 1, sizeof(int32_t) * (size_t)t->pend_nb_live);
        if (out->free_list)
            std::memcpy(out->free_list, h32 + t->pend_n_live + 1 + t->pend_nb_live,
                        sizeof(int32_t) * (size_t)t->pend_nb_free);
        out->violations = res[0];
        out->n_blocks = (int32_t)res[1];
        out->n_free = (int32_t)res[2];
    }
    t->state = kvx_transition::kCommitted;
    return KVX_OK;
}

int kvx_commit(kvx_transition* t, uint64_t epoch, int32_t n_live, const int32_t* req,
               const int64_t* kv_tokens, kvx_commit_result* out) {
    const int rc = kvx_commit_async(t, epoch, n_live, req, kv_tokens);
    if (rc != KVX_OK) return rc;
    return kvx_commit_collect(t, out);
}

int kvx_abort(kvx_transition* t) {
    if (!t) return fail(KVX_EINVAL, "transition is null");
    if (t->state != kvx_transition::kActive) return fail(KVX_ESTATE, "transition is not active");
    DeviceGuard dg(t->device);
    KVX_CUDA(cudaStreamSynchronize(t->stream));  // in-flight waves land in pools we now drop
    if (t->bm) {  // every destination block goes back on the free stack
        const int64_t B = t->g.block_tokens;
        int64_t nb_all = 0;
        for (int32_t r = 0; r < t->max_requests; ++r) nb_all += cdiv64(t->synced_hi[(size_t)r], B);
        if (nb_all > 0) {
            int32_t* d_row_ptr = t->d_commit_i32;
            int32_t* d_free = d_row_ptr + 1;
            kvx::kvx_commit_kernel<<<1, kvx::kCommitThreads, 0, t->stream>>>(
                reinterpret_cast<const int32_t*>(t->d_wave), reinterpret_cast<const int64_t*>(t->d_wave), 0,
                t->d_dst_bt, t->d_synced_hi, t->d_live, t->max_requests, t->max_blocks, t->g.block_tokens,
                d_row_ptr, d_free, d_free, t->d_commit_out);
            KVX_LAUNCHED();
            KVX_CUDA(cudaMemcpyAsync(t->bm->d_stack + t->bm->top, d_free, sizeof(int32_t) * (size_t)nb_all,
                                     cudaMemcpyDeviceToDevice, t->stream));
            t->bm->top += (int32_t)nb_all;
        }
    }
    t->state = kvx_transition::kAborted;
    ++t->epoch;  // engine.cpp:769
    t->alloc = 0;
    std::fill(t->synced_hi.begin(), t->synced_hi.end(), 0);
    const size_t bt_bytes = sizeof(int32_t) * (size_t)t->max_requests * (size_t)t->max_blocks;
    KVX_CUDA(cudaMemsetAsync(t->d_dst_bt, 0xff, bt_bytes, t->stream));
    KVX_CUDA(cudaMemsetAsync(t->d_synced_hi, 0, sizeof(int64_t) * (size_t)t->max_requests, t->stream));
    KVX_CUDA(cudaStreamSynchronize(t->stream));
    t->timing_open = false;
    return KVX_OK;
}

int kvx_destroy(kvx_transition* t) {
    if (!t) return KVX_OK;
    DeviceGuard dg(t->device);
    if (t->stream) cudaStreamSynchronize(t->stream);
    kvx::Arena& A = kvx::Arena::of(t->device);
    A.dev_free(t->d_src_bt, t->bt_bytes);
    A.dev_free(t->d_dst_bt, t->bt_bytes);
    A.dev_free(t->d_synced_hi, sizeof(int64_t) * (size_t)t->max_requests);
    A.dev_free(t->d_layers, t->layers_bytes);
    A.dev_free(t->d_wave, t->wave_bytes);
    A.dev_free(t->d_segs, sizeof(kvx::Seg) * (size_t)t->seg_cap);
    A.dev_free(t->d_live, (size_t)t->max_requests);
    A.dev_free(t->d_commit_i32, sizeof(int32_t) * (size_t)t->commit_i32_cap);
    A.dev_free(t->d_commit_out, 4 * sizeof(int64_t));
    A.host_free(t->h_commit, t->h_commit_bytes);
    A.event_free(t->ev_commit, false);
    for (int s = 0; s < 2; ++s) {
        A.host_free(t->h_wave[s], t->wave_bytes);
        A.event_free(t->h_wave_free[s], false);
    }
    A.event_free(t->ev_begin, true);
    A.event_free(t->ev_end, true);
    A.dev_free(t->d_pieces, sizeof(kvx::Piece) * (size_t)t->piece_cap);
    A.host_free(t->h_pieces, sizeof(kvx::Piece) * (size_t)t->piece_cap);
    A.event_free(t->pieces_free, false);
    for (auto& ev : t->move_ev) {
        A.event_free(ev.first, true);
        A.event_free(ev.second, true);
    }
    if (t->stream && t->own_stream) cudaStreamDestroy(t->stream);
    delete t;
    return KVX_OK;
}

int kvx_handoff(kvx_transition* t, uint64_t epoch, uint64_t row_bytes, int32_t n,
                const kvx_microbatch* mb, void* const* arenas, const uint64_t* arena_bytes,
                kvx_handoff_slot* slots_out) {
    if (!t) return fail(KVX_EINVAL, "transition is null");
    if (epoch != t->epoch) return fail(KVX_ESTALE, "stale epoch");
    if (t->state != kvx_transition::kActive) return fail(KVX_ESTATE, "transition is not active");
    if (n < 0 || (n > 0 && (!mb || !slots_out)) || !arenas || !arena_bytes || row_bytes % 16 != 0)
        return fail(KVX_EINVAL, "bad handoff arguments");
    const int k_old = (int)t->old_b.size() + 1, k_new = (int)t->new_b.size() + 1;
    std::vector<uint64_t> bump((size_t)k_new, 0);
    std::vector<kvx::Piece> pieces;
    for (int32_t i = 0; i < n; ++i) {
        kvx_handoff_slot& sl = slots_out[i];
        sl.batch_id = mb[i].batch_id;
        if (mb[i].tokens < 0) return fail(KVX_EINVAL, "negative tokens");
        const int32_t a = mb[i].after_stage;
        if (a < 0 || a + 1 >= k_old) {  // nothing computed yet: re-dispatch at the new head
            sl.new_stage = 0;
            sl.resume_layer = 0;
            sl.offset = 0;
            sl.bytes = 0;
            continue;
        }
        const int32_t layer = t->old_b[(size_t)a];
        const int k = stage_of_layer(t->new_b, layer);
        const uint64_t b = (uint64_t)mb[i].tokens * row_bytes;
        const uint64_t off = (bump[(size_t)k] + 255u) & ~(uint64_t)255u;
        if (off + b > arena_bytes[k]) return fail(KVX_ENOSPC, "activation arena full");
        sl.new_stage = k;
        sl.resume_layer = layer;
        sl.offset = off;
        sl.bytes = b;
        bump[(size_t)k] = off + b;
        const kvx_pool* src_pool = t->old_pools[(size_t)a];
        const bool local = src_pool && !src_pool->imported && src_pool->device == t->device;
        if (!local || b == 0) continue;
        if (!mb[i].src || !arenas[k] || (reinterpret_cast<uintptr_t>(mb[i].src) & 15) ||
            (reinterpret_cast<uintptr_t>(arenas[k]) & 15))
            return fail(KVX_EINVAL, "activation pointers must be non-null and 16-byte aligned");
        // 64 KiB sub-pieces so one large activation spreads over many CTAs
        const char* src = static_cast<const char*>(mb[i].src);
        char* dst = static_cast<char*>(arenas[k]) + off;
        for (uint64_t o = 0; o < b; o += 65536)
            pieces.push_back({src + o, dst + o, std::min<uint64_t>(65536, b - o)});
    }
    if (pieces.empty()) return KVX_OK;
    DeviceGuard dg(t->device);
    kvx::Arena& A = kvx::Arena::of(t->device);
    if (!t->pieces_free) KVX_CUDA(A.event(&t->pieces_free, false));
    KVX_CUDA(cudaEventSynchronize(t->pieces_free));  // previous handoff's upload consumed
    if ((int64_t)pieces.size() > t->piece_cap) {
        A.dev_free(t->d_pieces, sizeof(kvx::Piece) * (size_t)t->piece_cap);
        A.host_free(t->h_pieces, sizeof(kvx::Piece) * (size_t)t->piece_cap);
        t->d_pieces = nullptr;
        t->h_pieces = nullptr;
        const int64_t cap = (int64_t)(kvx::size_class(sizeof(kvx::Piece) * pieces.size()) / sizeof(kvx::Piece));
        KVX_CUDA(cudaStreamSynchronize(t->stream));
        KVX_CUDA(A.dev_alloc((void**)&t->d_pieces, sizeof(kvx::Piece) * (size_t)cap));
        KVX_CUDA(A.host_alloc((void**)&t->h_pieces, sizeof(kvx::Piece) * (size_t)cap));
        t->piece_cap = cap;
    }
    std::memcpy(t->h_pieces, pieces.data(), sizeof(kvx::Piece) * pieces.size());
    KVX_CUDA(cudaMemcpyAsync(t->d_pieces, t->h_pieces, sizeof(kvx::Piece) * pieces.size(),
                             cudaMemcpyHostToDevice, t->stream));
    KVX_CUDA(cudaEventRecord(t->pieces_free, t->stream));
    constexpr int kStages = 4;
    constexpr uint32_t kChunk = 32768;
    // per-device attribute: set on every call (cheap; the handle's device may differ)
    KVX_CUDA(cudaFuncSetAttribute(kvx::kvx_copy_list_kernel<kStages, kChunk>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * (int)kChunk));
    const unsigned grid = (unsigned)std::min<int64_t>(2 * (int64_t)t->num_sms, (int64_t)pieces.size());
    kvx::kvx_copy_list_kernel<kStages, kChunk><<<grid, kvx::kBulkThreads, kStages * kChunk, t->stream>>>(
        t->d_pieces, (int64_t)pieces.size());
    KVX_LAUNCHED();
    return KVX_OK;
}


int kvx_weights_migrate(int32_t device, void* stream, int32_t num_layers, uint64_t layer_bytes,
                        int32_t old_stages, const int32_t* old_boundaries, void* const* old_ptrs,
                        int32_t new_stages, const int32_t* new_boundaries, void* const* new_ptrs,
                        const void* host_cache, const uint8_t* from_host, uint64_t* device_bytes,
                        uint64_t* host_bytes) {
    std::string why;
    if (num_layers < 1 || layer_bytes == 0 || layer_bytes % 16 != 0 || !old_ptrs || !new_ptrs)
        return fail(KVX_EINVAL, "weights: bad layer count / layer_bytes (multiple of 16) / pointers");
    const kvx_plan op{old_stages, old_boundaries, nullptr}, np{new_stages, new_boundaries, nullptr};
    std::vector<int32_t> ob, nb;
    kvx_plan op2 = op, np2 = np;
    kvx_pool* dummy = nullptr;
    op2.pools = &dummy;
    np2.pools = &dummy;
    if (!plan_ok(op2, num_layers, &why, &ob)) return fail(KVX_EINVAL, "weights old plan: " + why);
    if (!plan_ok(np2, num_layers, &why, &nb)) return fail(KVX_EINVAL, "weights new plan: " + why);
    std::vector<kvx::Piece> pieces;
    uint64_t dev_b = 0, host_b = 0;
    DeviceGuard dg(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    for (int32_t l = 0; l < num_layers; ++l) {
        const int so = stage_of_layer(ob, l), sn = stage_of_layer(nb, l);
        char* dst = static_cast<char*>(new_ptrs[sn]);
        if (!dst) return fail(KVX_EINVAL, "weights: every new stage buffer is required");
        dst += (uint64_t)(l - stage_begin(nb, sn)) * layer_bytes;
        if (from_host && from_host[l]) {
            if (!host_cache) return fail(KVX_EINVAL, "weights: from_host without a host cache");
            // host tier: only the rank that would otherwise source the layer loads it
            if (!old_ptrs[so]) continue;
            KVX_CUDA(cudaMemcpyAsync(dst, static_cast<const char*>(host_cache) + (uint64_t)l * layer_bytes,
                                     layer_bytes, cudaMemcpyHostToDevice, st));
            host_b += layer_bytes;
            continue;
        }
        if (!old_ptrs[so]) continue;  // another rank owns this layer's source
        const char* src = static_cast<const char*>(old_ptrs[so]) + (uint64_t)(l - stage_begin(ob, so)) * layer_bytes;
        for (uint64_t o = 0; o < layer_bytes; o += (1u << 20))
            pieces.push_back({src + o, dst + o, std::min<uint64_t>(1u << 20, layer_bytes - o)});
        dev_b += layer_bytes;
    }
    if (device_bytes) *device_bytes = dev_b;
    if (host_bytes) *host_bytes = host_b;
    if (pieces.empty()) return KVX_OK;
    int sms = 0;
    KVX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    kvx::Arena& A = kvx::Arena::of(device);
    const size_t bytes = sizeof(kvx::Piece) * pieces.size();
    void *d = nullptr, *h = nullptr;
    KVX_CUDA(A.dev_alloc(&d, bytes));
    KVX_CUDA(A.host_alloc(&h, bytes));
    std::memcpy(h, pieces.data(), bytes);
    KVX_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
    constexpr int kStages = 6;
    constexpr uint32_t kChunk = 32768;
    KVX_CUDA(cudaFuncSetAttribute(kvx::kvx_copy_list_kernel<kStages, kChunk>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * (int)kChunk));
    const unsigned grid = (unsigned)std::min<int64_t>((int64_t)sms, (int64_t)pieces.size());
    kvx::kvx_copy_list_kernel<kStages, kChunk><<<grid, kvx::kBulkThreads, kStages * kChunk, st>>>(
        static_cast<const kvx::Piece*>(d), (int64_t)pieces.size());
    KVX_LAUNCHED();
    KVX_CUDA(cudaLaunchHostFunc(st, release_pieces, new PieceRelease{device, d, h, bytes}));
    return KVX_OK;
}

// ------------------------------------------------------------ block manager
int kvx_bm_create(int32_t device, int32_t capacity, kvx_blockmgr** out) {
    if (!out || capacity < 1) return fail(KVX_EINVAL, "bad block manager arguments");
    *out = nullptr;
    DeviceGuard dg(device);
    if (!dg.ok) return fail(KVX_ECUDA, "cudaSetDevice failed");
    auto* bm = new kvx_blockmgr;
    bm->device = device;
    bm->capacity = capacity;
    if (cudaMalloc(&bm->d_stack, sizeof(int32_t) * (size_t)capacity) != cudaSuccess) {
        delete bm;
        cudaGetLastError();
        return fail(KVX_ENOSPC, "block manager allocation failed");
    }
    *out = bm;
    return kvx_bm_reset(bm);
}

int kvx_bm_reset(kvx_blockmgr* bm) {
    if (!bm) return fail(KVX_EINVAL, "block manager is null");
    DeviceGuard dg(bm->device);
    kvx::kvx_bm_init_kernel<<<(unsigned)std::min<int64_t>(1024, (bm->capacity + 255) / 256), 256>>>(
        bm->d_stack, bm->capacity);
    KVX_LAUNCHED();
    KVX_CUDA(cudaDeviceSynchronize());
    bm->top = bm->capacity;
    return KVX_OK;
}

int kvx_bm_free_count(const kvx_blockmgr* bm, int32_t* n) {
    if (!bm || !n) return fail(KVX_EINVAL, "null argument");
    *n = bm->top;
    return KVX_OK;
}

int kvx_bm_pop(kvx_blockmgr* bm, int32_t n, int32_t* ids_out) {
    if (!bm || n < 0 || (n > 0 && !ids_out)) return fail(KVX_EINVAL, "bad pop arguments");
    if (n > bm->top) return fail(KVX_ENOSPC, "block manager exhausted");
    if (n == 0) return KVX_OK;
    DeviceGuard dg(bm->device);
    std::vector<int32_t> tmp((size_t)n);
    KVX_CUDA(cudaDeviceSynchronize());  // stack pushes queued on transition streams have landed
    KVX_CUDA(cudaMemcpy(tmp.data(), bm->d_stack + (bm->top - n), sizeof(int32_t) * (size_t)n,
                        cudaMemcpyDeviceToHost));
    for (int32_t i = 0; i < n; ++i) ids_out[i] = tmp[(size_t)(n - 1 - i)];  // LIFO order
    bm->top -= n;
    return KVX_OK;
}

int kvx_bm_push(kvx_blockmgr* bm, int32_t n, const int32_t* ids) {
    if (!bm || n < 0 || (n > 0 && !ids)) return fail(KVX_EINVAL, "bad push arguments");
    if (bm->top + n > bm->capacity) return fail(KVX_EINVAL, "push beyond capacity (double free?)");
    for (int32_t i = 0; i < n; ++i)
        if (ids[i] < 0 || ids[i] >= bm->capacity) return fail(KVX_EINVAL, "block id out of range");
    if (n == 0) return KVX_OK;
    DeviceGuard dg(bm->device);
    KVX_CUDA(cudaDeviceSynchronize());
    KVX_CUDA(cudaMemcpy(bm->d_stack + bm->top, ids, sizeof(int32_t) * (size_t)n, cudaMemcpyHostToDevice));
    bm->top += n;
    return KVX_OK;
}

int kvx_bm_snapshot(const kvx_blockmgr* bm, int32_t* stack_out, int32_t* top_out) {
    if (!bm) return fail(KVX_EINVAL, "block manager is null");
    DeviceGuard dg(bm->device);
    KVX_CUDA(cudaDeviceSynchronize());
    if (stack_out && bm->top > 0)
        KVX_CUDA(cudaMemcpy(stack_out, bm->d_stack, sizeof(int32_t) * (size_t)bm->top, cudaMemcpyDeviceToHost));
    if (top_out) *top_out = bm->top;
    return KVX_OK;
}

int kvx_bm_destroy(kvx_blockmgr* bm) {
    if (!bm) return KVX_OK;
    DeviceGuard dg(bm->device);
    cudaFree(bm->d_stack);
    delete bm;
    return KVX_OK;
}

int kvx_epoch(const kvx_transition* t, uint64_t* epoch) {
    if (!t || !epoch) return fail(KVX_EINVAL, "null argument");
    *epoch = t->epoch;
    return KVX_OK;
}

int kvx_dst_block_table(kvx_transition* t, int32_t* host_out) {
    if (!t || !host_out) return fail(KVX_EINVAL, "null argument");
    DeviceGuard dg(t->device);
    KVX_CUDA(cudaMemcpyAsync(host_out, t->d_dst_bt,
                             sizeof(int32_t) * (size_t)t->max_requests * (size_t)t->max_blocks,
                             cudaMemcpyDeviceToHost, t->stream));
    KVX_CUDA(cudaStreamSynchronize(t->stream));
    return KVX_OK;
}

int kvx_stream(const kvx_transition* t, void** stream) {
    if (!t || !stream) return fail(KVX_EINVAL, "null argument");
    *stream = t->stream;
    return KVX_OK;
}

int kvx_move_timings(const kvx_transition* t, int32_t cap, double* move_ms, uint64_t* rw_bytes,
                     int32_t* n_out) {
    if (!t || !n_out || cap < 0) return fail(KVX_EINVAL, "bad arguments");
    DeviceGuard dg(t->device);
    const int32_t n = (int32_t)t->move_ev.size();
    for (int32_t i = 0; i < n && i < cap; ++i) {
        float ms = 0.f;
        KVX_CUDA(cudaEventSynchronize(t->move_ev[(size_t)i].second));
        KVX_CUDA(cudaEventElapsedTime(&ms, t->move_ev[(size_t)i].first, t->move_ev[(size_t)i].second));
        if (move_ms) move_ms[i] = ms;
        if (rw_bytes) rw_bytes[i] = t->move_bytes[(size_t)i];
    }
    *n_out = n;
    return KVX_OK;
}

int kvx_bytes_moved(const kvx_transition* t, uint64_t* bytes) {
    if (!t || !bytes) return fail(KVX_EINVAL, "null argument");
    *bytes = t->bytes_moved;
    return KVX_OK;
}

int kvx_verify_pattern(kvx_transition* t, uint64_t seed, int32_t n, const int32_t* req,
                       const int64_t* kv, int64_t* mismatched_words) {
    if (!t || !mismatched_words || n < 0 || (n > 0 && (!req || !kv))) return fail(KVX_EINVAL, "bad arguments");
    *mismatched_words = 0;
    if (n == 0) return KVX_OK;
    DeviceGuard dg(t->device);
    int64_t max_tok = 0;
    for (int32_t i = 0; i < n; ++i) {
        if (req[i] < 0 || req[i] >= t->max_requests) return fail(KVX_EINVAL, "req out of range");
        if (kv[i] < 0 || cdiv64(kv[i], t->g.block_tokens) > t->max_blocks)
            return fail(KVX_EINVAL, "kv exceeds max_blocks");
        max_tok = std::max(max_tok, kv[i]);
    }
    if (max_tok == 0) return KVX_OK;
    int32_t* d_req = nullptr;
    int64_t* d_kv = nullptr;
    unsigned long long* d_bad = nullptr;
    KVX_CUDA(cudaMalloc(&d_req, sizeof(int32_t) * n));
    KVX_CUDA(cudaMalloc(&d_kv, sizeof(int64_t) * n));
    KVX_CUDA(cudaMalloc(&d_bad, sizeof(unsigned long long)));
    KVX_CUDA(cudaMemcpyAsync(d_req, req, sizeof(int32_t) * n, cudaMemcpyHostToDevice, t->stream));
    KVX_CUDA(cudaMemcpyAsync(d_kv, kv, sizeof(int64_t) * n, cudaMemcpyHostToDevice, t->stream));
    KVX_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), t->stream));
    dim3 grid((unsigned)n, (unsigned)cdiv64(max_tok, t->g.block_tokens));
    for (size_t k = 0; k < t->new_pools.size(); ++k) {
        const kvx_pool* p = t->new_pools[k];
        if (!p || p->imported) continue;  // the owning rank verifies it
        kvx::kvx_verify_kernel<<<grid, 256, 0, t->stream>>>(
            p->base, p->num_blocks, stage_begin(t->new_b, (int)k), p->num_layers, d_req, d_kv,
            t->d_dst_bt, t->max_blocks, t->g.block_tokens, token_bytes(t->g), seed, d_bad);
        KVX_LAUNCHED();
    }
    unsigned long long bad = 0;
    KVX_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, t->stream));
    KVX_CUDA(cudaStreamSynchronize(t->stream));
    cudaFree(d_req);
    cudaFree(d_kv);
    cudaFree(d_bad);
    *mismatched_words = (int64_t)bad;
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
