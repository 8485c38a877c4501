// kvx_common.h -- internal to the kvx library: the opaque handle types of
// include/kvx.h, error/launch bookkeeping and the small host helpers shared by
// the translation units (kvx_pool.cu, kvx_transition.cu, kvx_extras.cu,
// kvx_common.cu).  Device code lives in kvx_kernels.cuh.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "kvx.h"
#include "kvx_arena.h"
#include "kvx_internal.h"
#include "kvx_kernels.cuh"

namespace kvx_host {

std::string& last_error();          // thread-local message (kvx_common.cu)
std::atomic<uint64_t>& launches();   // process-wide launch counter

inline int fail(int code, const std::string& msg) {
    last_error() = msg;
    return code;
}

#define KVX_CUDA(call)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return kvx_host::fail(KVX_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
    } while (0)

#define KVX_LAUNCHED()                                                                    \
    do {                                                                                  \
        kvx_host::launches().fetch_add(1, std::memory_order_relaxed);                               \
        cudaError_t e_ = cudaGetLastError();                                              \
        if (e_ != cudaSuccess)                                                            \
            return kvx_host::fail(KVX_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
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

// A pool of this process on another GPU is usable over NVLink when the two
// devices have peer access (enabled here; idempotent).  One process may drive
// several GPUs, one transition handle per device -- the single-process
// analogue of one rank per GPU.
inline bool peer_ok(int dev, int other) {
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, dev, other) != cudaSuccess || !can) {
        cudaGetLastError();
        return false;
    }
    DeviceGuard dg(dev);
    const cudaError_t e = cudaDeviceEnablePeerAccess(other, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return true;
    }
    return e == cudaSuccess;
}

inline bool geometry_ok(const kvx_geometry* g, std::string* why) {
    if (!g) return *why = "geometry is null", false;
    if (g->num_layers < 1 || g->num_kv_heads < 1 || g->head_dim < 1 || g->elem_bytes < 1 ||
        g->block_tokens < 1)
        return *why = "geometry fields must be positive", false;
    const uint64_t tb = (uint64_t)g->num_kv_heads * g->head_dim * g->elem_bytes;
    if (tb % 16 != 0) return *why = "token_bytes must be a multiple of 16", false;
    return true;
}

inline bool layout_ok(int32_t layout) {
    return layout == KVX_LAYOUT_BLOCKS || layout == KVX_LAYOUT_KV_PLANES || layout == KVX_LAYOUT_HEADS;
}
// head-major rows are head_dim * elem_bytes long: 16-byte vectors / bulk-copy alignment
inline bool layout_fits(int32_t layout, const kvx_geometry& g) {
    return layout != KVX_LAYOUT_HEADS || ((int64_t)g.head_dim * g.elem_bytes) % 16 == 0;
}

inline uint64_t token_bytes(const kvx_geometry& g) {
    return (uint64_t)g.num_kv_heads * (uint64_t)g.head_dim * (uint64_t)g.elem_bytes;
}
inline uint64_t block_bytes(const kvx_geometry& g) { return 2ull * (uint64_t)g.block_tokens * token_bytes(g); }

inline int64_t cdiv64(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int stage_of_layer(const std::vector<int32_t>& b, int32_t layer) {  // modelgraph.cpp:55-62
    int s = 0;
    for (int32_t cut : b) {
        if (layer < cut) break;
        ++s;
    }
    return s;
}
inline int stage_begin(const std::vector<int32_t>& b, int s) { return s == 0 ? 0 : b[(size_t)s - 1]; }

inline bool plan_ok(const kvx_plan& p, int32_t L, std::string* why, std::vector<int32_t>* out) {
    if (p.num_stages < 1 || p.num_stages > L) return *why = "num_stages out of range", false;
    if (p.num_stages > 1 && !p.boundaries) return *why = "boundaries is null", false;
    out->assign(p.boundaries, p.boundaries + (p.num_stages - 1));
    int32_t prev = 0;
    for (int32_t b : *out) {
        if (b <= prev || b >= L) return *why = "boundaries must be strictly increasing in (0, L)", false;
        prev = b;
    }
    if (!p.pools) return *why = "plan pools array is null", false;
    return true;
}


struct PieceRelease {  // returns a call's descriptor buffers to the arena once the stream passed them
    int device;
    void* d;
    void* h;
    size_t bytes;
};
inline void CUDART_CB release_pieces(void* arg) {
    auto* r = static_cast<PieceRelease*>(arg);
    kvx::Arena& A = kvx::Arena::of(r->device);
    A.dev_free(r->d, r->bytes);
    A.host_free(r->h, r->bytes);
    delete r;
}

// Eager kernel loading.  Under CUDA lazy loading (the default) a kernel's
// module is loaded at its first launch or attribute query, and the load waits
// for the work already running on the device: the first refactor of a
// serving process would stall behind the serving kernels.  ensure_loaded()
// loads every kvx kernel the first time a device is touched (pool, block
// manager or transition creation; kvx_preload), once per device.
cudaError_t preload_transition_kernels();
cudaError_t preload_pool_kernels();
cudaError_t preload_extras_kernels();
int ensure_loaded(int device);

// (ring depth, chunk bytes, store lag, pieces per slot) of the TMA bulk
// mover (kvx_kernels.cuh bulk_stream).  Slab-sized waves (mostly full
// blocks) use kSlabVariant, token-granular waves (delta / final: a token's K
// or V row per run) kTokVariant; KVX_BULK_CFG pins one variant for both,
// KVX_BULK_CFG_SLAB / KVX_BULK_CFG_TOK one kind.
using BulkFn = void (*)(const kvx::Seg*, int32_t, const kvx::LayerPtr*, int32_t, uint64_t, uint64_t, int32_t,
                        int32_t, int32_t, unsigned long long*, unsigned long long*);
struct BulkVariant {
    int stages;
    uint32_t chunk;
    int lag, pack;
    BulkFn fn;
};
#define KVX_BV(S, C, G, P) {S, C, G, P, kvx::kvx_bulk_kernel<S, C, G, P>}
inline const BulkVariant kBulkVariants[] = {
    KVX_BV(6, 32768, 2, 1),  KVX_BV(4, 49152, 2, 1),  KVX_BV(3, 65536, 2, 1),  KVX_BV(12, 16384, 2, 1),
    KVX_BV(3, 32768, 2, 1),  KVX_BV(8, 16384, 2, 1),  KVX_BV(2, 65536, 1, 1),  KVX_BV(4, 16384, 2, 1),
    // packed rings for token-granular waves
    KVX_BV(6, 32768, 3, 4),  KVX_BV(12, 16384, 6, 2), KVX_BV(8, 24576, 4, 3),  KVX_BV(6, 32768, 2, 4),
    KVX_BV(3, 32768, 1, 4),  KVX_BV(6, 16384, 3, 2),  KVX_BV(12, 16384, 4, 2), KVX_BV(4, 49152, 2, 4),
    // small rings: several CTAs per SM for token-granular waves (more issuing threads)
    KVX_BV(3, 16384, 2, 1),  KVX_BV(6, 12288, 3, 1),  KVX_BV(8, 12288, 4, 1),  KVX_BV(4, 12288, 2, 1),
    KVX_BV(4, 24576, 2, 2),  KVX_BV(2, 24576, 1, 2),
};
#undef KVX_BV
constexpr int kSlabVariant = 2;  // 3 x 64 KiB, one chunk per slot
// 4 x 16 KiB, two CTAs per SM on a 296-CTA grid: the C3 final wave in 73.7-77.8 us on
// four boxes, against 88-96 us for round 1's 6 x 32 KiB on 148 (profiles/r02*_wave_sweep_tok*)
constexpr int kTokVariant = 7;
constexpr int kNumBulkVariants = sizeof(kBulkVariants) / sizeof(kBulkVariants[0]);

// TMA transposer ring (kvx_tmap_kernel): slots of up to kTmapSlot bytes
constexpr int kTmapStages = 6, kTmapLag = 2;
constexpr uint32_t kTmapSlot = 32768;



}  // namespace kvx_host

// ------------------------------------------------- opaque handle types
struct kvx_pool {
    int32_t device = -1;
    bool imported = false;
    bool wrapped = false;  // caller-owned memory
    bool per_layer = false;  // kvx_pool_wrap_layers: one allocation per layer
    char* base = nullptr;    // single allocation (layer 0 of a per-layer pool)
    uint64_t bytes = 0;
    kvx_geometry g{};
    int32_t num_layers = 0;
    int32_t num_blocks = 0;
    int32_t layout = KVX_LAYOUT_BLOCKS;
    std::vector<char*> layer_base;  // per layer, in every pool

    uint64_t layer_bytes() const { return (uint64_t)num_blocks * 2ull * g.block_tokens * kvx_host::token_bytes(g); }
    // Address of (block b, K|V k, token t, head h) in a layer:
    //   base + b*blk_stride + k*kv_stride + t*tok_stride + h*head_stride
    uint64_t head_bytes() const { return (uint64_t)g.head_dim * (uint64_t)g.elem_bytes; }
    uint64_t blk_stride() const {
        const uint64_t plane = (uint64_t)g.block_tokens * kvx_host::token_bytes(g);
        return layout == KVX_LAYOUT_KV_PLANES ? plane : 2 * plane;
    }
    uint64_t kv_stride() const {
        const uint64_t plane = (uint64_t)g.block_tokens * kvx_host::token_bytes(g);
        return layout == KVX_LAYOUT_KV_PLANES ? (uint64_t)num_blocks * plane : plane;
    }
    uint64_t tok_stride() const { return layout == KVX_LAYOUT_HEADS ? head_bytes() : kvx_host::token_bytes(g); }
    uint64_t head_stride() const {
        return layout == KVX_LAYOUT_HEADS ? (uint64_t)g.block_tokens * head_bytes() : head_bytes();
    }
    bool head_major() const { return layout == KVX_LAYOUT_HEADS; }
    void set_contiguous_layers() {
        layer_base.resize((size_t)num_layers);
        for (int32_t l = 0; l < num_layers; ++l) layer_base[(size_t)l] = base + (uint64_t)l * layer_bytes();
    }
};

// A pool's addressing for the payload kernels; d_layers = its layer_base on the device.
inline kvx::PoolAddr pool_addr(const kvx_pool* p, char* const* d_layers) {
    return kvx::PoolAddr{d_layers, p->blk_stride(), p->kv_stride(), p->tok_stride(), p->head_stride(),
                         (uint32_t)p->head_bytes()};
}

// True when any layer span of `a` shares an address with one of `b`'s (both
// mapped in this process: local or imported).  Layer spans are
// [layer_base, layer_base + layer_bytes) in every layout.
inline bool pools_overlap(const kvx_pool* a, const kvx_pool* b) {
    if (!a || !b) return false;
    const uint64_t na = a->layer_bytes(), nb = b->layer_bytes();
    for (const char* x : a->layer_base)
        for (const char* y : b->layer_base)
            if (x < y + nb && y < x + na) return true;
    return false;
}

// Device-resident block manager: a free-id stack on the GPU, its top mirrored
// on the host so every capacity decision is synchronous and deterministic.
struct kvx_blockmgr {
    int32_t device = -1;
    int32_t capacity = 0;
    int32_t top = 0;          // free blocks (host mirror of the device stack top)
    int32_t* d_stack = nullptr;
    // Orders stream-side stack operations (wave pops in the plan kernel,
    // commit / abort pushes) of transitions on different streams in host
    // issue order, which is the order the host mirror `top` assumed.
    cudaEvent_t order = nullptr;
    bool order_live = false;
    // Host-array pop/push/snapshot/reset run on this private stream (after
    // `order`) and wait for it alone -- never for the device -- so they do not
    // stall behind serving kernels on other streams.
    cudaStream_t stream = nullptr;
    int32_t* h_stage = nullptr;  // pinned staging of host ids
    int32_t h_stage_cap = 0;
    int32_t* err = nullptr;      // pinned, device-mapped: a bad id pushed from the device
};

// Stack-op ordering across streams (see kvx_blockmgr::order).
inline cudaError_t bm_order_before(kvx_blockmgr* bm, cudaStream_t s) {
    return bm->order_live ? cudaStreamWaitEvent(s, bm->order, 0) : cudaSuccess;
}
inline cudaError_t bm_order_after(kvx_blockmgr* bm, cudaStream_t s) {
    const cudaError_t e = cudaEventRecord(bm->order, s);
    if (e == cudaSuccess) bm->order_live = true;
    return e;
}

struct kvx_transition {
    kvx_geometry g{};
    int32_t device = -1;
    cudaStream_t stream = nullptr;
    bool own_stream = true;
    int num_sms = 0;
    int move_ctas_per_sm = 1;
    int bulk_ctas[32] = {};  // resident CTAs per SM of each bulk variant
    int bulk_variant_slab = kvx_host::kSlabVariant;  // ring of slab-sized waves (KVX_BULK_CFG[_SLAB])
    int bulk_variant_tok = kvx_host::kTokVariant;    // ring of token-granular waves (KVX_BULK_CFG[_TOK])
    bool use_bulk = false;   // TMA bulk mover for local destinations
    bool peer_bulk = false;  // ... and for peer (NVLink) destinations
    bool lsu256 = false;     // LSU mover with 256-bit accesses (KVX_MOVE_IMPL=lsu256)
    std::vector<int32_t> old_b, new_b;
    std::vector<kvx_pool*> old_pools, new_pools;
    int32_t max_requests = 0, max_blocks = 0, dst_num_blocks = 0;
    kvx_blockmgr* bm = nullptr;  // destination block manager (NULL: bump rule)
    uint64_t epoch = 0;
    enum State { kActive, kCommitPending, kCommitted, kAborted } state = kActive;

    // device state
    int32_t* d_err = nullptr;  // error word (plan/commit bounds check) in pinned, device-mapped memory
    int32_t src_cap = 0;       // smallest old-pool block count: valid source ids are [0, src_cap)
    int32_t* d_src_bt = nullptr;
    int32_t* d_dst_bt = nullptr;
    int64_t* d_synced_hi = nullptr;
    kvx::LayerPtr* d_layers = nullptr;
    int32_t n_local_layers = 0;
    int32_t n_peer_layers = 0;  // layers [0, n_peer_layers) of d_layers cross NVLink (pushed or pulled)
    int32_t n_pull_layers = 0;  // of which pulled (read from a peer's old pool)
    bool transpose = false;     // some layer pairs a token-major with a head-major pool
    bool head_tails = false;    // head-major to head-major layers (H > 1): partial blocks go to the row mover
    // TMA tensor-map transposer (kvx_tmap_kernel) for the whole blocks of a
    // transposing transition: one map per local layer over its token-major side
    CUtensorMap* d_maps = nullptr;
    size_t maps_bytes = 0;
    int tmap_t2h = -1;          // -1: not used; 1: token-major -> head-major; 0: the reverse
    int tmap_hc = 0;            // heads per box
    cudaStream_t side = nullptr;  // side stream (arena-cached): head-major tails, the commit kernel
    cudaEvent_t ev_side_commit = nullptr;
    int last_plan_slot = -1;      // h_wave_free[slot] recorded after the most recent plan kernel
    bool handoff_since_plan = false;
    int32_t max_ctas = 0;         // cap on mover CTAs per wave (0 = tuned grid)
    cudaEvent_t ev_join = nullptr;
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
    // the handle's most recent work on its (possibly shared) stream: kvx_destroy
    // waits for this event, not for the whole stream, so a caller that reuses
    // one stream for consecutive transitions never drains it at a destroy
    cudaEvent_t ev_ready = nullptr;  // recorded at the end of kvx_begin
    cudaEvent_t last_ev = nullptr;
    // timing
    cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
    bool timing_open = false;
    // per move-kernel launch of this handle: its duration from the bulk mover's
    // own %globaltimer slots (timer >= 0), else a (start, end) event pair
    struct MoveRec {
        cudaEvent_t a = nullptr, b = nullptr;
        int32_t timer = -1;
    };
    std::vector<MoveRec> move_rec;
    std::vector<uint64_t> move_bytes;
    static constexpr int32_t kTimerSlots = 64;
    unsigned long long* d_timer = nullptr;  // [start x kTimerSlots | end x kTimerSlots]
    int32_t n_timers = 0;

    // activation handoff pieces (grown on demand, freed at destroy)
    kvx::Piece* d_pieces = nullptr;
    kvx::Piece* h_pieces = nullptr;
    int64_t piece_cap = 0;
    cudaEvent_t pieces_free = nullptr;

    // kvx_src_rows staging (pinned, read by kvx_rows_kernel) and its reuse event
    int32_t* h_rows = nullptr;
    size_t h_rows_bytes = 0;
    cudaEvent_t rows_free = nullptr;

    // host mirror of the destination rule (capacity checks are synchronous)
    std::vector<int64_t> synced_hi;
    std::vector<int32_t> src_bt;  // host copy: every wave's source blocks must be backed
    int32_t alloc = 0;
    uint64_t bytes_moved = 0;       // by this handle (local-source layers)
    uint64_t bytes_all_layers = 0;  // reference-accounted, all layers

    kvx::CtlState ctl;  // control-plane mirror (kvx_ctl.cpp)
};

