// kvx_extras.cu -- SURVEY 8(f): stage-boundary activation handoff, stage weight
// migration, and the device-resident block manager.
#include "kvx_common.h"

using namespace kvx_host;

namespace {
// copy-list rings: handoff rows (short runs) and weight layers (long runs)
constexpr int kHandoffStages = 4, kWeightStages = 6;
constexpr uint32_t kCopyChunk = 32768;
// weight layers are long contiguous runs: the slab ring (3 x 64 KiB)
constexpr int kWeightSlabStages = 3;
constexpr uint32_t kWeightSlabChunk = 65536;
}  // namespace

namespace kvx_host {
cudaError_t preload_extras_kernels() {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(kvx::kvx_copy_list_kernel<kHandoffStages, kCopyChunk>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kHandoffStages * (int)kCopyChunk)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(kvx::kvx_copy_list_kernel<kWeightStages, kCopyChunk>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kWeightStages * (int)kCopyChunk)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(kvx::kvx_copy_list_kernel<kWeightSlabStages, kWeightSlabChunk>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kWeightSlabStages * (int)kWeightSlabChunk)) != cudaSuccess)
        return e;
    // every block-manager kernel: a lazily loaded one would wait for the
    // serving kernels running at its first launch
    cudaFuncAttributes a;
    for (const void* fn : {(const void*)kvx::kvx_bm_init_kernel, (const void*)kvx::kvx_bm_pop_kernel,
                           (const void*)kvx::kvx_bm_push_kernel})
        if ((e = cudaFuncGetAttributes(&a, fn)) != cudaSuccess) return e;
    return cudaSuccess;
}
}  // namespace kvx_host

extern "C" {

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
        if (a >= k_old) return fail(KVX_EINVAL, "after_stage beyond the old pipeline");
        if (a < 0 || a + 1 == k_old) {
            // a < 0: nothing computed yet, re-dispatch at the new head;
            // a == K_old-1: the forward pass is complete, not in flight (no slot)
            sl.new_stage = a < 0 ? 0 : -1;
            sl.resume_layer = a < 0 ? 0 : -1;
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
    t->handoff_since_plan = true;  // the commit then stays on the main stream (kvx_commit_async)
    DeviceGuard dg(t->device);
    kvx::Arena& A = kvx::Arena::of(t->device);
    if (!t->pieces_free) KVX_CUDA(A.event(&t->pieces_free, false));
    KVX_CUDA(cudaEventSynchronize(t->pieces_free));  // previous handoff's upload consumed
    if ((int64_t)pieces.size() > t->piece_cap) {
        KVX_CUDA(cudaStreamSynchronize(t->stream));  // a previous copy-list kernel may still read them
        A.dev_free(t->d_pieces, sizeof(kvx::Piece) * (size_t)t->piece_cap);
        A.host_free(t->h_pieces, sizeof(kvx::Piece) * (size_t)t->piece_cap);
        t->d_pieces = nullptr;
        t->h_pieces = nullptr;
        const int64_t cap = (int64_t)(kvx::size_class(sizeof(kvx::Piece) * pieces.size()) / sizeof(kvx::Piece));
        KVX_CUDA(A.dev_alloc((void**)&t->d_pieces, sizeof(kvx::Piece) * (size_t)cap));
        KVX_CUDA(A.host_alloc((void**)&t->h_pieces, sizeof(kvx::Piece) * (size_t)cap));
        t->piece_cap = cap;
    }
    std::memcpy(t->h_pieces, pieces.data(), sizeof(kvx::Piece) * pieces.size());
    KVX_CUDA(cudaMemcpyAsync(t->d_pieces, t->h_pieces, sizeof(kvx::Piece) * pieces.size(),
                             cudaMemcpyHostToDevice, t->stream));
    KVX_CUDA(cudaEventRecord(t->pieces_free, t->stream));
    constexpr int kStages = kHandoffStages;
    constexpr uint32_t kChunk = kCopyChunk;  // smem attribute set by preload_extras_kernels
    const unsigned grid = (unsigned)std::min<int64_t>(2 * (int64_t)t->num_sms, (int64_t)pieces.size());
    kvx::kvx_copy_list_kernel<kStages, kChunk><<<grid, kvx::kBulkThreads, kStages * kChunk, t->stream>>>(
        t->d_pieces, (int64_t)pieces.size());
    KVX_LAUNCHED();
    KVX_CUDA(cudaEventRecord(t->ev_end, t->stream));  // the handoff lands inside the wave window
    t->last_ev = t->ev_end;
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
    // validate every layer before anything is enqueued (nothing half-applied)
    for (int32_t l = 0; l < num_layers; ++l) {
        if (!new_ptrs[stage_of_layer(nb, l)]) return fail(KVX_EINVAL, "weights: every new stage buffer is required");
        if (from_host && from_host[l] && !host_cache)
            return fail(KVX_EINVAL, "weights: from_host without a host cache");
    }
    std::vector<kvx::Piece> pieces;
    uint64_t dev_b = 0, host_b = 0;
    DeviceGuard dg(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    for (int32_t l = 0; l < num_layers; ++l) {
        const int so = stage_of_layer(ob, l), sn = stage_of_layer(nb, l);
        char* dst = static_cast<char*>(new_ptrs[sn]) + (uint64_t)(l - stage_begin(nb, sn)) * layer_bytes;
        if (from_host && from_host[l]) {
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
    if (const int rc = ensure_loaded(device)) return rc;  // also sets the smem attributes
    // experiment knobs: KVX_WEIGHTS_RING=slab|32k, KVX_WEIGHTS_GRID=<ctas>
    const char* ring = getenv("KVX_WEIGHTS_RING");
    const bool slab = !(ring && std::string(ring) == "32k");
    int64_t gcap = slab ? 96 : (int64_t)sms;
    if (const char* gg = getenv("KVX_WEIGHTS_GRID")) gcap = std::max<int64_t>(1, atoll(gg));
    const unsigned grid = (unsigned)std::min<int64_t>(std::min<int64_t>(gcap, sms), (int64_t)pieces.size());
    if (slab)
        kvx::kvx_copy_list_kernel<kWeightSlabStages, kWeightSlabChunk>
            <<<grid, kvx::kBulkThreads, kWeightSlabStages * kWeightSlabChunk, st>>>(
                static_cast<const kvx::Piece*>(d), (int64_t)pieces.size());
    else
        kvx::kvx_copy_list_kernel<kWeightStages, kCopyChunk><<<grid, kvx::kBulkThreads, kWeightStages * kCopyChunk, st>>>(
            static_cast<const kvx::Piece*>(d), (int64_t)pieces.size());
    KVX_LAUNCHED();
    KVX_CUDA(cudaLaunchHostFunc(st, release_pieces, new PieceRelease{device, d, h, bytes}));
    return KVX_OK;
}

}  // extern "C"

// ------------------------------------------------------------ block manager
// Every stack operation is stream-ordered behind bm->order (the previous
// stack op, on whatever stream it ran); the host-array calls run on the
// manager's private stream and wait for that stream alone.
namespace {
int bm_check_err(const kvx_blockmgr* bm) {
    if (bm->err && *reinterpret_cast<volatile int32_t*>(bm->err))
        return fail(KVX_EINVAL, "block manager: a device push carried an id outside [0, capacity)");
    return KVX_OK;
}
cudaError_t bm_stage(kvx_blockmgr* bm, int32_t n) {  // pinned staging of >= n ids
    if (n <= bm->h_stage_cap) return cudaSuccess;
    kvx::Arena& A = kvx::Arena::of(bm->device);
    if (bm->h_stage) {
        const cudaError_t e = cudaStreamSynchronize(bm->stream);
        if (e != cudaSuccess) return e;
        A.host_free(bm->h_stage, sizeof(int32_t) * (size_t)bm->h_stage_cap);
        bm->h_stage = nullptr;
    }
    const size_t bytes = kvx::size_class(sizeof(int32_t) * (size_t)n);
    const cudaError_t e = A.host_alloc((void**)&bm->h_stage, bytes);
    bm->h_stage_cap = e == cudaSuccess ? (int32_t)(bytes / sizeof(int32_t)) : 0;
    return e;
}
unsigned bm_grid(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(1024, (n + 255) / 256)); }
}  // namespace

extern "C" {

int kvx_bm_create(int32_t device, int32_t capacity, kvx_blockmgr** out) {
    if (!out || capacity < 1) return fail(KVX_EINVAL, "bad block manager arguments");
    *out = nullptr;
    DeviceGuard dg(device);
    if (!dg.ok) return fail(KVX_ECUDA, "cudaSetDevice failed");
    if (const int rc = ensure_loaded(device)) return rc;
    auto* bm = new kvx_blockmgr;
    bm->device = device;
    bm->capacity = capacity;
    kvx::Arena& A = kvx::Arena::of(device);
    if (A.dev_alloc((void**)&bm->d_stack, sizeof(int32_t) * (size_t)capacity) != cudaSuccess) {
        delete bm;
        cudaGetLastError();
        return fail(KVX_ENOSPC, "block manager allocation failed");
    }
    if (cudaEventCreateWithFlags(&bm->order, cudaEventDisableTiming) != cudaSuccess ||
        A.stream(&bm->stream) != cudaSuccess || A.host_alloc((void**)&bm->err, sizeof(int32_t)) != cudaSuccess) {
        kvx_bm_destroy(bm);
        return fail(KVX_ECUDA, "block manager stream / event / error word");
    }
    *bm->err = 0;
    *out = bm;
    return kvx_bm_reset(bm);
}

int kvx_bm_reset(kvx_blockmgr* bm) {
    if (!bm) return fail(KVX_EINVAL, "block manager is null");
    DeviceGuard dg(bm->device);
    KVX_CUDA(bm_order_before(bm, bm->stream));
    kvx::kvx_bm_init_kernel<<<bm_grid(bm->capacity), 256, 0, bm->stream>>>(bm->d_stack, bm->capacity);
    KVX_LAUNCHED();
    KVX_CUDA(bm_order_after(bm, bm->stream));
    KVX_CUDA(cudaStreamSynchronize(bm->stream));
    *bm->err = 0;
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
    if (const int rc = bm_check_err(bm)) return rc;
    if (n > bm->top) return fail(KVX_ENOSPC, "block manager exhausted");
    if (n == 0) return KVX_OK;
    DeviceGuard dg(bm->device);
    KVX_CUDA(bm_stage(bm, n));
    // behind the stack's last op (pushes queued on transition streams), on the
    // manager's own stream: no wait on unrelated streams
    KVX_CUDA(bm_order_before(bm, bm->stream));
    KVX_CUDA(cudaMemcpyAsync(bm->h_stage, bm->d_stack + (bm->top - n), sizeof(int32_t) * (size_t)n,
                             cudaMemcpyDeviceToHost, bm->stream));
    KVX_CUDA(bm_order_after(bm, bm->stream));
    KVX_CUDA(cudaStreamSynchronize(bm->stream));
    for (int32_t i = 0; i < n; ++i) ids_out[i] = bm->h_stage[n - 1 - i];  // LIFO order
    bm->top -= n;
    return KVX_OK;
}

int kvx_bm_push(kvx_blockmgr* bm, int32_t n, const int32_t* ids) {
    if (!bm || n < 0 || (n > 0 && !ids)) return fail(KVX_EINVAL, "bad push arguments");
    if (const int rc = bm_check_err(bm)) return rc;
    if (bm->top + n > bm->capacity) return fail(KVX_EINVAL, "push beyond capacity (double free?)");
    for (int32_t i = 0; i < n; ++i)
        if (ids[i] < 0 || ids[i] >= bm->capacity) return fail(KVX_EINVAL, "block id out of range");
    if (n == 0) return KVX_OK;
    DeviceGuard dg(bm->device);
    KVX_CUDA(bm_stage(bm, n));
    KVX_CUDA(cudaStreamSynchronize(bm->stream));  // the staging buffer's previous upload is consumed
    std::memcpy(bm->h_stage, ids, sizeof(int32_t) * (size_t)n);
    KVX_CUDA(bm_order_before(bm, bm->stream));
    KVX_CUDA(cudaMemcpyAsync(bm->d_stack + bm->top, bm->h_stage, sizeof(int32_t) * (size_t)n,
                             cudaMemcpyHostToDevice, bm->stream));
    KVX_CUDA(bm_order_after(bm, bm->stream));
    bm->top += n;
    return KVX_OK;
}

int kvx_bm_pop_async(kvx_blockmgr* bm, int32_t n, int32_t* dev_ids_out, void* stream) {
    if (!bm || n < 0 || (n > 0 && !dev_ids_out)) return fail(KVX_EINVAL, "bad pop arguments");
    if (const int rc = bm_check_err(bm)) return rc;
    if (n > bm->top) return fail(KVX_ENOSPC, "block manager exhausted");
    if (n == 0) return KVX_OK;
    DeviceGuard dg(bm->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    KVX_CUDA(bm_order_before(bm, s));
    kvx::kvx_bm_pop_kernel<<<bm_grid(n), 256, 0, s>>>(bm->d_stack, bm->top, n, dev_ids_out);
    KVX_LAUNCHED();
    KVX_CUDA(bm_order_after(bm, s));
    bm->top -= n;
    return KVX_OK;
}

int kvx_bm_push_async(kvx_blockmgr* bm, int32_t n, const int32_t* dev_ids, void* stream) {
    if (!bm || n < 0 || (n > 0 && !dev_ids)) return fail(KVX_EINVAL, "bad push arguments");
    if (const int rc = bm_check_err(bm)) return rc;
    if (bm->top + n > bm->capacity) return fail(KVX_EINVAL, "push beyond capacity (double free?)");
    if (n == 0) return KVX_OK;
    DeviceGuard dg(bm->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    KVX_CUDA(bm_order_before(bm, s));
    kvx::kvx_bm_push_kernel<<<bm_grid(n), 256, 0, s>>>(bm->d_stack, bm->top, n, dev_ids, bm->capacity, bm->err);
    KVX_LAUNCHED();
    KVX_CUDA(bm_order_after(bm, s));
    bm->top += n;
    return KVX_OK;
}

int kvx_bm_snapshot(const kvx_blockmgr* bm, int32_t* stack_out, int32_t* top_out) {
    if (!bm) return fail(KVX_EINVAL, "block manager is null");
    if (const int rc = bm_check_err(bm)) return rc;
    DeviceGuard dg(bm->device);
    auto* m = const_cast<kvx_blockmgr*>(bm);  // ordering state only; the stack is not modified
    KVX_CUDA(bm_order_before(m, m->stream));
    if (stack_out && bm->top > 0)
        KVX_CUDA(cudaMemcpyAsync(stack_out, bm->d_stack, sizeof(int32_t) * (size_t)bm->top, cudaMemcpyDeviceToHost,
                                 m->stream));
    KVX_CUDA(cudaStreamSynchronize(m->stream));
    if (top_out) *top_out = bm->top;
    return KVX_OK;
}

int kvx_bm_destroy(kvx_blockmgr* bm) {
    if (!bm) return KVX_OK;
    DeviceGuard dg(bm->device);
    kvx::Arena& A = kvx::Arena::of(bm->device);
    if (bm->order) {
        if (bm->order_live) cudaEventSynchronize(bm->order);  // the stack's last op, on any stream
        cudaEventDestroy(bm->order);
    }
    if (bm->stream) {
        cudaStreamSynchronize(bm->stream);
        A.stream_free(bm->stream);
    }
    A.dev_free(bm->d_stack, sizeof(int32_t) * (size_t)bm->capacity);
    A.host_free(bm->h_stage, sizeof(int32_t) * (size_t)bm->h_stage_cap);
    A.host_free(bm->err, sizeof(int32_t));
    delete bm;
    return KVX_OK;
}


}  // extern "C"
