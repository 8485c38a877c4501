// kvx_pool.cu -- paged KV pools (create / wrap / IPC export-import / read-write)
// and the synthetic payload helpers (fill, decode-append emulation).
#include "kvx_common.h"

using namespace kvx_host;

namespace kvx_host {
cudaError_t preload_pool_kernels() {
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, (const void*)kvx::kvx_fill_kernel);
}
}  // namespace kvx_host

extern "C" {

// ------------------------------------------------------------------ pools
int kvx_stage_kv_bytes(const kvx_geometry* g, int32_t num_stages, const int32_t* boundaries,
                       int32_t dst_num_blocks, uint64_t* out) {
    std::string why;
    if (!geometry_ok(g, &why)) return fail(KVX_EINVAL, why);
    if (!out || dst_num_blocks < 0) return fail(KVX_EINVAL, "bad arguments");
    kvx_pool* dummy = nullptr;
    const kvx_plan p{num_stages, boundaries, &dummy};
    std::vector<int32_t> b;
    if (!plan_ok(p, g->num_layers, &why, &b)) return fail(KVX_EINVAL, why);
    for (int k = 0; k < num_stages; ++k) {
        const int32_t layers = (k + 1 < num_stages ? b[(size_t)k] : g->num_layers) - stage_begin(b, k);
        out[k] = (uint64_t)layers * (uint64_t)dst_num_blocks * block_bytes(*g);
    }
    return KVX_OK;
}

int kvx_pool_create(int32_t device, const kvx_geometry* g, int32_t num_layers, int32_t num_blocks,
                    kvx_pool** out) {
    return kvx_pool_create_layout(device, g, num_layers, num_blocks, KVX_LAYOUT_BLOCKS, out);
}

int kvx_pool_create_layout(int32_t device, const kvx_geometry* g, int32_t num_layers, int32_t num_blocks,
                           int32_t layout, kvx_pool** out) {
    std::string why;
    if (!out) return fail(KVX_EINVAL, "out is null");
    *out = nullptr;
    if (!geometry_ok(g, &why)) return fail(KVX_EINVAL, why);
    if (num_layers < 1 || num_blocks < 1) return fail(KVX_EINVAL, "num_layers/num_blocks must be >= 1");
    if (!layout_ok(layout)) return fail(KVX_EINVAL, "unknown layout");
    if (!layout_fits(layout, *g)) return fail(KVX_EINVAL, "head-major layout needs head_dim * elem_bytes % 16 == 0");
    DeviceGuard dg(device);
    if (!dg.ok) return fail(KVX_ECUDA, "cudaSetDevice failed for pool device");
    if (const int rc = ensure_loaded(device)) return rc;
    auto* p = new kvx_pool;
    p->device = device;
    p->g = *g;
    p->num_layers = num_layers;
    p->num_blocks = num_blocks;
    p->layout = layout;
    p->bytes = (uint64_t)num_layers * (uint64_t)num_blocks * block_bytes(*g);
    cudaError_t e = cudaMalloc(&p->base, p->bytes);
    if (e != cudaSuccess) {
        delete p;
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? KVX_ENOSPC : KVX_ECUDA,
                    std::string("pool cudaMalloc: ") + cudaGetErrorString(e));
    }
    p->set_contiguous_layers();
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
    p->set_contiguous_layers();
    *out = p;
    return KVX_OK;
}

int kvx_pool_wrap_layers(int32_t device, int32_t num_layers, void* const* layer_ptrs, uint64_t layer_bytes,
                         const kvx_geometry* g, int32_t num_blocks, int32_t layout, kvx_pool** out) {
    std::string why;
    if (!out) return fail(KVX_EINVAL, "out is null");
    *out = nullptr;
    if (!geometry_ok(g, &why)) return fail(KVX_EINVAL, why);
    if (num_layers < 1 || num_blocks < 1) return fail(KVX_EINVAL, "num_layers/num_blocks must be >= 1");
    if (!layout_ok(layout)) return fail(KVX_EINVAL, "unknown layout");
    if (!layout_fits(layout, *g)) return fail(KVX_EINVAL, "head-major layout needs head_dim * elem_bytes % 16 == 0");
    if (!layer_ptrs) return fail(KVX_EINVAL, "layer_ptrs is null");
    if (layer_bytes < (uint64_t)num_blocks * block_bytes(*g))
        return fail(KVX_EINVAL, "layer allocation smaller than num_blocks blocks");
    for (int32_t l = 0; l < num_layers; ++l)
        if (!layer_ptrs[l] || (reinterpret_cast<uintptr_t>(layer_ptrs[l]) & 15))
            return fail(KVX_EINVAL, "layer pointers must be non-null and 16-byte aligned");
    auto* p = new kvx_pool;
    p->device = device;
    p->wrapped = true;
    p->per_layer = true;
    p->base = static_cast<char*>(layer_ptrs[0]);
    p->g = *g;
    p->num_layers = num_layers;
    p->num_blocks = num_blocks;
    p->layout = layout;
    p->bytes = (uint64_t)num_layers * (uint64_t)num_blocks * block_bytes(*g);
    p->layer_base.assign((char* const*)layer_ptrs, (char* const*)layer_ptrs + num_layers);
    *out = p;
    return KVX_OK;
}

int kvx_pool_layout(const kvx_pool* p, int32_t* layout) {
    if (!p || !layout) return fail(KVX_EINVAL, "null argument");
    *layout = p->layout;
    return KVX_OK;
}

int kvx_pool_export(const kvx_pool* p, uint8_t handle[KVX_IPC_HANDLE_BYTES]) {
    if (!p || !handle || p->imported || p->per_layer) return fail(KVX_EINVAL, "export needs a local single-allocation pool");
    static_assert(sizeof(cudaIpcMemHandle_t) == KVX_IPC_HANDLE_BYTES, "ipc handle size");
    DeviceGuard dg(p->device);
    cudaIpcMemHandle_t h;
    KVX_CUDA(cudaIpcGetMemHandle(&h, p->base));
    std::memcpy(handle, &h, sizeof(h));
    return KVX_OK;
}

int kvx_pool_import(int32_t device, const uint8_t handle[KVX_IPC_HANDLE_BYTES],
                    const kvx_geometry* g, int32_t num_layers, int32_t num_blocks, kvx_pool** out) {
    return kvx_pool_import_layout(device, handle, g, num_layers, num_blocks, KVX_LAYOUT_BLOCKS, out);
}

int kvx_pool_import_layout(int32_t device, const uint8_t handle[KVX_IPC_HANDLE_BYTES], const kvx_geometry* g,
                           int32_t num_layers, int32_t num_blocks, int32_t layout, kvx_pool** out) {
    std::string why;
    if (!out || !handle) return fail(KVX_EINVAL, "null argument");
    *out = nullptr;
    if (!geometry_ok(g, &why)) return fail(KVX_EINVAL, why);
    if (num_layers < 1 || num_blocks < 1) return fail(KVX_EINVAL, "num_layers/num_blocks must be >= 1");
    if (!layout_ok(layout)) return fail(KVX_EINVAL, "unknown layout");
    if (!layout_fits(layout, *g)) return fail(KVX_EINVAL, "head-major layout needs head_dim * elem_bytes % 16 == 0");
    DeviceGuard dg(device);
    if (const int rc = ensure_loaded(device)) return rc;
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
    p->layout = layout;
    p->bytes = (uint64_t)num_layers * (uint64_t)num_blocks * block_bytes(*g);
    p->set_contiguous_layers();
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
    if (p->per_layer) {
        for (char* b : p->layer_base) KVX_CUDA(cudaMemset(b, 0, p->layer_bytes()));
    } else {
        KVX_CUDA(cudaMemset(p->base, 0, p->bytes));
    }
    KVX_CUDA(cudaDeviceSynchronize());
    return KVX_OK;
}

int kvx_pool_read(const kvx_pool* p, uint64_t offset, uint64_t bytes, void* host) {
    if (!p || !host || offset + bytes > p->bytes) return fail(KVX_EINVAL, "read out of range");
    if (p->per_layer) return fail(KVX_EINVAL, "per-layer pool: read each layer's own allocation");
    DeviceGuard dg(p->device);
    KVX_CUDA(cudaMemcpy(host, p->base + offset, bytes, cudaMemcpyDeviceToHost));
    return KVX_OK;
}

int kvx_pool_write(kvx_pool* p, uint64_t offset, uint64_t bytes, const void* host) {
    if (!p || !host || offset + bytes > p->bytes) return fail(KVX_EINVAL, "write out of range");
    if (p->per_layer) return fail(KVX_EINVAL, "per-layer pool: write each layer's own allocation");
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
        void *req = nullptr, *tok = nullptr, *bt = nullptr, *lay = nullptr;
        size_t nreq, ntok, nbt, nlay;
        ~Scratch() {
            a.dev_free(req, nreq);
            a.dev_free(tok, ntok);
            a.dev_free(bt, nbt);
            a.dev_free(lay, nlay);
        }
    } sc{A, nullptr, nullptr, nullptr, nullptr, sizeof(int32_t) * n, sizeof(int64_t) * n, bt_bytes,
         sizeof(char*) * p->layer_base.size()};
    KVX_CUDA(A.dev_alloc(&sc.req, sc.nreq));
    KVX_CUDA(A.dev_alloc(&sc.tok, sc.ntok));
    KVX_CUDA(A.dev_alloc(&sc.bt, sc.nbt));
    KVX_CUDA(A.dev_alloc(&sc.lay, sc.nlay));
    KVX_CUDA(cudaMemcpy(sc.req, req, sc.nreq, cudaMemcpyHostToDevice));
    KVX_CUDA(cudaMemcpy(sc.tok, tokens, sc.ntok, cudaMemcpyHostToDevice));
    KVX_CUDA(cudaMemcpy(sc.bt, bt, sc.nbt, cudaMemcpyHostToDevice));
    KVX_CUDA(cudaMemcpy(sc.lay, p->layer_base.data(), sc.nlay, cudaMemcpyHostToDevice));
    dim3 grid((unsigned)n, (unsigned)std::min<int64_t>(65535, cdiv64(max_tok, p->g.block_tokens)));
    kvx::kvx_fill_kernel<<<grid, 256>>>(pool_addr(p, static_cast<char* const*>(sc.lay)), first_layer, p->num_layers,
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
    const size_t o_lay = (o_bt + sizeof(int32_t) * (size_t)max_requests * (size_t)max_blocks + 15) & ~size_t(15);
    const size_t bytes = o_lay + sizeof(char*) * p->layer_base.size();
    void *d = nullptr, *h = nullptr;
    KVX_CUDA(A.dev_alloc(&d, bytes));
    KVX_CUDA(A.host_alloc(&h, bytes));
    char* hc = static_cast<char*>(h);
    std::memcpy(hc, req, sizeof(int32_t) * (size_t)n);
    std::memcpy(hc + o_from, from, sizeof(int64_t) * (size_t)n);
    std::memcpy(hc + o_to, to, sizeof(int64_t) * (size_t)n);
    std::memcpy(hc + o_bt, bt, sizeof(int32_t) * (size_t)max_requests * (size_t)max_blocks);
    std::memcpy(hc + o_lay, p->layer_base.data(), sizeof(char*) * p->layer_base.size());
    KVX_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
    char* dc = static_cast<char*>(d);
    dim3 grid((unsigned)n, (unsigned)std::min<int64_t>(65535, cdiv64(max_tok, p->g.block_tokens)));
    kvx::kvx_fill_kernel<<<grid, 256, 0, st>>>(pool_addr(p, reinterpret_cast<char* const*>(dc + o_lay)),
                                               first_layer, p->num_layers,
                                               reinterpret_cast<const int32_t*>(dc),
                                               reinterpret_cast<const int64_t*>(dc + o_to),
                                               reinterpret_cast<const int32_t*>(dc + o_bt), max_blocks,
                                               p->g.block_tokens, token_bytes(p->g), seed,
                                               reinterpret_cast<const int64_t*>(dc + o_from));
    KVX_LAUNCHED();
    KVX_CUDA(cudaLaunchHostFunc(st, release_pieces, new PieceRelease{p->device, d, h, bytes}));
    return KVX_OK;
}


}  // extern "C"
