// kvx_transition.cu -- one inflight refactor on one local GPU (RefactorCtx,
// /root/reference/proj/include/pipesim/engine.hpp:149-158): grant, waves,
// wait, commit (sync / async), abort, destroy and introspection.
//
// In a multi-GPU transition every rank opens its own handle over the same
// plans; each moves the layers whose OLD stage lives on its GPU and pushes
// them into the destination pools (local, or a peer's through NVLink P2P) --
// or, with desc.pull, the layers whose NEW stage is local.  The destination
// block rule is deterministic, so every rank derives the same destination
// block table without exchanging it.
#include "kvx_common.h"

#include <cudaTypedefs.h>

#include <map>
#include <mutex>

using namespace kvx_host;

namespace {
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tmap_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// The token-major side of one layer as a 5-D tensor (D, B, H, K|V, block),
// dims ordered head-outer so a (D, B, hc) box is a head-major smem tile.
struct TmSide {
    char* base;
    int32_t num_blocks;
    uint64_t ts, hs, kv, bs;
    bool local;  // the pool is this device's own (tensor maps only over local memory)
};
}  // namespace

namespace {
// What kvx_begin needs to know about a device's occupancy, queried once per
// device: a grant is on the engine's refactor path, and 20+ occupancy /
// attribute queries per grant cost ~0.1-0.5 ms of host time.
struct DeviceCaps {
    int num_sms = 0;
    int move_ctas_per_sm = 1;
    int bulk_ctas[kNumBulkVariants] = {};
};
int device_caps(int device, DeviceCaps* out) {
    static std::mutex mu;
    static std::map<int, DeviceCaps> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(device);
    if (it != cache.end()) {
        *out = it->second;
        return KVX_OK;
    }
    DeviceCaps c;
    int occ = 0;
    if (cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
        return fail(KVX_ECUDA, "query SM count");
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kvx::kvx_move_kernel, kvx::kMoveThreads, 0) != cudaSuccess)
        return fail(KVX_ECUDA, "occupancy query");
    c.move_ctas_per_sm = std::max(1, occ);
    for (int v = 0; v < kNumBulkVariants; ++v) {
        const BulkVariant& bv = kBulkVariants[v];
        const int smem = bv.stages * (int)bv.chunk;
        if (cudaFuncSetAttribute(bv.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bv.fn, kvx::kBulkThreads, smem) != cudaSuccess)
            return fail(KVX_ECUDA, "bulk kernel attributes");
        c.bulk_ctas[v] = std::max(1, occ);
    }
    cache[device] = c;
    *out = c;
    return KVX_OK;
}
}  // namespace

namespace kvx_host {
cudaError_t preload_transition_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaSuccess;
    for (const void* fn : {(const void*)kvx::kvx_plan_kernel, (const void*)kvx::kvx_move_kernel,
                           (const void*)kvx::kvx_rows_kernel,
                           (const void*)kvx::kvx_move_any_kernel,
                           (const void*)kvx::kvx_move256_kernel, (const void*)kvx::kvx_commit_kernel,
                           (const void*)kvx::kvx_verify_kernel})
        if ((e = cudaFuncGetAttributes(&a, fn)) != cudaSuccess) return e;
    for (const BulkVariant& bv : kBulkVariants)
        if ((e = cudaFuncSetAttribute(bv.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      bv.stages * (int)bv.chunk)) != cudaSuccess)
            return e;
    if ((e = cudaFuncSetAttribute(kvx::kvx_tmap_kernel<kTmapStages, kTmapLag>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kTmapStages * (int)kTmapSlot)) !=
        cudaSuccess)
        return e;
    return e;
}
}  // namespace kvx_host

extern "C" {

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
    if (d->max_ctas < 0) return fail(KVX_EINVAL, "max_ctas must be >= 0");
    const bool dev_table = d->src_block_table_dev != nullptr;  // serving engine's device copy
    if (!d->src_block_table && !dev_table) return fail(KVX_EINVAL, "src_block_table is null");
    for (int k = 0; k < d->new_plan.num_stages; ++k) {
        const kvx_pool* p = d->new_plan.pools[k];
        if (!p) {
            // pull / per-layer movers: only the pools of layers moved here are needed
            // (checked per layer below)
            if (d->pull || d->layer_pull) continue;
            return fail(KVX_EINVAL, "every new-stage pool is required");
        }
        const int32_t layers = (k + 1 < d->new_plan.num_stages ? nb[(size_t)k] : g.num_layers) -
                               stage_begin(nb, k);
        if (p->num_layers != layers) return fail(KVX_EINVAL, "new pool layer count != stage layer range");
        if (p->num_blocks < d->dst_num_blocks) return fail(KVX_EINVAL, "new pool smaller than dst_num_blocks");
        if (!p->imported && p->device != d->device && !peer_ok(d->device, p->device))
            return fail(KVX_EINVAL, "local new pool on another device without peer access");
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
        if (!p->imported && p->device != d->device && !peer_ok(d->device, p->device))
            return fail(KVX_EINVAL, "local old pool on another device without peer access");
        if (p->imported && p->device != d->device) return fail(KVX_EINVAL, "imported old pool mapped for another device");
        if (p->g.num_kv_heads != g.num_kv_heads || p->g.head_dim != g.head_dim ||
            p->g.elem_bytes != g.elem_bytes || p->g.block_tokens != g.block_tokens)
            return fail(KVX_EINVAL, "old pool geometry mismatch");
    }
    // A destination must not alias a source: destination ids are allocated
    // from 0 and would overwrite source blocks a later wave still reads.
    for (int j = 0; j < d->new_plan.num_stages; ++j)
        for (int k = 0; k < d->old_plan.num_stages; ++k)
            if (pools_overlap(d->new_plan.pools[j], d->old_plan.pools[k]))
                return fail(KVX_EINVAL, "a new-stage pool overlaps an old-stage pool");
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
    if (!dev_table)  // a device table is checked per segment by the plan kernel instead
        for (size_t c = 0; c < cells; ++c) {
            const int32_t v = d->src_block_table[c];
            if (v >= min_old_blocks) return fail(KVX_EINVAL, "src_block_table id beyond an old pool");
        }

    DeviceGuard dg(d->device);
    if (!dg.ok) return fail(KVX_ECUDA, "cudaSetDevice failed");
    if (const int rc = ensure_loaded(d->device)) return rc;
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
    t->max_ctas = d->max_ctas;
    t->epoch = d->epoch;
    t->synced_hi.assign((size_t)d->max_requests, 0);
    if (!dev_table) t->src_bt.assign(d->src_block_table, d->src_block_table + cells);  // host mirror
    t->ctl.init(d->max_requests, d->max_sync_rounds,
                d->kv_bytes_per_token > 0.0 ? d->kv_bytes_per_token
                                            : (double)g.num_layers * (double)block_bytes(g) /
                                                  (double)g.block_tokens);
    auto bail = [&](int code) {
        kvx_destroy(t);
        return code;
    };
    DeviceCaps caps;
    if (const int rc = device_caps(d->device, &caps)) return bail(rc);
    t->num_sms = caps.num_sms;
    t->move_ctas_per_sm = caps.move_ctas_per_sm;
    {
        // Ring per wave kind (kvx_wave): slab waves (mostly full blocks) and
        // token-granular waves.  KVX_BULK_CFG pins one variant for both,
        // KVX_BULK_CFG_SLAB / _TOK one kind (sweeps).
        static_assert(kNumBulkVariants <= (int)(sizeof(t->bulk_ctas) / sizeof(t->bulk_ctas[0])), "variants");
        auto pick = [](const char* name, int dflt) {
            const char* v = getenv(name);
            return v ? std::max(0, std::min(kNumBulkVariants - 1, atoi(v))) : dflt;
        };
        t->bulk_variant_slab = pick("KVX_BULK_CFG_SLAB", pick("KVX_BULK_CFG", kSlabVariant));
        t->bulk_variant_tok = pick("KVX_BULK_CFG_TOK", pick("KVX_BULK_CFG", kTokVariant));
        for (int v = 0; v < kNumBulkVariants; ++v) t->bulk_ctas[v] = caps.bulk_ctas[v];
        // Bulk (TMA engine) mover by default, for local and peer (NVLink)
        // destinations alike; KVX_PEER_BULK=0 keeps the LSU mover for peer
        // pushes, KVX_MOVE_IMPL=lsu everywhere.
        const char* impl = getenv("KVX_MOVE_IMPL");
        t->use_bulk = !(impl && (std::string(impl) == "lsu" || std::string(impl) == "lsu256"));
        t->lsu256 = impl && std::string(impl) == "lsu256";
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
        A.dev_alloc((void**)&t->d_commit_out, 4 * sizeof(int64_t)) != cudaSuccess ||
        A.host_alloc((void**)&t->d_err, sizeof(int32_t)) != cudaSuccess)
        return bail(fail(KVX_ENOSPC, "transition state allocation failed"));
    *t->d_err = 0;  // pinned, device-mapped error word: no stream op resets or reads it
    t->src_cap = min_old_blocks;  // INT32_MAX when no old pool is visible here (no local sources)
    for (int s = 0; s < 2; ++s)
        if (A.host_alloc((void**)&t->h_wave[s], wave_bytes) != cudaSuccess ||
            A.event(&t->h_wave_free[s], false) != cudaSuccess)
            return bail(fail(KVX_ECUDA, "pinned staging allocation failed"));
    if (cudaMemcpyAsync(t->d_src_bt, dev_table ? d->src_block_table_dev : d->src_block_table, bt_bytes,
                        dev_table ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, t->stream) != cudaSuccess ||
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
        constexpr size_t kTimerBytes = sizeof(unsigned long long) * kvx_transition::kTimerSlots;
        if (A.dev_alloc((void**)&t->d_timer, 2 * kTimerBytes) != cudaSuccess ||
            cudaMemsetAsync(t->d_timer, 0xff, kTimerBytes, t->stream) != cudaSuccess ||  // starts: +inf
            cudaMemsetAsync(t->d_timer + kvx_transition::kTimerSlots, 0, kTimerBytes, t->stream) != cudaSuccess)
            return bail(fail(KVX_ENOSPC, "timer slots"));
        if (A.dev_alloc((void**)&t->d_segs, sizeof(kvx::Seg) * (size_t)t->seg_cap) != cudaSuccess ||
            A.dev_alloc((void**)&t->d_commit_i32, sizeof(int32_t) * (size_t)t->commit_i32_cap) != cudaSuccess ||
            A.host_alloc((void**)&t->h_commit, t->h_commit_bytes) != cudaSuccess ||
            A.event(&t->ev_commit, false) != cudaSuccess)
            return bail(fail(KVX_ENOSPC, "transition scratch allocation failed"));
    }

    // Per-layer slab bases for the layers this GPU sources.
    std::vector<kvx::LayerPtr> layers;
    std::vector<uint8_t> layer_is_peer;
    std::vector<TmSide> tm_side;  // per layer: the token-major pool of a transposing pair
    std::vector<int> tm_dir;      // 1: src token-major -> dst head-major, 0: the reverse, -1: same family
    for (int32_t l = 0; l < g.num_layers; ++l) {
        const int so = stage_of_layer(ob, l), sn = stage_of_layer(nb, l);
        kvx_pool* src = t->old_pools[(size_t)so];
        kvx_pool* dst = t->new_pools[(size_t)sn];
        // remote = behind NVLink: a peer rank's pool (CUDA IPC) or this process's pool on another GPU
        auto remote = [&](const kvx_pool* p) { return p->imported || p->device != d->device; };
        const bool src_local = src && !remote(src);
        const bool dst_local = dst && !remote(dst);
        const bool pulled = d->layer_pull ? d->layer_pull[l] != 0 : d->pull != 0;
        if (src_local && dst_local) {
            // both pools here: a local move whichever side would otherwise move it
        } else if (pulled) {  // this GPU owns the layer's destination; the source is a peer's
            if (!dst_local) continue;
            if (!src) return bail(fail(KVX_EINVAL, "pull: a local destination layer has no mapped source pool"));
            t->has_peer_dst = true;  // peer traffic on this handle
            ++t->n_pull_layers;
        } else {  // this GPU owns the layer's source and pushes it into the (peer) destination
            if (!src_local) continue;
            if (!dst) return bail(fail(KVX_EINVAL, "push: a local source layer has no mapped destination pool"));
        }
        // run copies need both sides token-major or both head-major; otherwise the
        // wave goes through the transposing mover (kvx_move_any_kernel)
        const bool heads_runs = src->head_major() && dst->head_major();
        if (src->head_major() != dst->head_major()) t->transpose = true;
        if (heads_runs && g.num_kv_heads > 1) t->head_tails = true;
        layers.push_back({src->layer_base[(size_t)(l - stage_begin(ob, so))],
                          dst->layer_base[(size_t)(l - stage_begin(nb, sn))], src->blk_stride(), dst->blk_stride(),
                          src->kv_stride(), dst->kv_stride(), src->tok_stride(), dst->tok_stride(),
                          src->head_stride(), dst->head_stride(),
                          (uint32_t)(heads_runs ? src->head_bytes() : token_bytes(g)),
                          heads_runs ? (uint32_t)g.num_kv_heads : 1u});
        layer_is_peer.push_back(remote(dst) || remote(src) ? 1 : 0);
        {
            const kvx_pool* tmp = src->head_major() ? dst : src;  // token-major side
            const size_t ll = (size_t)(l - (tmp == src ? stage_begin(ob, so) : stage_begin(nb, sn)));
            tm_side.push_back({tmp->layer_base[ll], tmp->num_blocks, tmp->tok_stride(), tmp->head_stride(),
                               tmp->kv_stride(), tmp->blk_stride(), !remote(tmp)});
            tm_dir.push_back(src->head_major() == dst->head_major() ? -1 : (dst->head_major() ? 1 : 0));
        }
        if (remote(dst)) t->has_peer_dst = true;
    }
    // peer-destination layers first (see kvx_bulk_kernel's CTA split)
    {
        std::vector<kvx::LayerPtr> peer, local;
        std::vector<TmSide> tpeer, tlocal;
        std::vector<int> dpeer, dlocal;
        for (size_t i = 0; i < layers.size(); ++i) {
            (layer_is_peer[i] ? peer : local).push_back(layers[i]);
            (layer_is_peer[i] ? tpeer : tlocal).push_back(tm_side[i]);
            (layer_is_peer[i] ? dpeer : dlocal).push_back(tm_dir[i]);
        }
        t->n_peer_layers = (int32_t)peer.size();
        layers = peer;
        layers.insert(layers.end(), local.begin(), local.end());
        tm_side = tpeer;
        tm_side.insert(tm_side.end(), tlocal.begin(), tlocal.end());
        tm_dir = dpeer;
        tm_dir.insert(tm_dir.end(), dlocal.begin(), dlocal.end());
    }
    // Whole blocks of a transposing transition on the TMA transposer: every
    // local layer pairs the two families in the same direction, the geometry
    // fits one box (D <= 256 elements, a head plane <= one ring slot) and the
    // driver encodes the maps; else everything stays on the row mover.
    // Default (KVX_TMAP=0 disables): 0.941-0.954 of the copy peak on whole blocks
    // on five of six boxes, against 0.93 for the row mover at best
    // (profiles/r02af_ab_transposers_same_box.jsonl and the r02*_ab_tmap files).
    if (t->transpose && !layers.empty() && !(getenv("KVX_TMAP") && std::string(getenv("KVX_TMAP")) == "0")) {
        const uint64_t head_plane = (uint64_t)g.block_tokens * g.head_dim * g.elem_bytes;
        bool ok = tm_dir[0] >= 0 && g.head_dim <= 256 && g.block_tokens <= 256 && head_plane <= kTmapSlot &&
                  (g.elem_bytes == 1 || g.elem_bytes == 2 || g.elem_bytes == 4) &&
                  ((uint64_t)g.head_dim * g.elem_bytes) % 16 == 0 && tmap_encode() != nullptr;
        for (int dir : tm_dir) ok = ok && dir == tm_dir[0];
        // tensor maps only over this device's own pools: a pulled token-major source
        // or a pushed token-major destination behind NVLink stays on the row mover
        for (const TmSide& s : tm_side) ok = ok && s.local;
        std::vector<CUtensorMap> maps(layers.size());
        const int hc = (int)std::min<uint64_t>((uint64_t)g.num_kv_heads, kTmapSlot / std::max<uint64_t>(1, head_plane));
        for (size_t i = 0; ok && i < layers.size(); ++i) {
            const TmSide& s = tm_side[i];
            const cuuint64_t dims[5] = {(cuuint64_t)g.head_dim, (cuuint64_t)g.block_tokens, (cuuint64_t)g.num_kv_heads, 2,
                                        (cuuint64_t)s.num_blocks};
            const cuuint64_t strides[4] = {s.ts, s.hs, s.kv, s.bs};
            const cuuint32_t box[5] = {(cuuint32_t)g.head_dim, (cuuint32_t)g.block_tokens, (cuuint32_t)hc, 1, 1};
            const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
            const CUtensorMapDataType dt = g.elem_bytes == 1   ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                           : g.elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                                               : CU_TENSOR_MAP_DATA_TYPE_UINT32;
            ok = tmap_encode()(&maps[i], dt, 5, s.base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
        if (ok) {
            t->maps_bytes = sizeof(CUtensorMap) * maps.size();
            if (kvx::Arena::of(d->device).dev_alloc((void**)&t->d_maps, t->maps_bytes) != cudaSuccess ||
                cudaMemcpyAsync(t->d_maps, maps.data(), t->maps_bytes, cudaMemcpyHostToDevice, t->stream) != cudaSuccess)
                return bail(fail(KVX_ECUDA, "tensor map upload"));
            t->tmap_t2h = tm_dir[0];
            t->tmap_hc = hc;
        }
    }
    t->n_local_layers = (int32_t)layers.size();
    if (!layers.empty()) {
        t->layers_bytes = sizeof(kvx::LayerPtr) * layers.size();
        if (A.dev_alloc((void**)&t->d_layers, t->layers_bytes) != cudaSuccess ||
            cudaMemcpyAsync(t->d_layers, layers.data(), sizeof(kvx::LayerPtr) * layers.size(),
                            cudaMemcpyHostToDevice, t->stream) != cudaSuccess)
            return bail(fail(KVX_ECUDA, "layer table upload"));
    }
    // side stream: the head-major tail mover beside the bulk mover, and the commit
    // kernel beside the last wave's mover (see kvx_wave / kvx_commit_async)
    if (A.stream(&t->side) != cudaSuccess || A.event(&t->ev_join, false) != cudaSuccess ||
        A.event(&t->ev_side_commit, false) != cudaSuccess)
        return bail(fail(KVX_ECUDA, "side stream"));
    // No host sync: the uploads above were staged from pageable memory
    // (copied out before cudaMemcpyAsync returned) and are stream-ordered
    // before every wave.
    if (A.event(&t->ev_ready, false) != cudaSuccess || cudaEventRecord(t->ev_ready, t->stream) != cudaSuccess)
        return bail(fail(KVX_ECUDA, "ready event"));
    t->last_ev = t->ev_ready;
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
    static const bool skip_host_checks = getenv("KVX_TEST_SKIP_HOST_CHECKS") != nullptr;
    int64_t nseg = 0, new_blocks = 0, tokens = 0, full_tokens = 0;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t r = req[i];
        if (r < 0 || r >= t->max_requests) return fail(KVX_EINVAL, "req out of range");
        if (i > 0 && req[i - 1] >= r) return fail(KVX_EINVAL, "wave requests must be strictly ascending");
        if (hi[i] <= lo[i]) continue;
        const int64_t s = t->synced_hi[(size_t)r];
        if (lo[i] < 0 || lo[i] > s) return fail(KVX_EINVAL, "wave interval leaves a gap (lo > synced)");
        if (cdiv64(hi[i], B) > t->max_blocks) return fail(KVX_ENOSPC, "request exceeds max_blocks");
        // (a device-resident source table has no host mirror: the plan kernel checks it)
        const int32_t* srow = t->src_bt.empty() ? nullptr : t->src_bt.data() + (size_t)r * (size_t)t->max_blocks;
        if (srow && !skip_host_checks)  // test hook: lets tests/test_gpu_edges.py reach the device check
            for (int64_t b = lo[i] / B; b < cdiv64(hi[i], B); ++b)
                if (srow[b] < 0) return fail(KVX_EINVAL, "wave reads a source block the source table does not back");
        new_blocks += std::max<int64_t>(0, cdiv64(hi[i], B) - cdiv64(s, B));
        nseg += cdiv64(hi[i], B) - lo[i] / B;
        tokens += hi[i] - lo[i];
        full_tokens += std::max<int64_t>(0, hi[i] / B - cdiv64(lo[i], B)) * B;  // tokens in whole blocks
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
    // The plan kernel reads the entries straight from the pinned (UVA-mapped)
    // staging slot: no separate H2D copy on the stream.  The slot is free
    // again once the plan kernel has run.
    if (t->bm && new_blocks > 0) KVX_CUDA(bm_order_before(t->bm, t->stream));
    const int32_t* h_req = reinterpret_cast<const int32_t*>(h);
    const int64_t* h_lo = reinterpret_cast<const int64_t*>(h + off_lo);
    const int64_t* h_hi = reinterpret_cast<const int64_t*>(h + off_hi);
    kvx::kvx_plan_kernel<<<1, kvx::kPlanThreads, 0, t->stream>>>(
        h_req, h_lo, h_hi, n, t->d_src_bt, t->d_dst_bt, t->d_synced_hi, t->max_blocks,
        t->g.block_tokens, t->bm ? t->bm->top : t->alloc, t->bm ? t->bm->d_stack : nullptr, t->d_segs,
        t->src_cap, t->dst_num_blocks, t->d_err);
    KVX_LAUNCHED();
    KVX_CUDA(cudaEventRecord(t->h_wave_free[slot], t->stream));
    t->last_plan_slot = slot;  // this event now marks the table / synced marks as final
    t->handoff_since_plan = false;
    if (t->bm && new_blocks > 0) KVX_CUDA(bm_order_after(t->bm, t->stream));
    if (t->n_local_layers > 0) {
        const int64_t units = nseg * t->n_local_layers;
        int64_t full = (int64_t)t->num_sms * t->move_ctas_per_sm;
        if (t->max_ctas > 0) full = std::min<int64_t>(full, t->max_ctas);  // sharing HBM with serving
        const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(units, full));
        // Timing: the bulk mover times itself (%globaltimer slots; timing events
        // around it cost ~7 us of stall, profiles/r02m_ab_tight.jsonl); the other
        // movers get an event pair.
        const bool bulk_path = !t->transpose && t->use_bulk && (!t->has_peer_dst || t->peer_bulk);
        kvx_transition::MoveRec rec;
        if (bulk_path && t->d_timer && t->n_timers < kvx_transition::kTimerSlots) {
            rec.timer = t->n_timers++;
        } else {
            KVX_CUDA(kvx::Arena::of(t->device).event(&rec.a, true));
            KVX_CUDA(kvx::Arena::of(t->device).event(&rec.b, true));
            KVX_CUDA(cudaEventRecord(rec.a, t->stream));
        }
        t->move_rec.push_back(rec);
        t->move_bytes.push_back(2ull * (uint64_t)tokens * 2ull * token_bytes(t->g) *
                                (uint64_t)t->n_local_layers);
        // A wave is slab-sized when most of its bytes sit in whole blocks
        // (each one contiguous run of 2 * block_tokens * token_bytes), else
        // token-granular.  (Round 1 used the average run >= 64 KiB, which put
        // the 70B-GQA slab waves -- 64 KiB blocks, partial tails pulling the
        // average to 65,015 B -- on the token ring.)
        const bool slab = 2 * full_tokens >= tokens;
        if (t->transpose && t->tmap_t2h >= 0 && full_tokens > 0) {
            // whole blocks: the TMA transposer; partial blocks: the row mover beside it
            // on the side stream (joined before the wave's end event)
            const uint32_t head_plane = (uint32_t)(t->g.block_tokens * t->g.head_dim * t->g.elem_bytes);
            // 128 CTAs: 0.957-0.969 of the copy peak against 0.946-0.954 on 96 (112 and
            // 136 slower still) on two boxes (profiles/r02am_tmap_grid_sweep*.jsonl)
            int64_t tgrid = std::min<int64_t>(units, 128);
            if (const char* tg = getenv("KVX_TMAP_GRID")) tgrid = std::max<int64_t>(1, atoll(tg));
            if (t->max_ctas > 0) tgrid = std::min<int64_t>(tgrid, t->max_ctas);
            kvx::kvx_tmap_kernel<kTmapStages, kTmapLag><<<(unsigned)std::max<int64_t>(1, tgrid), 32,
                                                          kTmapStages * (size_t)t->tmap_hc * head_plane, t->stream>>>(
                t->d_segs, (int32_t)nseg, t->d_layers, t->n_local_layers, t->d_maps, t->g.num_kv_heads, t->tmap_hc,
                head_plane, t->g.block_tokens, t->tmap_t2h);
            if (full_tokens < tokens) {
                KVX_LAUNCHED();
                cudaStream_t ts = t->max_ctas > 0 ? t->stream : t->side;
                if (ts == t->side) KVX_CUDA(cudaStreamWaitEvent(t->side, t->h_wave_free[slot], 0));
                kvx::kvx_move_any_kernel<<<grid, kvx::kMoveThreads, 0, ts>>>(
                    t->d_segs, (int32_t)nseg, t->d_layers, t->n_local_layers, t->g.num_kv_heads,
                    (uint32_t)(t->g.head_dim * t->g.elem_bytes), t->g.block_tokens, 2, t->has_peer_dst ? 1 : 0);
                if (ts == t->side) {
                    KVX_CUDA(cudaEventRecord(t->ev_join, t->side));
                    KVX_CUDA(cudaStreamWaitEvent(t->stream, t->ev_join, 0));
                }
            }
        } else if (t->transpose) {  // token-major <-> head-major pools: per-(token, head) rows
            kvx::kvx_move_any_kernel<<<grid, kvx::kMoveThreads, 0, t->stream>>>(
                t->d_segs, (int32_t)nseg, t->d_layers, t->n_local_layers, t->g.num_kv_heads,
                (uint32_t)(t->g.head_dim * t->g.elem_bytes), t->g.block_tokens, 0, t->has_peer_dst ? 1 : 0);
        } else if (t->use_bulk && (!t->has_peer_dst || t->peer_bulk)) {
            const int vi = slab ? t->bulk_variant_slab : t->bulk_variant_tok;
            const BulkVariant& bv = kBulkVariants[vi];
            // Grid: measured on B200 across boxes (profiles/grid_cross_box/): 96
            // one-CTA-per-SM streams are the best HBM-bound grid on every chip tried
            // (5.02-5.07 ms for C3 wave 0); 128 ranged 5.02-5.40 and all 148 SMs
            // 5.26-5.30, depending on the chip.  Mixed waves give the peer layers their
            // own CTAs and the local layers the rest: NVLink pushes saturate with
            // ~16-32 CTAs, pulls (TMA loads from the peer) want ~64
            // (profiles/r01_nvlink_split.jsonl, r01_movers_n2.jsonl).
            // Token-granular waves (delta / final: runs of a few KiB) want every SM,
            // two small-ring CTAs on each: the 4 x 16 KiB ring on 296 CTAs is at or
            // within 2 us of the best of 40 (ring, grid) pairs on four boxes
            // (profiles/r02*_wave_sweep_tok*; KVX_BULK_GRID_TOK overrides).
            constexpr int64_t kLocalGrid = 96, kLocalGridTok = 296, kPushCtas = 32, kPullCtas = 64;
            const char* gt = getenv("KVX_BULK_GRID_TOK");
            const int64_t grid_tok = gt ? std::max<int64_t>(1, atoll(gt)) : kLocalGridTok;
            const int64_t local_grid = slab ? kLocalGrid : grid_tok;
            int32_t peer_ctas = (int32_t)(t->n_pull_layers > 0 ? kPullCtas : kPushCtas);
            if (const char* pc = getenv("KVX_PEER_CTAS")) peer_ctas = std::max(0, atoi(pc));
            int64_t full_b = std::min<int64_t>((int64_t)t->num_sms * t->bulk_ctas[vi], local_grid);
            if (t->n_peer_layers > 0 && t->n_peer_layers < t->n_local_layers)
                full_b = std::min<int64_t>((int64_t)t->num_sms * t->bulk_ctas[vi], local_grid + peer_ctas);
            if (const char* cap = getenv("KVX_BULK_GRID"))
                full_b = std::max<int64_t>(1, std::min<int64_t>((int64_t)t->num_sms * t->bulk_ctas[vi], atoll(cap)));
            if (t->max_ctas > 0) full_b = std::min<int64_t>(full_b, t->max_ctas);
            const unsigned grid_b = (unsigned)std::max<int64_t>(1, std::min<int64_t>(units, full_b));
            // programmatic dependent launch: the mover's launch overlaps the
            // plan kernel; it waits (griddepcontrol.wait) for its segments
            cudaLaunchAttribute attr{};
            attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr.val.programmaticStreamSerializationAllowed = 1;
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(grid_b);
            cfg.blockDim = dim3(kvx::kBulkThreads);
            cfg.dynamicSmemBytes = (size_t)bv.stages * bv.chunk;
            cfg.stream = t->stream;
            cfg.attrs = &attr;
            cfg.numAttrs = 1;
            KVX_CUDA(cudaLaunchKernelEx(&cfg, bv.fn, (const kvx::Seg*)t->d_segs, (int32_t)nseg,
                                        (const kvx::LayerPtr*)t->d_layers, t->n_local_layers,
                                        block_bytes(t->g), token_bytes(t->g), t->g.block_tokens,
                                        t->n_peer_layers, peer_ctas,
                                        rec.timer >= 0 ? t->d_timer + rec.timer : nullptr,
                                        rec.timer >= 0 ? t->d_timer + kvx_transition::kTimerSlots + rec.timer : nullptr));
            if (t->head_tails && t->max_ctas > 0) {
                // capped wave (HBM shared with serving): the tail mover runs after the
                // bulk mover on the same stream, so the wave never holds more than
                // max_ctas CTAs at once
                KVX_LAUNCHED();
                kvx::kvx_move_any_kernel<<<grid, kvx::kMoveThreads, 0, t->stream>>>(
                    t->d_segs, (int32_t)nseg, t->d_layers, t->n_local_layers, t->g.num_kv_heads,
                    (uint32_t)(t->g.head_dim * t->g.elem_bytes), t->g.block_tokens, 1, t->has_peer_dst ? 1 : 0);
            } else if (t->head_tails) {
                // head-major partial blocks (the bulk mover skips them): the row mover on a
                // side stream forked after the plan kernel, so it runs beside the bulk
                // mover (which holds only ~96 SMs) and joins before the wave's end event
                KVX_LAUNCHED();
                KVX_CUDA(cudaStreamWaitEvent(t->side, t->h_wave_free[slot], 0));
                kvx::kvx_move_any_kernel<<<grid, kvx::kMoveThreads, 0, t->side>>>(
                    t->d_segs, (int32_t)nseg, t->d_layers, t->n_local_layers, t->g.num_kv_heads,
                    (uint32_t)(t->g.head_dim * t->g.elem_bytes), t->g.block_tokens, 1, t->has_peer_dst ? 1 : 0);
                KVX_CUDA(cudaEventRecord(t->ev_join, t->side));
                KVX_CUDA(cudaStreamWaitEvent(t->stream, t->ev_join, 0));
            }
        } else if (t->lsu256 && token_bytes(t->g) % 32 == 0) {
            kvx::kvx_move256_kernel<<<grid, kvx::kMoveThreads, 0, t->stream>>>(
                t->d_segs, (int32_t)nseg, t->d_layers, t->n_local_layers, block_bytes(t->g),
                token_bytes(t->g), t->g.block_tokens, t->has_peer_dst ? 1 : 0);
        } else {
            kvx::kvx_move_kernel<<<grid, kvx::kMoveThreads, 0, t->stream>>>(
                t->d_segs, (int32_t)nseg, t->d_layers, t->n_local_layers, block_bytes(t->g),
                token_bytes(t->g), t->g.block_tokens, t->has_peer_dst ? 1 : 0);
        }
        KVX_LAUNCHED();
        if (rec.b) KVX_CUDA(cudaEventRecord(rec.b, t->stream));
    }
    KVX_CUDA(cudaEventRecord(t->ev_end, t->stream));
    t->last_ev = t->ev_end;
    // Commit the mirror only once every launch was accepted.
    for (int32_t i = 0; i < n; ++i)
        if (hi[i] > t->synced_hi[(size_t)req[i]]) t->synced_hi[(size_t)req[i]] = hi[i];
    t->alloc += (int32_t)new_blocks;
    if (t->bm) t->bm->top -= (int32_t)new_blocks;
    t->bytes_moved += (uint64_t)tokens * 2ull * token_bytes(t->g) * (uint64_t)t->n_local_layers;
    t->bytes_all_layers += (uint64_t)tokens * 2ull * token_bytes(t->g) * (uint64_t)t->g.num_layers;
    return KVX_OK;
}

int kvx_src_rows(kvx_transition* t, uint64_t epoch, int32_t n, const int32_t* req, const int32_t* rows) {
    if (!t) return fail(KVX_EINVAL, "transition is null");
    if (epoch != t->epoch) return fail(KVX_ESTALE, "stale epoch");
    if (t->state != kvx_transition::kActive) return fail(KVX_ESTATE, "transition is not active");
    if (n < 0 || n > t->max_requests || (n > 0 && (!req || !rows))) return fail(KVX_EINVAL, "bad row arrays");
    if (n == 0) return KVX_OK;
    const size_t mb = (size_t)t->max_blocks;
    for (int32_t i = 0; i < n; ++i) {
        if (req[i] < 0 || req[i] >= t->max_requests) return fail(KVX_EINVAL, "req out of range");
        for (size_t b = 0; b < mb; ++b) {
            const int32_t v = rows[(size_t)i * mb + b];
            if (v >= t->src_cap) return fail(KVX_EINVAL, "src_block_table id beyond an old pool");
            if (!t->src_bt.empty()) {  // host mirror (host-table grants): blocks already set stay put
                const int32_t old = t->src_bt[(size_t)req[i] * mb + b];
                if (old >= 0 && v != old)
                    return fail(KVX_EINVAL, "a source block an earlier wave may have read was remapped");
            }
        }
    }
    DeviceGuard dg(t->device);
    kvx::Arena& A = kvx::Arena::of(t->device);
    const size_t bytes = sizeof(int32_t) * ((size_t)n + (size_t)n * mb);
    if (!t->rows_free) KVX_CUDA(A.event(&t->rows_free, false));
    KVX_CUDA(cudaEventSynchronize(t->rows_free));  // the previous update's staging was consumed
    if (bytes > t->h_rows_bytes) {
        A.host_free(t->h_rows, t->h_rows_bytes);
        t->h_rows = nullptr;
        const size_t cap = kvx::size_class(bytes);
        KVX_CUDA(A.host_alloc((void**)&t->h_rows, cap));
        t->h_rows_bytes = cap;
    }
    std::memcpy(t->h_rows, req, sizeof(int32_t) * (size_t)n);
    std::memcpy(t->h_rows + n, rows, sizeof(int32_t) * (size_t)n * mb);
    kvx::kvx_rows_kernel<<<(unsigned)std::min<int32_t>(n, 1024), 128, 0, t->stream>>>(
        t->h_rows, t->h_rows + n, n, t->max_blocks, t->d_src_bt);
    KVX_LAUNCHED();
    KVX_CUDA(cudaEventRecord(t->rows_free, t->stream));
    t->last_ev = t->rows_free;
    if (!t->src_bt.empty())
        for (int32_t i = 0; i < n; ++i)
            std::memcpy(t->src_bt.data() + (size_t)req[i] * mb, rows + (size_t)i * mb, sizeof(int32_t) * mb);
    return KVX_OK;
}

int kvx_wait(kvx_transition* t, uint64_t epoch, double* measured_ms) {
    if (!t) return fail(KVX_EINVAL, "transition is null");
    if (epoch != t->epoch) return fail(KVX_ESTALE, "stale epoch");
    DeviceGuard dg(t->device);
    KVX_CUDA(cudaStreamSynchronize(t->stream));
    int32_t err = 0;
    err = *reinterpret_cast<volatile int32_t*>(t->d_err);  // zero-copy word; the stream has drained
    if (err) return fail(KVX_ECUDA, "device bounds check failed: a wave referenced a block outside its pool");
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
    if (t->bm && (int64_t)t->bm->top + nb_free > t->bm->capacity)
        return fail(KVX_EINVAL, "block manager overflow: the freed blocks exceed its capacity (double free?)");
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
    }
    // The commit kernel reads the live set from the pinned (UVA-mapped)
    // staging slot and writes its results straight into the pinned landing
    // zone h_commit = [int64 x4 | row_ptr | blocks | free]: no copies on the
    // stream.  A device copy of the free list feeds the block-manager push.
    // The commit kernel reads only the block table, the synced marks and the
    // plan error word -- final once the last plan kernel ran -- not the KV bytes:
    // it runs on the side stream beside the last wave's mover, and the commit
    // event below joins both (the stall is plan + max(mover, commit)).
    // (not after a handoff: there the fork/join cost more than they hid, same-box A/B
    // profiles/r01_ab_stall.txt)
    cudaStream_t cs = t->stream;
    if (t->last_plan_slot >= 0 && t->side && !t->handoff_since_plan) {
        KVX_CUDA(cudaStreamWaitEvent(t->side, t->h_wave_free[t->last_plan_slot], 0));
        cs = t->side;
    }
    int32_t* h32 = reinterpret_cast<int32_t*>(t->h_commit + 32);
    kvx::kvx_commit_kernel<<<1, kvx::kCommitThreads, 0, cs>>>(
        reinterpret_cast<const int32_t*>(h), reinterpret_cast<const int64_t*>(h + off_kv), n_live, t->d_dst_bt,
        t->d_synced_hi, t->d_live, t->max_requests, t->max_blocks, t->g.block_tokens, h32, h32 + (n_live + 1),
        h32 + (n_live + 1) + nb_live, reinterpret_cast<int64_t*>(t->h_commit), t->bm ? d_free : nullptr,
        t->d_err);
    KVX_LAUNCHED();
    KVX_CUDA(cudaEventRecord(t->h_wave_free[slot], cs));
    if (cs != t->stream) {
        KVX_CUDA(cudaEventRecord(t->ev_side_commit, cs));
        KVX_CUDA(cudaStreamWaitEvent(t->stream, t->ev_side_commit, 0));
    }
    (void)d_row_ptr;
    (void)d_blocks;
    if (t->bm && nb_free > 0) {  // free-list update: dead rows' blocks back on the stack
        KVX_CUDA(bm_order_before(t->bm, t->stream));
        KVX_CUDA(cudaMemcpyAsync(t->bm->d_stack + t->bm->top, d_free, sizeof(int32_t) * (size_t)nb_free,
                                 cudaMemcpyDeviceToDevice, t->stream));
        KVX_CUDA(bm_order_after(t->bm, t->stream));
        t->bm->top += (int32_t)nb_free;
    }
    KVX_CUDA(cudaEventRecord(t->ev_commit, t->stream));
    t->last_ev = t->ev_commit;
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
    int64_t res[4];
    std::memcpy(res, t->h_commit, sizeof(res));
    if (res[3]) return fail(KVX_ECUDA, "device bounds check failed: a wave referenced a block outside its pool");
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
        if ((int64_t)t->bm->top + nb_all > t->bm->capacity)
            return fail(KVX_EINVAL, "block manager overflow: the taken blocks exceed its capacity");
        if (nb_all > 0) {
            int32_t* d_row_ptr = t->d_commit_i32;
            int32_t* d_free = d_row_ptr + 1;
            kvx::kvx_commit_kernel<<<1, kvx::kCommitThreads, 0, t->stream>>>(
                reinterpret_cast<const int32_t*>(t->d_wave), reinterpret_cast<const int64_t*>(t->d_wave), 0,
                t->d_dst_bt, t->d_synced_hi, t->d_live, t->max_requests, t->max_blocks, t->g.block_tokens,
                d_row_ptr, nullptr, d_free, t->d_commit_out, nullptr);
            KVX_LAUNCHED();
            KVX_CUDA(bm_order_before(t->bm, t->stream));
            KVX_CUDA(cudaMemcpyAsync(t->bm->d_stack + t->bm->top, d_free, sizeof(int32_t) * (size_t)nb_all,
                                     cudaMemcpyDeviceToDevice, t->stream));
            KVX_CUDA(bm_order_after(t->bm, t->stream));
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
    if (t->last_ev)
        cudaEventSynchronize(t->last_ev);  // this handle's work only; later work on a shared stream runs on
    else if (t->stream)
        cudaStreamSynchronize(t->stream);  // (a handle that failed inside kvx_begin)
    kvx::Arena& A = kvx::Arena::of(t->device);
    A.dev_free(t->d_src_bt, t->bt_bytes);
    A.dev_free(t->d_dst_bt, t->bt_bytes);
    A.dev_free(t->d_synced_hi, sizeof(int64_t) * (size_t)t->max_requests);
    A.dev_free(t->d_layers, t->layers_bytes);
    A.dev_free(t->d_maps, t->maps_bytes);
    A.dev_free(t->d_wave, t->wave_bytes);
    A.dev_free(t->d_segs, sizeof(kvx::Seg) * (size_t)t->seg_cap);
    A.dev_free(t->d_live, (size_t)t->max_requests);
    A.dev_free(t->d_commit_i32, sizeof(int32_t) * (size_t)t->commit_i32_cap);
    A.dev_free(t->d_commit_out, 4 * sizeof(int64_t));
    A.host_free(t->d_err, sizeof(int32_t));
    A.host_free(t->h_commit, t->h_commit_bytes);
    A.event_free(t->ev_commit, false);
    for (int s = 0; s < 2; ++s) {
        A.host_free(t->h_wave[s], t->wave_bytes);
        A.event_free(t->h_wave_free[s], false);
    }
    A.event_free(t->ev_ready, false);
    A.event_free(t->ev_begin, true);
    A.event_free(t->ev_end, true);
    A.dev_free(t->d_pieces, sizeof(kvx::Piece) * (size_t)t->piece_cap);
    A.host_free(t->h_pieces, sizeof(kvx::Piece) * (size_t)t->piece_cap);
    A.event_free(t->pieces_free, false);
    A.host_free(t->h_rows, t->h_rows_bytes);
    A.event_free(t->rows_free, false);
    for (auto& rec : t->move_rec) {
        A.event_free(rec.a, true);
        A.event_free(rec.b, true);
    }
    A.dev_free(t->d_timer, sizeof(unsigned long long) * 2 * kvx_transition::kTimerSlots);
    if (t->side) {
        cudaStreamSynchronize(t->side);
        A.stream_free(t->side);
    }
    A.event_free(t->ev_join, false);
    A.event_free(t->ev_side_commit, false);
    if (t->stream && t->own_stream) cudaStreamDestroy(t->stream);
    delete t;
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
    const int32_t n = (int32_t)t->move_rec.size();
    unsigned long long ts[2 * kvx_transition::kTimerSlots];
    if (t->n_timers > 0) {  // the bulk mover's own start / end stamps
        KVX_CUDA(cudaMemcpyAsync(ts, t->d_timer, sizeof(ts), cudaMemcpyDeviceToHost, t->stream));
        KVX_CUDA(cudaStreamSynchronize(t->stream));
    }
    for (int32_t i = 0; i < n && i < cap; ++i) {
        const kvx_transition::MoveRec& r = t->move_rec[(size_t)i];
        double ms = 0.0;
        if (r.timer >= 0) {
            const unsigned long long s = ts[r.timer], e = ts[kvx_transition::kTimerSlots + r.timer];
            ms = e > s && s != ~0ull ? (double)(e - s) * 1e-6 : 0.0;
        } else {
            float f = 0.f;
            KVX_CUDA(cudaEventSynchronize(r.b));
            KVX_CUDA(cudaEventElapsedTime(&f, r.a, r.b));
            ms = f;
        }
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
    // scratch from the arena: cudaMalloc / cudaFree would synchronise the device
    kvx::Arena& A = kvx::Arena::of(t->device);
    int32_t* d_req = nullptr;
    int64_t* d_kv = nullptr;
    unsigned long long* d_bad = nullptr;
    KVX_CUDA(A.dev_alloc((void**)&d_req, sizeof(int32_t) * n));
    KVX_CUDA(A.dev_alloc((void**)&d_kv, sizeof(int64_t) * n));
    KVX_CUDA(A.dev_alloc((void**)&d_bad, sizeof(unsigned long long)));
    KVX_CUDA(cudaMemcpyAsync(d_req, req, sizeof(int32_t) * n, cudaMemcpyHostToDevice, t->stream));
    KVX_CUDA(cudaMemcpyAsync(d_kv, kv, sizeof(int64_t) * n, cudaMemcpyHostToDevice, t->stream));
    KVX_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), t->stream));
    std::vector<char*> lay;  // every local new pool's layer bases, back to back
    for (const kvx_pool* p : t->new_pools)
        if (p && !p->imported && p->device == t->device) lay.insert(lay.end(), p->layer_base.begin(), p->layer_base.end());
    char** d_lay = nullptr;
    const size_t lay_bytes = sizeof(char*) * std::max<size_t>(1, lay.size());
    KVX_CUDA(A.dev_alloc((void**)&d_lay, lay_bytes));
    if (!lay.empty())
        KVX_CUDA(cudaMemcpyAsync(d_lay, lay.data(), sizeof(char*) * lay.size(), cudaMemcpyHostToDevice, t->stream));
    dim3 grid((unsigned)n, (unsigned)std::min<int64_t>(65535, cdiv64(max_tok, t->g.block_tokens)));
    size_t at = 0;
    for (size_t k = 0; k < t->new_pools.size(); ++k) {
        const kvx_pool* p = t->new_pools[k];
        if (!p || p->imported || p->device != t->device) continue;  // the owning rank / device verifies it
        kvx::kvx_verify_kernel<<<grid, 256, 0, t->stream>>>(
            pool_addr(p, d_lay + at), stage_begin(t->new_b, (int)k), p->num_layers, d_req, d_kv,
            t->d_dst_bt, t->max_blocks, t->g.block_tokens, token_bytes(t->g), seed, d_bad);
        KVX_LAUNCHED();
        at += p->layer_base.size();
    }
    unsigned long long bad = 0;
    KVX_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, t->stream));
    KVX_CUDA(cudaStreamSynchronize(t->stream));
    A.dev_free(d_req, sizeof(int32_t) * n);
    A.dev_free(d_kv, sizeof(int64_t) * n);
    A.dev_free(d_bad, sizeof(unsigned long long));
    A.dev_free(d_lay, lay_bytes);
    *mismatched_words = (int64_t)bad;
    return KVX_OK;
}


}  // extern "C"
