/*
 * kvx.h -- C-ABI of the B200-native inflight-refactor KV transition.
 *
 * Drop-in data plane for FlexPipe's pipeline-refactoring cache transition
 * (reference: /root/reference/proj, "pipesim").  The reference engine keeps
 * its control plane -- which tokens move in which snapshot / delta / final
 * wave, the barrier, commit and abort -- and calls this library at exactly
 * the points where it charges simulated KV movement today:
 *
 *   kvx_begin / kvx_wave   engine.cpp:633-647  begin_refactor, wave 0
 *   kvx_wave               engine.cpp:665-674  delta waves
 *   kvx_wave               engine.cpp:680-687  final post-barrier wave
 *   kvx_wait               engine.cpp:651-662  KvSyncComplete (wave done)
 *   kvx_commit             engine.cpp:697-713  final apply + Eq. 10 check
 *   kvx_abort              engine.cpp:759-772  abort_refactor (revocation)
 *   kvx_destroy            engine.cpp:747-750  ctx reset after commit
 *
 * The kvx_ctl_* entry points additionally restate the reference's
 * RefactorCtx state machine (engine.hpp:149-158) on the library side, so a
 * caller that does not keep its own synced/target maps can drive a whole
 * transition with live (request, kv_tokens) snapshots only.
 *
 * Conventions:
 *   - every function returns an int status (KVX_OK == 0) and never throws;
 *     kvx_last_error() returns a thread-local message for the last failure;
 *   - caller arrays are copied before return; the handle owns device memory
 *     and one CUDA stream; kvx_wait / kvx_commit are the only host syncs;
 *   - calls on one handle are single-threaded (the engine is);
 *   - results are deterministic: destination block ids are a pure function
 *     of the wave inputs;
 *   - a destination overflow returns KVX_ENOSPC, which the engine maps to a
 *     refactor hold (engine.cpp:563,592-593), not to an error;
 *   - an epoch mismatch returns KVX_ESTALE, the analogue of the reference's
 *     stale-event drop (engine.cpp:654,693).
 *
 * HBM layout of one stage pool (per physical GPU):
 *     pool[layer_local][block][kv][token_in_block][kv_head][head_dim]
 * so one (layer, block) slab of K and V is 2 * block_tokens * token_bytes
 * contiguous bytes (320 KiB for Llama-2-13B, 64 KiB for 70B GQA).
 */
#ifndef KVX_H
#define KVX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVX_ABI_VERSION 4  /* 2: kvx_transition_desc.layer_pull; 3: .max_ctas;
                              4: .src_block_table_dev, kvx_bm_*_async, kvx_stage_kv_bytes,
                                 kvx_src_rows */

#define KVX_OK 0
#define KVX_EINVAL (-1)  /* bad argument (null, out of range, unsorted wave) */
#define KVX_ESTALE (-2)  /* epoch mismatch: event of an aborted/older transition */
#define KVX_ENOSPC (-3)  /* destination pool or block table full -> refactor hold */
#define KVX_ECUDA (-4)   /* CUDA runtime / driver failure */
#define KVX_ESTATE (-5)  /* call out of order (wave after commit, double commit) */

#define KVX_IPC_HANDLE_BYTES 64

const char* kvx_last_error(void);
int kvx_abi_version(void);
/* Kernels this library launched in this process (evidence for bench.py). */
uint64_t kvx_launch_count(void);
int kvx_device_count(int32_t* out);
/* Loads every kvx kernel on `device` now.  CUDA lazy loading would load a
 * kernel at its first launch, and a load waits for the work running on the
 * device, so the first refactor would stall behind the serving kernels.
 * Pool / block-manager / transition creation call this implicitly (once per
 * device); a server may call it at start-up. */
int kvx_preload(int32_t device);

/* Model geometry.  token_bytes = num_kv_heads * head_dim * elem_bytes must
 * be a multiple of 16 (vectorised 16-byte moves).  Replaces the scalar
 * ExecModelParams::kv_bytes_per_token (modelgraph.hpp:115), which equals
 * 2 * num_layers * token_bytes. */
typedef struct kvx_geometry {
    int32_t num_layers;   /* ops of the chain, one op per decoder layer */
    int32_t num_kv_heads;
    int32_t head_dim;
    int32_t elem_bytes;   /* 2: fp16 / bf16 */
    int32_t block_tokens; /* paged-KV block size, 16 */
} kvx_geometry;

/* ------------------------------------------------------------------ pools
 * One paged KV pool = the KV of one pipeline stage (a contiguous layer range)
 * on one physical GPU.  Stage k of a plan covers layers [b[k-1], b[k])
 * (PartitionPlan::boundaries, modelgraph.hpp:45; stage_loads engine.cpp:115). */
typedef struct kvx_pool kvx_pool;

int kvx_pool_create(int32_t device, const kvx_geometry* g, int32_t num_layers,
                    int32_t num_blocks, kvx_pool** out);
/* A pool over caller-owned device memory (e.g. the serving engine's KV cache
 * tensor): `ptr` must hold num_layers * num_blocks * 2 * block_tokens *
 * token_bytes bytes on `device`, 16-byte aligned.  Not freed by destroy. */
int kvx_pool_wrap(int32_t device, void* ptr, uint64_t bytes, const kvx_geometry* g,
                  int32_t num_layers, int32_t num_blocks, kvx_pool** out);
/* CUDA IPC handle of a local pool, for a peer process on the same node. */
int kvx_pool_export(const kvx_pool* p, uint8_t handle[KVX_IPC_HANDLE_BYTES]);
/* Maps a peer's pool into `device`'s address space (NVLink P2P). */
int kvx_pool_import(int32_t device, const uint8_t handle[KVX_IPC_HANDLE_BYTES],
                    const kvx_geometry* g, int32_t num_layers, int32_t num_blocks,
                    kvx_pool** out);

/* Per-layer KV layouts.  A transition reads and writes each pool in its own
 * layout, so a refactor can also convert the cache between serving backends.
 *   KVX_LAYOUT_BLOCKS    layer = [num_blocks][2][block_tokens][H][D]: K and V
 *                        rows of a block side by side (FlashInfer NHD paged
 *                        cache; the default of every call above)
 *   KVX_LAYOUT_KV_PLANES layer = [2][num_blocks][block_tokens][H][D]: a K plane
 *                        and a V plane (FlashAttention paged cache)
 *   KVX_LAYOUT_HEADS     layer = [num_blocks][2][H][block_tokens][D]: head-major
 *                        blocks (FlashInfer HND, which vLLM's FlashInfer backend
 *                        requires on compute capability 10, i.e. B200)
 * Token-major (BLOCKS, KV_PLANES) to token-major and head-major to head-major
 * moves are run copies; a move between the two families transposes each
 * block's (token, head) rows. */
#define KVX_LAYOUT_BLOCKS 0
#define KVX_LAYOUT_KV_PLANES 1
#define KVX_LAYOUT_HEADS 2
/* kvx_pool_create / _import with an explicit per-layer layout (one
 * allocation, layers back to back). */
int kvx_pool_create_layout(int32_t device, const kvx_geometry* g, int32_t num_layers,
                           int32_t num_blocks, int32_t layout, kvx_pool** out);
int kvx_pool_import_layout(int32_t device, const uint8_t handle[KVX_IPC_HANDLE_BYTES],
                           const kvx_geometry* g, int32_t num_layers, int32_t num_blocks,
                           int32_t layout, kvx_pool** out);
/* A pool over one caller-owned allocation PER LAYER, as serving engines keep
 * their caches (e.g. one [2, num_blocks, block, H, D] tensor per layer):
 * layer_ptrs[l] holds >= num_blocks * 2 * block_tokens * token_bytes bytes
 * (layer_bytes), 16-byte aligned, on `device`.  Not freed by destroy; not
 * readable through kvx_pool_read / _write (no single allocation), not
 * exportable. */
int kvx_pool_wrap_layers(int32_t device, int32_t num_layers, void* const* layer_ptrs,
                         uint64_t layer_bytes, const kvx_geometry* g, int32_t num_blocks,
                         int32_t layout, kvx_pool** out);
int kvx_pool_layout(const kvx_pool* p, int32_t* layout);
int kvx_pool_info(const kvx_pool* p, void** dptr, uint64_t* bytes, int32_t* device,
                  int32_t* imported);
int kvx_pool_destroy(kvx_pool* p);
/* Synchronous helpers for tests and the bench (not on the transition path). */
int kvx_pool_zero(kvx_pool* p);
int kvx_pool_read(const kvx_pool* p, uint64_t offset, uint64_t bytes, void* host);
int kvx_pool_write(kvx_pool* p, uint64_t offset, uint64_t bytes, const void* host);
/* Writes the deterministic synthetic KV pattern for
 * tokens [0, tokens[i]) of requests req[i] into the pool, which holds model
 * layers [first_layer, first_layer + num_layers), through the block table
 * bt[req * max_blocks + logical_block] (host array). */
int kvx_pool_fill_pattern(kvx_pool* p, uint64_t seed, int32_t first_layer, int32_t n,
                          const int32_t* req, const int64_t* tokens, const int32_t* bt,
                          int32_t max_requests, int32_t max_blocks);

/* ---------------------------------------------------------- block manager
 * Device-resident free list of one pool set (all stages of a plan share block
 * ids): a stack of free block ids in HBM whose top is mirrored on the host,
 * so capacity decisions are synchronous and deterministic.  A fresh or reset
 * manager pops 0, 1, 2, ... (identical to the bump rule); freed blocks are
 * pushed back and reused LIFO.  A transition given dst_blockmgr pops its new
 * blocks from it (plan kernel) and, at commit, pushes the blocks of requests
 * that finished meanwhile; an abort pushes every block it took.  The serving
 * pipeline uses pop/push for its own appends and releases.  Replaces the
 * reference's unmodelled KV memory (only parameter bytes are
 * bound, cluster.cpp:75-96). */
typedef struct kvx_blockmgr kvx_blockmgr;
int kvx_bm_create(int32_t device, int32_t capacity, kvx_blockmgr** out);
int kvx_bm_reset(kvx_blockmgr* bm);
int kvx_bm_free_count(const kvx_blockmgr* bm, int32_t* n);
int kvx_bm_pop(kvx_blockmgr* bm, int32_t n, int32_t* ids_out);   /* host out, LIFO order */
int kvx_bm_push(kvx_blockmgr* bm, int32_t n, const int32_t* ids);
int kvx_bm_snapshot(const kvx_blockmgr* bm, int32_t* stack_out, int32_t* top_out);
/* Serving-side, per decode step: the same pop / push on the caller's stream
 * with DEVICE id arrays -- stream-ordered behind the manager's previous stack
 * op, no host synchronisation (the free count is mirrored on the host, so
 * KVX_ENOSPC / capacity errors are still decided synchronously).
 * dev_ids_out[i] = the i-th pop (LIFO, as kvx_bm_pop).  A pushed id outside
 * [0, capacity) is dropped on the device and reported (KVX_EINVAL) by the
 * manager's next call.  (The host-array calls above wait only for the
 * manager's own stream, never for the device.) */
int kvx_bm_pop_async(kvx_blockmgr* bm, int32_t n, int32_t* dev_ids_out, void* stream);
int kvx_bm_push_async(kvx_blockmgr* bm, int32_t n, const int32_t* dev_ids, void* stream);
int kvx_bm_destroy(kvx_blockmgr* bm);

/* The serving pipeline's decode appends, as test / bench emulation: the
 * payload for tokens [from[i], to[i]) of each request, stream-ordered on
 * `stream` (NULL = legacy default), so it can run concurrently with a wave
 * reading the same pool (KV is append-only, engine.cpp:494-499). */
int kvx_pool_append_pattern(kvx_pool* p, void* stream, uint64_t seed, int32_t first_layer, int32_t n,
                            const int32_t* req, const int64_t* from, const int64_t* to, const int32_t* bt,
                            int32_t max_requests, int32_t max_blocks);

/* ------------------------------------------------------------- transition */
typedef struct kvx_plan {
    int32_t num_stages;           /* K */
    const int32_t* boundaries;    /* K-1 cut indices */
    kvx_pool* const* pools;       /* K pools; NULL for a remote old stage */
} kvx_plan;

typedef struct kvx_transition_desc {
    kvx_geometry geometry;
    kvx_plan old_plan;            /* source: the serving pipeline */
    kvx_plan new_plan;            /* destination: every pool required (local or imported) */
    int32_t device;               /* local GPU: moves every layer whose old pool lives here */
    int32_t max_requests;         /* request ids are in [0, max_requests) */
    int32_t max_blocks;           /* logical blocks per request */
    int32_t dst_num_blocks;       /* block capacity of every new-stage pool */
    const int32_t* src_block_table; /* host [max_requests * max_blocks], the old pipeline's */
    uint64_t epoch;               /* InstanceRt::epoch after ++ (engine.cpp:634) */
    int32_t max_sync_rounds;      /* EngineConfig::max_sync_rounds (engine.hpp:75; default 8), kvx_ctl_*;
                                     taken as given: 0 = no delta wave, wave 0 then the barrier */
    double kv_bytes_per_token;    /* accounting of kvx_ctl_* (engine.cpp:644); 0 = from geometry */
    void* stream;                 /* cudaStream_t to run on (not owned); NULL = a private stream */
    void* dst_blockmgr;           /* kvx_blockmgr* of the new pools; NULL = bump rule from id 0 */
    int32_t pull;                 /* 0: move the layers whose OLD pool is local (push to peers);
                                     1: move the layers whose NEW pool is local, reading peers'
                                     (imported) old pools over NVLink (pull) */
    const uint8_t* layer_pull;    /* optional, per layer (overrides `pull`): 1 = the GPU holding
                                     the layer's NEW pool pulls it, 0 = the GPU holding its OLD
                                     pool pushes it.  Every rank passes the same array.  One-way
                                     NVLink traffic is faster pulled, two-way faster pushed
                                     (DESIGN.md 4); shard.py derives it from the placement.
                                     Layers whose old and new pools are both local always move
                                     here.  NULL = `pull` for every layer. */
    int32_t max_ctas;             /* optional cap on the mover's CTAs per wave (0 = the tuned grid):
                                     waves 0 / delta overlap serving, and fewer CTAs leave serving
                                     more HBM bandwidth */
    const int32_t* src_block_table_dev; /* optional DEVICE copy of the source table (same shape), as
                                     serving engines keep it: when non-NULL it is used instead of
                                     src_block_table (which may then be NULL) -- copied on the
                                     device, no host scan; ids are bounds-checked by the plan
                                     kernel on the device (an out-of-pool id fails kvx_wait /
                                     the commit with KVX_ECUDA, nothing out of range is touched) */
} kvx_transition_desc;

typedef struct kvx_transition kvx_transition;

/* Grants the destination: allocates the transition state on `device`.
 * No bytes move until the first kvx_wave.
 * Replaces: the data-plane side of Engine::begin_refactor once the grant
 * succeeded -- RefactorCtx creation, engine.cpp:633-635 (grant and binding
 * :584-619 stay the engine's).  KVX_ENOSPC maps to a refactor hold
 * (engine.cpp:563,592-593). */
int kvx_begin(const kvx_transition_desc* d, kvx_transition** out);

/* KV bytes each new stage's GPU holds for a grant of dst_num_blocks blocks
 * per layer: out[k] = layers(k) * dst_num_blocks * 2 * block_tokens *
 * token_bytes (pools are dense in every layout).  Host-only, no GPU.  The
 * engine adds out[k] to stage k's binding (engine.cpp:584-619), so a KV
 * shortfall is a refactor hold at allocation time (:592-593) instead of
 * KVX_ENOSPC after the grant.  The reference never accounts KV
 * (cluster.cpp:75-82 charges stage_param_bytes only). */
int kvx_stage_kv_bytes(const kvx_geometry* g, int32_t num_stages, const int32_t* boundaries,
                       int32_t dst_num_blocks, uint64_t* out);

/* Replaces: the simulated sync charge sync_ms = tokens * bpt / kv_bw of
 * wave 0 (engine.cpp:637-647), delta waves (:665-674) and the final wave
 * (:680-687) -- the bytes move instead of being charged.
 * Enqueues one wave: for each entry, tokens [lo[i], hi[i]) of request req[i]
 * across every layer.  req must be strictly ascending (the std::map order of
 * RefactorCtx::sync_target, engine.hpp:153-154); entries with lo == hi are
 * allowed (the reference snapshots zero-delta requests too, engine.cpp:548).
 * Asynchronous: destination blocks are allocated and the slabs moved by
 * device kernels on the handle's stream. */
int kvx_wave(kvx_transition* t, uint64_t epoch, int32_t n, const int32_t* req,
             const int64_t* lo, const int64_t* hi);
/* Serving-side growth of the source block table during a transition: rows
 * req[i] become rows[i * max_blocks .. +max_blocks) (host arrays), stream-
 * ordered before the next wave.  A serving engine appends blocks as decode
 * grows a request, or admits new requests, while the refactor runs
 * (engine.cpp:267,494-499); the grant's table only covers what existed then.
 * Ids must lie in the old pools; a block id already set in the row must not
 * change (an earlier wave may have read it) -- both KVX_EINVAL. */
int kvx_src_rows(kvx_transition* t, uint64_t epoch, int32_t n, const int32_t* req, const int32_t* rows);
/* Blocks until every enqueued wave finished; *measured_ms = device time of
 * the waves since the previous wait (CUDA events on the handle's stream).
 * Replaces: the modelled arrival of KvSyncComplete (engine.cpp:646,651). */
int kvx_wait(kvx_transition* t, uint64_t epoch, double* measured_ms);

typedef struct kvx_commit_result {
    int64_t violations;  /* Eq. 10, engine.cpp:707-713, evaluated on the device */
    int32_t* row_ptr;    /* optional [n_live + 1]: compacted block table (CSR) */
    int32_t* blocks;     /* optional [blocks_cap] */
    int32_t blocks_cap;
    int32_t n_blocks;    /* out */
    int32_t* free_list;  /* optional [free_cap]: blocks of requests no longer live */
    int32_t free_cap;
    int32_t n_free;      /* out */
} kvx_commit_result;

/* Final apply + consistency check + block-table compaction for the live
 * (req, kv_tokens) set, ascending req.  After a successful commit the
 * destination pools with the returned block table are the stage's KV.
 * Replaces: Engine::on_refactor_commit's final apply and Eq. 10 check,
 * engine.cpp:697-713 (violations == the host loop's count). */
int kvx_commit(kvx_transition* t, uint64_t epoch, int32_t n_live, const int32_t* req,
               const int64_t* kv_tokens, kvx_commit_result* out);
/* The same commit split in two: _async enqueues the check + compaction and
 * the copy of its results into pinned memory, bumps the epoch (later waves
 * are stale) and returns without a host sync; _collect waits for it and
 * fills `out`.  Lets the engine resume routing (engine.cpp:747-756) while
 * the commit's bookkeeping is still on the device. */
int kvx_commit_async(kvx_transition* t, uint64_t epoch, int32_t n_live, const int32_t* req,
                     const int64_t* kv_tokens);
int kvx_commit_collect(kvx_transition* t, kvx_commit_result* out);
/* Drops every destination allocation, invalidates the epoch (++epoch,
 * engine.cpp:769).  The source pools were never modified.
 * Replaces: abort_refactor, engine.cpp:759-772. */
int kvx_abort(kvx_transition* t);
/* Frees the handle (after its stream drained).  Replaces: inst.refactor.reset(),
 * engine.cpp:750. */
int kvx_destroy(kvx_transition* t);

/* Introspection: current epoch, and the dense destination block table
 * [max_requests * max_blocks] (-1 = unallocated). */
int kvx_epoch(const kvx_transition* t, uint64_t* epoch);
int kvx_dst_block_table(kvx_transition* t, int32_t* host_out);
/* Raw CUDA stream (cudaStream_t) of the handle, e.g. to record events. */
int kvx_stream(const kvx_transition* t, void** stream);
/* Device time of each move-kernel launch of this handle, in wave order
 * (CUDA events around the launch itself), and the algorithmic bytes it moved
 * (read + written).  Fills min(cap, n) entries; *n_out = n.  Synchronises
 * on the recorded events. */
int kvx_move_timings(const kvx_transition* t, int32_t cap, double* move_ms, uint64_t* rw_bytes,
                     int32_t* n_out);
/* Bytes this handle moved (reads at the source == writes at the destination). */
int kvx_bytes_moved(const kvx_transition* t, uint64_t* bytes);
/* Device-side check of the destination pools this handle can see against
 * the synthetic pattern, tokens [0, kv[i]) of each live request. */
int kvx_verify_pattern(kvx_transition* t, uint64_t seed, int32_t n, const int32_t* req,
                       const int64_t* kv, int64_t* mismatched_words);

/* ------------------------------------------- stage-boundary activation handoff
 * Alternative to the barrier drain (engine.cpp:676-678): the in-flight
 * micro-batches are moved to the new pipeline instead of finishing on the
 * old one.  A batch holding the output of old stage `after_stage` goes to the
 * new stage owning layer old_boundaries[after_stage] and resumes there
 * (same layer range semantics as stage_loads, engine.cpp:115-126); a batch
 * that has not finished any stage (after_stage < 0) is re-dispatched at new
 * stage 0 with no bytes; a batch that finished the LAST old stage
 * (after_stage == K_old - 1) is not in flight any more -- its output is the
 * pipeline's -- and gets no slot (new_stage = -1, bytes 0).  after_stage >=
 * K_old is KVX_EINVAL.  Destination = a caller-provided activation arena
 * per new stage (device pointer, local or peer-mapped); each arena is filled
 * by a bump pointer in batch order, offsets aligned to 256 B.  Slots are
 * computed for every batch (deterministic on every rank); bytes move only
 * for batches whose old stage lives on this handle's GPU.  row_bytes (hidden
 * size x element bytes) must be a multiple of 16, src 16-byte aligned. */
typedef struct kvx_microbatch {
    int64_t batch_id;
    int32_t after_stage;   /* last OLD stage whose output the batch holds; -1 = none */
    int32_t tokens;        /* activation rows */
    const void* src;       /* device pointer on the GPU of old stage after_stage */
} kvx_microbatch;

typedef struct kvx_handoff_slot {
    int64_t batch_id;
    int32_t new_stage;     /* new owner; -1 = finished on the old pipeline, no slot */
    int32_t resume_layer;  /* first layer the new owner runs for this batch */
    uint64_t offset;       /* byte offset in the new stage's activation arena */
    uint64_t bytes;
} kvx_handoff_slot;

int kvx_handoff(kvx_transition* t, uint64_t epoch, uint64_t row_bytes, int32_t n,
                const kvx_microbatch* mb, void* const* arenas, const uint64_t* arena_bytes,
                kvx_handoff_slot* slots_out);

/* ------------------------------------------------- stage weight migration
 * The parameters a new stage needs before commit (the reference models them
 * as per-server loads the commit waits on: engine.cpp:621-631,686 and
 * warm_start_latency_ms, cluster.cpp:525-536).  Each stage's weights are one
 * contiguous layer-major buffer of layer_bytes per layer.  For every layer
 * whose old stage buffer is local (old_ptrs[k] non-NULL, on `device`), the
 * layer is copied into the new stage buffer that owns it (local, or a
 * peer-mapped pointer over NVLink) by the bulk copy engine kernel; layers
 * with from_host[l] == 1 are instead loaded from the pinned host cache
 * host_cache + l * layer_bytes (the reference's host tier).  Asynchronous on
 * `stream` (NULL = the legacy default stream); *device_bytes / *host_bytes
 * receive the bytes scheduled. */
int kvx_weights_migrate(int32_t device, void* stream, int32_t num_layers, uint64_t layer_bytes,
                        int32_t old_stages, const int32_t* old_boundaries, void* const* old_ptrs,
                        int32_t new_stages, const int32_t* new_boundaries, void* const* new_ptrs,
                        const void* host_cache, const uint8_t* from_host, uint64_t* device_bytes,
                        uint64_t* host_bytes);

/* ---------------------------------------------------- control-plane mirror
 * RefactorCtx (engine.hpp:149-158) restated over the handle.  live = the
 * (req, kv_tokens) of every live request homed on the instance, ascending
 * req, i.e. what snapshot_sync_targets iterates (engine.cpp:548-556). */
enum {
    KVX_ACT_DELTA = 0,        /* a delta wave was issued (engine.cpp:666-674) */
    KVX_ACT_BARRIER_WAIT = 1, /* barrier set, pipe still draining (engine.cpp:676-678) */
    KVX_ACT_FINAL = 2,        /* final wave issued, commit may follow (engine.cpp:680-687) */
};
typedef struct kvx_ctl_state {
    int32_t rounds;
    int32_t barrier;
    int32_t commit_scheduled;
    int32_t waves;
    double kv_synced_bytes;   /* EngineResult::kv_synced_bytes contribution */
    int64_t last_wave_tokens;
} kvx_ctl_state;

/* Replaces begin_refactor's snapshot + wave 0 + byte accounting,
 * engine.cpp:637-647 (snapshot_sync_targets :548-556).  (n, req, kv) = the
 * live homed requests and their kv_tokens, ascending. */
int kvx_ctl_begin(kvx_transition* t, int32_t n, const int32_t* req, const int64_t* kv,
                  int64_t* tokens_out);
/* Replaces on_kv_sync_complete, engine.cpp:651-688: apply, then a delta wave
 * (kv_tokens_unsynced :534-546, max_sync_rounds), the barrier, or the final
 * wave once inflight_batches == 0 (or at once in handoff mode). */
int kvx_ctl_sync_complete(kvx_transition* t, uint64_t epoch, int32_t n, const int32_t* req,
                          const int64_t* kv, int32_t inflight_batches, int32_t* action_out,
                          int64_t* tokens_out);
/* Replaces on_refactor_commit's apply + Eq. 10, engine.cpp:697-713; the
 * device count must equal the mirror's (else KVX_ECUDA). */
int kvx_ctl_commit(kvx_transition* t, uint64_t epoch, int32_t n, const int32_t* req,
                   const int64_t* kv, kvx_commit_result* out);
int kvx_ctl_commit_async(kvx_transition* t, uint64_t epoch, int32_t n, const int32_t* req,
                         const int64_t* kv);
int kvx_ctl_commit_collect(kvx_transition* t, kvx_commit_result* out);
int kvx_ctl_state_get(const kvx_transition* t, kvx_ctl_state* out);
/* Handoff mode: at the barrier the caller hands the in-flight micro-batches
 * to the new pipeline (kvx_handoff) instead of draining them, so the final
 * wave is issued at once -- the wait on inflight_batches (engine.cpp:678) is
 * dropped and the drain leaves the stall.  Off by default (reference
 * semantics). */
int kvx_ctl_set_handoff(kvx_transition* t, int32_t enable);

#ifdef __cplusplus
}
#endif
#endif /* KVX_H */
