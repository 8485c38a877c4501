/*
 * kvx_oracle.h -- CPU restatement of the inflight-refactor KV transition.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * product (paper_2510_11938_b200/csrc, include/kvx.h).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it; the product never links, calls or falls back to it.
 *
 * Two halves:
 *   1. Control plane (kvo_ctx_*): the reference's RefactorCtx bookkeeping,
 *      restated over dense per-request arrays.  Pinned against the golden
 *      vectors in tests/golden (jsonl), which oracle/extract_waves.cpp pulls
 *      out of the UNMODIFIED reference engine.
 *        /root/reference/proj/src/engine.cpp:534-546  kv_tokens_unsynced
 *        /root/reference/proj/src/engine.cpp:548-556  snapshot_sync_targets
 *        /root/reference/proj/src/engine.cpp:637-647  wave 0 (begin_refactor)
 *        /root/reference/proj/src/engine.cpp:651-688  on_kv_sync_complete
 *        /root/reference/proj/src/engine.cpp:697-713  final apply + Eq. 10 check
 *        /root/reference/proj/src/engine.cpp:759-772  abort_refactor
 *   2. Data plane (kvo_*): paged KV pools, the deterministic destination
 *      block rule, the per-token memcpy executor, commit-time compaction.
 *      The reference moves no bytes (it charges tokens * kv_bytes_per_token,
 *      engine.cpp:644,670,683), so byte-level parity is defined HERE and the
 *      product must match it bit for bit; see DESIGN.md "Parity contract".
 *
 * Layout of one stage pool (HBM layout of the product, restated):
 *     pool[layer_local][block][kv(0=K,1=V)][token_in_block][kv_head][head_dim]
 * i.e. a (layer, block) slab is 2 * block_tokens * token_bytes contiguous bytes
 * and token_bytes = num_kv_heads * head_dim * elem_bytes.
 */
#ifndef KVX_ORACLE_H
#define KVX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kvo_geometry {
    int32_t num_layers;   /* L: ops of the chain, one op per decoder layer */
    int32_t num_kv_heads; /* H_kv */
    int32_t head_dim;     /* D */
    int32_t elem_bytes;   /* 2 for fp16 / bf16 */
    int32_t block_tokens; /* 16 */
} kvo_geometry;

/* ---- synthetic KV payload (identical formula in the CUDA fill/verify) ---- */
uint64_t kvo_mix64(uint64_t z);
uint64_t kvo_token_hash(uint64_t seed, int32_t req, int32_t layer, int32_t kv, int64_t tok);
uint16_t kvo_word(uint64_t token_hash, uint32_t word);

/* stage_of_op (modelgraph.cpp:55-62): stage k covers [b[k-1], b[k]). */
int32_t kvo_stage_of_layer(int32_t num_stages, const int32_t* boundaries, int32_t layer);
/* stage_loads (engine.cpp:115-126): first layer of stage k. */
int32_t kvo_stage_begin(int32_t num_stages, const int32_t* boundaries, int32_t stage);

/* ------------------------------ control plane ----------------------------- */
typedef struct kvo_ctx {
    int32_t max_requests;
    int64_t* synced;      /* [max_requests]; absent == 0 (engine.cpp:540-542) */
    int64_t* target;      /* [max_requests] */
    uint8_t* in_target;   /* [max_requests] membership of sync_target */
    int32_t rounds;
    int32_t barrier;
    int32_t commit_scheduled;
    int32_t max_sync_rounds;
    double kv_bytes_per_token;
    double* kv_synced_bytes; /* caller-owned accumulator (EngineResult) */
} kvo_ctx;

/* snapshot_sync_targets + the lo of each interval.  Writes lo/hi for the n
 * live requests (in the order given; callers pass ascending request ids, the
 * std::map order) and returns the tokens the wave moves. */
int64_t kvo_ctx_snapshot(kvo_ctx* c, int32_t n, const int32_t* req, const int64_t* kv,
                         int64_t* lo_out, int64_t* hi_out);
/* kv_tokens_unsynced over the live set. */
int64_t kvo_ctx_unsynced(const kvo_ctx* c, int32_t n, const int32_t* req, const int64_t* kv);
/* A wave finished: synced = max(synced, target); clear targets (engine.cpp:657-662). */
void kvo_ctx_apply(kvo_ctx* c);
/* Eq. 10 (engine.cpp:704-713). */
int64_t kvo_ctx_violations(const kvo_ctx* c, int32_t n, const int32_t* req, const int64_t* kv);

enum { KVO_ACT_DELTA = 0, KVO_ACT_BARRIER_WAIT = 1, KVO_ACT_FINAL = 2, KVO_ACT_NONE = 3 };
/* Wave 0 of begin_refactor (engine.cpp:637-647). */
int64_t kvo_ctx_begin(kvo_ctx* c, int32_t n, const int32_t* req, const int64_t* kv,
                      int64_t* lo_out, int64_t* hi_out);
/* on_kv_sync_complete (engine.cpp:651-688); *tokens_out = tokens of the wave it issued. */
int32_t kvo_ctx_on_sync_complete(kvo_ctx* c, int32_t n, const int32_t* req, const int64_t* kv,
                                 int32_t inflight_batches, int64_t* lo_out, int64_t* hi_out,
                                 int64_t* tokens_out);

/* ------------------------------- data plane ------------------------------- */
uint64_t kvo_token_bytes(const kvo_geometry* g);
uint64_t kvo_block_bytes(const kvo_geometry* g); /* one (layer, block) slab, K and V */

/* Writes the synthetic pattern for tokens [0, tokens[i]) of each request into
 * the pools of a plan, through a per-request block table
 * bt[req * max_blocks + logical_block].  Used for both source and, in tests,
 * expected destination images. */
void kvo_fill(const kvo_geometry* g, uint64_t seed, int32_t num_stages, const int32_t* boundaries,
              uint8_t* const* pools, int32_t blocks_per_pool, int32_t n, const int32_t* req,
              const int64_t* tokens, const int32_t* bt, int32_t max_blocks);

/* The expected image of ONE layer (model layer `layer`) of a block-layout
 * pool: zero everywhere except tokens [0, tokens[i]) of each request req[i],
 * which hold the payload, placed through bt -- i.e. kvo_fill restricted to
 * one layer on a zeroed buffer.  Given the oracle's destination table and
 * synced high-water marks it is the oracle's destination layer after a
 * transition (rows never written stay zero), so a full-size pool can be
 * compared byte for byte one layer at a time.  layer_buf holds
 * blocks_per_pool * kvo_block_bytes(g) bytes; `threads` pthreads. */
void kvo_fill_layer(const kvo_geometry* g, uint64_t seed, int32_t layer, uint8_t* layer_buf,
                    int32_t blocks_per_pool, int32_t n, const int32_t* req, const int64_t* tokens,
                    const int32_t* bt, int32_t max_blocks, int32_t threads);

typedef struct kvo_dst {
    int32_t max_requests;
    int32_t max_blocks;    /* per request */
    int32_t num_blocks;    /* capacity of every destination pool */
    int32_t next_block;    /* bump pointer of the deterministic block rule */
    int32_t* bt;           /* [max_requests * max_blocks], -1 = unallocated */
    int64_t* synced_hi;    /* [max_requests] high-water mark of copied tokens */
    int32_t* stack;        /* optional block-manager free stack (NULL: bump rule) */
    int32_t top;           /* free ids on the stack; pops take stack[top-1] */
} kvo_dst;

/* Block manager restated: a fresh stack holds capacity-1 ... 0 (pops yield
 * 0, 1, 2, ...); commit pushes the free list in order; abort pushes every
 * allocated block (ascending request, ascending block). */
void kvo_bm_init(int32_t* stack, int32_t capacity);
void kvo_abort(const kvo_geometry* g, kvo_dst* d);

/* Executes one wave: destination block allocation (new blocks in ascending
 * request order, ascending logical block, from the bump pointer; entries
 * must be strictly ascending in req and start at lo <= synced_hi) then a
 * per-token copy of every layer's K and V rows [lo, hi) from the old stage
 * owning the layer to the new stage owning it.  With old_pools or new_pools
 * NULL only the block rule runs (allocation-only replay at full scale).
 * Returns 0, or -1 on an invalid wave or a pool / table overflow. */
int kvo_apply_wave(const kvo_geometry* g, kvo_dst* d, int32_t old_stages,
                   const int32_t* old_boundaries, uint8_t* const* old_pools,
                   int32_t old_blocks, const int32_t* src_bt, int32_t new_stages,
                   const int32_t* new_boundaries, uint8_t* const* new_pools, int32_t n,
                   const int32_t* req, const int64_t* lo, const int64_t* hi);

/* Same wave with run-granular memcpy (whole (layer, block) slabs when a block
 * is fully covered) on `threads` pthreads -- the CPU baseline executor. */
int kvo_apply_wave_mt(const kvo_geometry* g, kvo_dst* d, int32_t old_stages,
                      const int32_t* old_boundaries, uint8_t* const* old_pools,
                      int32_t old_blocks, const int32_t* src_bt, int32_t new_stages,
                      const int32_t* new_boundaries, uint8_t* const* new_pools, int32_t n,
                      const int32_t* req, const int64_t* lo, const int64_t* hi, int32_t threads);

/* Commit: Eq. 10 per live request (synced_hi == kv_tokens), the compacted block table of the live requests (CSR in the given
 * order: row_ptr[n+1], blocks[]) and the free list of every allocated block
 * of a request that is no longer live (ascending request, ascending block).
 * Returns the violation count; *n_blocks / *n_free receive the sizes. */
int64_t kvo_commit(const kvo_geometry* g, kvo_dst* d, int32_t n, const int32_t* req,
                   const int64_t* kv, int32_t* row_ptr, int32_t* blocks, int32_t* n_blocks,
                   int32_t* free_list, int32_t* n_free);

/* Counts 16-bit words of the destination image that differ from the pattern,
 * over tokens [0, kv[i]) of each live request, read through d->bt. */
int64_t kvo_verify(const kvo_geometry* g, uint64_t seed, const kvo_dst* d, int32_t new_stages,
                   const int32_t* new_boundaries, uint8_t* const* new_pools, int32_t n,
                   const int32_t* req, const int64_t* kv);

/* Stage-boundary activation handoff (engine.cpp:449-456 in_transit batches):
 * the activation of a micro-batch that left old stage s is owned after the
 * refactor by the new stage containing layer old_boundary[s]. */
int32_t kvo_activation_owner(int32_t old_stages, const int32_t* old_boundaries,
                             int32_t new_stages, const int32_t* new_boundaries,
                             int32_t from_old_stage);

/* Handoff plan for n in-flight micro-batches (instead of the barrier drain,
 * engine.cpp:676-678).  Batch i holds the output of old stage after[i]
 * (-1: none yet), tokens[i] rows of row_bytes each.  It goes to the new
 * stage owning layer old_boundary[after[i]] and resumes there; batches with
 * after < 0 are re-dispatched at new stage 0, layer 0, with no bytes.  Each
 * new stage's arena is filled by a bump pointer in batch order, offsets
 * aligned to 256 B.  Outputs per batch: new stage, resume layer, offset,
 * bytes.  Returns 0, or -1 if an arena (arena_bytes[k]) would overflow. */
int kvo_handoff_plan(int32_t old_stages, const int32_t* old_boundaries, int32_t new_stages,
                     const int32_t* new_boundaries, uint64_t row_bytes, int32_t n,
                     const int32_t* after, const int32_t* tokens, const uint64_t* arena_bytes,
                     int32_t* new_stage, int32_t* resume_layer, uint64_t* offset, uint64_t* bytes);

/* Stage weight migration: the new stage k needs the parameters of layers
 * [nb[k-1], nb[k]) (stage_loads, engine.cpp:115-126), which the reference
 * loads from host cache or storage before commit (engine.cpp:621-631,686;
 * warm_start_latency_ms, cluster.cpp:525-536).  With layer-major contiguous
 * stage buffers, layer l moves from old stage so(l) at offset
 * (l - begin(so)) * layer_bytes to new stage sn(l) at (l - begin(sn)) *
 * layer_bytes.  Fills per-layer (src_stage, src_off, dst_stage, dst_off). */
void kvo_weights_plan(int32_t num_layers, uint64_t layer_bytes, int32_t old_stages,
                      const int32_t* old_boundaries, int32_t new_stages,
                      const int32_t* new_boundaries, int32_t* src_stage, uint64_t* src_off,
                      int32_t* dst_stage, uint64_t* dst_off);
/* The reference's own parameter-load time for one server's new stages:
 * sum over stages of bytes / (host bw if the range is host-cached, else
 * storage bw) -- warm_start_latency_ms restated (cached[k] = cache_covers). */
double kvo_warm_start_ms(int32_t n, const double* stage_bytes, const uint8_t* cached,
                         double host_bw_bytes_per_ms, double storage_bw_bytes_per_ms);

#ifdef __cplusplus
}
#endif
#endif /* KVX_ORACLE_H */
