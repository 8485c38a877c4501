/*
 * kvx_oracle.c -- CPU restatement of the inflight-refactor KV transition.
 * TEST INFRASTRUCTURE ONLY (see kvx_oracle.h).  Every function cites the
 * reference lines it restates; the data-plane rules are the parity contract
 * of DESIGN.md because the reference itself moves no bytes.
 */
#define _GNU_SOURCE
#include "kvx_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ----------------------------------------------------------------- payload */

uint64_t kvo_mix64(uint64_t z) { /* splitmix64 finaliser */
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t kvo_token_hash(uint64_t seed, int32_t req, int32_t layer, int32_t kv, int64_t tok) {
    uint64_t h = kvo_mix64(seed ^ (uint64_t)(uint32_t)req);
    h = kvo_mix64(h ^ (((uint64_t)(uint32_t)layer << 1) | (uint64_t)(kv & 1)));
    return kvo_mix64(h ^ (uint64_t)tok);
}

uint16_t kvo_word(uint64_t th, uint32_t word) {
    return (uint16_t)(((th + (uint64_t)word * 0x9E3779B97F4A7C15ull) * 0xBF58476D1CE4E5B9ull) >> 48);
}

/* modelgraph.cpp:55-62 */
int32_t kvo_stage_of_layer(int32_t num_stages, const int32_t* b, int32_t layer) {
    int32_t s = 0;
    for (int32_t k = 0; k + 1 < num_stages; ++k) {
        if (layer < b[k]) break;
        ++s;
    }
    return s;
}

/* engine.cpp:115-126 */
int32_t kvo_stage_begin(int32_t num_stages, const int32_t* b, int32_t stage) {
    (void)num_stages;
    return stage == 0 ? 0 : b[stage - 1];
}

/* ----------------------------------------------------------- control plane */

int64_t kvo_ctx_unsynced(const kvo_ctx* c, int32_t n, const int32_t* req, const int64_t* kv) {
    /* engine.cpp:534-546, restricted to the live homed set the caller passes. */
    int64_t total = 0;
    for (int32_t i = 0; i < n; ++i) {
        const int64_t d = kv[i] - c->synced[req[i]];
        total += d > 0 ? d : 0;
    }
    return total;
}

int64_t kvo_ctx_snapshot(kvo_ctx* c, int32_t n, const int32_t* req, const int64_t* kv,
                         int64_t* lo_out, int64_t* hi_out) {
    /* engine.cpp:548-556: sync_target.clear(); target[r] = kv_tokens for every
     * live homed request (zero-delta ones included). */
    memset(c->in_target, 0, (size_t)c->max_requests);
    int64_t tokens = 0;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t r = req[i];
        c->target[r] = kv[i];
        c->in_target[r] = 1;
        if (lo_out) lo_out[i] = c->synced[r];
        if (hi_out) hi_out[i] = kv[i];
        const int64_t d = kv[i] - c->synced[r];
        tokens += d > 0 ? d : 0;
    }
    return tokens;
}

void kvo_ctx_apply(kvo_ctx* c) {
    /* engine.cpp:657-662 (and 697-702 for the final wave). */
    for (int32_t r = 0; r < c->max_requests; ++r) {
        if (!c->in_target[r]) continue;
        if (c->target[r] > c->synced[r]) c->synced[r] = c->target[r];
        c->in_target[r] = 0;
    }
}

int64_t kvo_ctx_violations(const kvo_ctx* c, int32_t n, const int32_t* req, const int64_t* kv) {
    /* engine.cpp:707-713 */
    int64_t v = 0;
    for (int32_t i = 0; i < n; ++i)
        if (c->synced[req[i]] != kv[i]) ++v;
    return v;
}

int64_t kvo_ctx_begin(kvo_ctx* c, int32_t n, const int32_t* req, const int64_t* kv,
                      int64_t* lo_out, int64_t* hi_out) {
    /* engine.cpp:633-647: fresh ctx, snapshot, charge every current token. */
    memset(c->synced, 0, sizeof(int64_t) * (size_t)c->max_requests);
    memset(c->target, 0, sizeof(int64_t) * (size_t)c->max_requests);
    c->rounds = 0;
    c->barrier = 0;
    c->commit_scheduled = 0;
    kvo_ctx_snapshot(c, n, req, kv, lo_out, hi_out);
    int64_t tokens = 0;
    for (int32_t i = 0; i < n; ++i) tokens += kv[i];
    if (c->kv_synced_bytes) *c->kv_synced_bytes += (double)tokens * c->kv_bytes_per_token;
    return tokens;
}

int32_t kvo_ctx_on_sync_complete(kvo_ctx* c, int32_t n, const int32_t* req, const int64_t* kv,
                                 int32_t inflight_batches, int64_t* lo_out, int64_t* hi_out,
                                 int64_t* tokens_out) {
    /* engine.cpp:651-688 */
    if (tokens_out) *tokens_out = 0;
    kvo_ctx_apply(c);
    if (!c->barrier) {
        const int64_t delta = kvo_ctx_unsynced(c, n, req, kv);
        if (delta > 0 && c->rounds < c->max_sync_rounds) {
            ++c->rounds;
            kvo_ctx_snapshot(c, n, req, kv, lo_out, hi_out);
            if (c->kv_synced_bytes) *c->kv_synced_bytes += (double)delta * c->kv_bytes_per_token;
            if (tokens_out) *tokens_out = delta;
            return KVO_ACT_DELTA;
        }
        c->barrier = 1;
    }
    if (c->commit_scheduled || inflight_batches > 0) return KVO_ACT_BARRIER_WAIT;
    const int64_t final_delta = kvo_ctx_unsynced(c, n, req, kv);
    kvo_ctx_snapshot(c, n, req, kv, lo_out, hi_out);
    if (c->kv_synced_bytes) *c->kv_synced_bytes += (double)final_delta * c->kv_bytes_per_token;
    c->commit_scheduled = 1;
    if (tokens_out) *tokens_out = final_delta;
    return KVO_ACT_FINAL;
}

/* -------------------------------------------------------------- data plane */

uint64_t kvo_token_bytes(const kvo_geometry* g) {
    return (uint64_t)g->num_kv_heads * (uint64_t)g->head_dim * (uint64_t)g->elem_bytes;
}

uint64_t kvo_block_bytes(const kvo_geometry* g) {
    return 2ull * (uint64_t)g->block_tokens * kvo_token_bytes(g);
}

/* Byte offset of (layer_local, block, kv, token_in_block) inside a pool. */
static uint64_t row_offset(const kvo_geometry* g, int32_t blocks_per_pool, int32_t layer_local,
                           int32_t block, int32_t kv, int32_t tib) {
    const uint64_t tb = kvo_token_bytes(g);
    const uint64_t slab = ((uint64_t)layer_local * (uint64_t)blocks_per_pool + (uint64_t)block);
    return slab * kvo_block_bytes(g) + ((uint64_t)kv * (uint64_t)g->block_tokens + (uint64_t)tib) * tb;
}

void kvo_fill(const kvo_geometry* g, uint64_t seed, int32_t num_stages, const int32_t* b,
              uint8_t* const* pools, int32_t blocks_per_pool, int32_t n, const int32_t* req,
              const int64_t* tokens, const int32_t* bt, int32_t max_blocks) {
    const uint64_t tb = kvo_token_bytes(g);
    const uint32_t words = (uint32_t)(tb / 2);
    for (int32_t i = 0; i < n; ++i) {
        const int32_t r = req[i];
        for (int32_t l = 0; l < g->num_layers; ++l) {
            const int32_t s = kvo_stage_of_layer(num_stages, b, l);
            const int32_t ll = l - kvo_stage_begin(num_stages, b, s);
            for (int64_t t = 0; t < tokens[i]; ++t) {
                const int32_t blk = bt[(int64_t)r * max_blocks + t / g->block_tokens];
                for (int32_t kv = 0; kv < 2; ++kv) {
                    uint16_t* row = (uint16_t*)(pools[s] +
                                                row_offset(g, blocks_per_pool, ll, blk, kv,
                                                           (int32_t)(t % g->block_tokens)));
                    const uint64_t th = kvo_token_hash(seed, r, l, kv, t);
                    for (uint32_t w = 0; w < words; ++w) row[w] = kvo_word(th, w);
                }
            }
        }
    }
}

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

/* kvo_fill restricted to ONE model layer of one pool, on a zeroed image,
 * striped over `threads` pthreads: phase 1 zeroes a slice of the layer per
 * thread, phase 2 writes the rows of every (tid + k * threads)-th request. */
typedef struct {
    const kvo_geometry* g;
    uint64_t seed;
    int32_t layer, blocks_per_pool, n, max_blocks, tid, nthreads;
    uint8_t* buf;
    const int32_t *req, *bt;
    const int64_t* tokens;
} fill_job;

static void* fill_zero_worker(void* arg) {
    const fill_job* j = (const fill_job*)arg;
    const uint64_t bytes = (uint64_t)j->blocks_per_pool * kvo_block_bytes(j->g);
    const uint64_t per = (bytes + (uint64_t)j->nthreads - 1) / (uint64_t)j->nthreads;
    const uint64_t b0 = per * (uint64_t)j->tid;
    if (b0 < bytes) memset(j->buf + b0, 0, b0 + per < bytes ? per : bytes - b0);
    return NULL;
}

static void* fill_rows_worker(void* arg) {
    const fill_job* j = (const fill_job*)arg;
    const kvo_geometry* g = j->g;
    const uint32_t words = (uint32_t)(kvo_token_bytes(g) / 2);
    for (int32_t i = j->tid; i < j->n; i += j->nthreads) {
        const int32_t r = j->req[i];
        for (int64_t t = 0; t < j->tokens[i]; ++t) {
            const int32_t blk = j->bt[(int64_t)r * j->max_blocks + t / g->block_tokens];
            for (int32_t kv = 0; kv < 2; ++kv) {
                uint16_t* row = (uint16_t*)(j->buf + row_offset(g, j->blocks_per_pool, 0, blk, kv,
                                                                (int32_t)(t % g->block_tokens)));
                const uint64_t th = kvo_token_hash(j->seed, r, j->layer, kv, t);
                for (uint32_t w = 0; w < words; ++w) row[w] = kvo_word(th, w);
            }
        }
    }
    return NULL;
}

static void run_fill_phase(void* (*fn)(void*), fill_job* jobs, int32_t threads) {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int32_t t = 0; t < threads; ++t)
        if (threads == 1 || pthread_create(&th[t], NULL, fn, &jobs[t]) != 0) fn(&jobs[t]), th[t] = 0;
    for (int32_t t = 0; t < threads; ++t)
        if (th[t]) pthread_join(th[t], NULL);
    free(th);
}

void kvo_fill_layer(const kvo_geometry* g, uint64_t seed, int32_t layer, uint8_t* layer_buf,
                    int32_t blocks_per_pool, int32_t n, const int32_t* req, const int64_t* tokens,
                    const int32_t* bt, int32_t max_blocks, int32_t threads) {
    if (threads < 1) threads = 1;
    fill_job* jobs = (fill_job*)malloc(sizeof(fill_job) * (size_t)threads);
    for (int32_t t = 0; t < threads; ++t)
        jobs[t] = (fill_job){g, seed, layer, blocks_per_pool, n, max_blocks, t, threads, layer_buf, req, bt, tokens};
    run_fill_phase(fill_zero_worker, jobs, threads);
    run_fill_phase(fill_rows_worker, jobs, threads);
    free(jobs);
}

/* Destination block rule: a wave entry must start inside the already-copied
 * prefix (lo <= synced_hi; the reference guarantees lo == synced,
 * engine.cpp:548-556,657-661).  For the entries in the order given (ascending
 * request id == std::map order of sync_target, engine.hpp:153-154) the new
 * logical blocks [ceil(synced_hi/B), ceil(hi/B)) get consecutive ids from the
 * bump pointer.  Records the synced high-water mark. */
static int allocate_wave(const kvo_geometry* g, kvo_dst* d, int32_t n, const int32_t* req,
                         const int64_t* lo, const int64_t* hi) {
    const int64_t B = g->block_tokens;
    /* validate the whole wave first: a rejected wave changes nothing */
    int64_t need = 0;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t r = req[i];
        if (r < 0 || r >= d->max_requests || (i > 0 && req[i - 1] >= r)) return -1;
        if (hi[i] <= lo[i]) continue;
        if (lo[i] < 0 || lo[i] > d->synced_hi[r]) return -1;
        if (ceil_div(hi[i], B) > d->max_blocks) return -1;
        const int64_t add = ceil_div(hi[i], B) - ceil_div(d->synced_hi[r], B);
        need += add > 0 ? add : 0;
    }
    if (d->stack ? need > d->top : d->next_block + need > d->num_blocks) return -1;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t r = req[i];
        if (r < 0 || r >= d->max_requests || (i > 0 && req[i - 1] >= r)) return -1;
        if (hi[i] <= lo[i]) continue;
        if (lo[i] < 0 || lo[i] > d->synced_hi[r]) return -1; /* gap: tokens would be lost */
        const int64_t b0 = ceil_div(d->synced_hi[r], B), b1 = ceil_div(hi[i], B);
        if (b1 > d->max_blocks) return -1;
        for (int64_t b = b0; b < b1; ++b) {
            int32_t id;
            if (d->stack) {
                if (d->top <= 0) return -1;
                id = d->stack[--d->top];
            } else {
                if (d->next_block >= d->num_blocks) return -1;
                id = d->next_block++;
            }
            d->bt[(int64_t)r * d->max_blocks + b] = id;
        }
        if (hi[i] > d->synced_hi[r]) d->synced_hi[r] = hi[i];
    }
    return 0;
}

int kvo_apply_wave(const kvo_geometry* g, kvo_dst* d, int32_t old_stages, const int32_t* ob,
                   uint8_t* const* old_pools, int32_t old_blocks, const int32_t* src_bt,
                   int32_t new_stages, const int32_t* nb, uint8_t* const* new_pools, int32_t n,
                   const int32_t* req, const int64_t* lo, const int64_t* hi) {
    if (allocate_wave(g, d, n, req, lo, hi)) return -1;
    if (!old_pools || !new_pools) return 0; /* allocation-only replay */
    const uint64_t tb = kvo_token_bytes(g);
    const int32_t B = g->block_tokens;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t r = req[i];
        for (int32_t l = 0; l < g->num_layers; ++l) {
            const int32_t so = kvo_stage_of_layer(old_stages, ob, l);
            const int32_t sn = kvo_stage_of_layer(new_stages, nb, l);
            const int32_t lo_l = l - kvo_stage_begin(old_stages, ob, so);
            const int32_t ln_l = l - kvo_stage_begin(new_stages, nb, sn);
            for (int64_t t = lo[i]; t < hi[i]; ++t) {
                const int32_t sblk = src_bt[(int64_t)r * d->max_blocks + t / B];
                const int32_t dblk = d->bt[(int64_t)r * d->max_blocks + t / B];
                for (int32_t kv = 0; kv < 2; ++kv) {
                    memcpy(new_pools[sn] + row_offset(g, d->num_blocks, ln_l, dblk, kv, (int32_t)(t % B)),
                           old_pools[so] + row_offset(g, old_blocks, lo_l, sblk, kv, (int32_t)(t % B)),
                           tb);
                }
            }
        }
    }
    return 0;
}

/* ---- multi-threaded run-granular executor (CPU baseline) ---- */

typedef struct seg {
    int32_t req, blk;   /* logical block */
    int32_t t0, t1;     /* token range inside the block */
} seg;

typedef struct mt_job {
    const kvo_geometry* g;
    const kvo_dst* d;
    int32_t old_stages, new_stages, old_blocks;
    const int32_t *ob, *nb, *src_bt;
    uint8_t* const* old_pools;
    uint8_t* const* new_pools;
    const seg* segs;
    int64_t nseg;
    int32_t tid, nthreads;
} mt_job;

static void* mt_worker(void* arg) {
    const mt_job* j = (const mt_job*)arg;
    const kvo_geometry* g = j->g;
    const uint64_t tb = kvo_token_bytes(g);
    const int32_t B = g->block_tokens;
    const int64_t units = j->nseg * g->num_layers;
    /* contiguous chunk of (segment, layer) units per thread */
    const int64_t per = (units + j->nthreads - 1) / j->nthreads;
    const int64_t u0 = per * j->tid, u1 = u0 + per < units ? u0 + per : units;
    for (int64_t u = u0; u < u1; ++u) {
        const seg* s = &j->segs[u / g->num_layers];
        const int32_t l = (int32_t)(u % g->num_layers);
        const int32_t so = kvo_stage_of_layer(j->old_stages, j->ob, l);
        const int32_t sn = kvo_stage_of_layer(j->new_stages, j->nb, l);
        const int32_t lo_l = l - kvo_stage_begin(j->old_stages, j->ob, so);
        const int32_t ln_l = l - kvo_stage_begin(j->new_stages, j->nb, sn);
        const int32_t sblk = j->src_bt[(int64_t)s->req * j->d->max_blocks + s->blk];
        const int32_t dblk = j->d->bt[(int64_t)s->req * j->d->max_blocks + s->blk];
        if (s->t0 == 0 && s->t1 == B) {
            memcpy(j->new_pools[sn] + row_offset(g, j->d->num_blocks, ln_l, dblk, 0, 0),
                   j->old_pools[so] + row_offset(g, j->old_blocks, lo_l, sblk, 0, 0),
                   kvo_block_bytes(g));
        } else {
            for (int32_t kv = 0; kv < 2; ++kv)
                memcpy(j->new_pools[sn] + row_offset(g, j->d->num_blocks, ln_l, dblk, kv, s->t0),
                       j->old_pools[so] + row_offset(g, j->old_blocks, lo_l, sblk, kv, s->t0),
                       (uint64_t)(s->t1 - s->t0) * tb);
        }
    }
    return NULL;
}

int kvo_apply_wave_mt(const kvo_geometry* g, kvo_dst* d, int32_t old_stages, const int32_t* ob,
                      uint8_t* const* old_pools, int32_t old_blocks, const int32_t* src_bt,
                      int32_t new_stages, const int32_t* nb, uint8_t* const* new_pools, int32_t n,
                      const int32_t* req, const int64_t* lo, const int64_t* hi, int32_t threads) {
    if (allocate_wave(g, d, n, req, lo, hi)) return -1;
    const int64_t B = g->block_tokens;
    int64_t nseg = 0;
    for (int32_t i = 0; i < n; ++i)
        if (hi[i] > lo[i]) nseg += ceil_div(hi[i], B) - lo[i] / B;
    seg* segs = (seg*)malloc(sizeof(seg) * (size_t)(nseg > 0 ? nseg : 1));
    if (!segs) return -1;
    int64_t k = 0;
    for (int32_t i = 0; i < n; ++i) {
        if (hi[i] <= lo[i]) continue;
        for (int64_t b = lo[i] / B; b < ceil_div(hi[i], B); ++b) {
            const int64_t t0 = lo[i] > b * B ? lo[i] - b * B : 0;
            const int64_t t1 = hi[i] < (b + 1) * B ? hi[i] - b * B : B;
            segs[k++] = (seg){req[i], (int32_t)b, (int32_t)t0, (int32_t)t1};
        }
    }
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    mt_job* jobs = (mt_job*)malloc(sizeof(mt_job) * (size_t)threads);
    for (int32_t t = 0; t < threads; ++t) {
        jobs[t] = (mt_job){g, d, old_stages, new_stages, old_blocks, ob, nb, src_bt,
                           old_pools, new_pools, segs, nseg, t, threads};
        if (threads == 1) mt_worker(&jobs[t]);
        else pthread_create(&th[t], NULL, mt_worker, &jobs[t]);
    }
    if (threads > 1)
        for (int32_t t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    free(segs);
    return 0;
}

int64_t kvo_commit(const kvo_geometry* g, kvo_dst* d, int32_t n, const int32_t* req,
                   const int64_t* kv, int32_t* row_ptr, int32_t* blocks, int32_t* n_blocks,
                   int32_t* free_list, int32_t* n_free) {
    const int64_t B = g->block_tokens;
    int64_t violations = 0;
    uint8_t* live = (uint8_t*)calloc((size_t)d->max_requests, 1);
    int32_t nb = 0;
    if (row_ptr) row_ptr[0] = 0;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t r = req[i];
        live[r] = 1;
        /* Eq. 10 (engine.cpp:707-713) lifted to the copied high-water mark. */
        if (d->synced_hi[r] != kv[i]) ++violations;
        const int64_t have = ceil_div(d->synced_hi[r], B);
        for (int64_t b = 0; b < have; ++b)
            if (blocks) blocks[nb++] = d->bt[(int64_t)r * d->max_blocks + b];
            else ++nb;
        if (row_ptr) row_ptr[i + 1] = nb;
    }
    int32_t nf = 0;
    for (int32_t r = 0; r < d->max_requests; ++r) {
        if (live[r]) continue;
        const int64_t have = ceil_div(d->synced_hi[r], B);
        for (int64_t b = 0; b < have; ++b) {
            const int32_t id = d->bt[(int64_t)r * d->max_blocks + b];
            if (free_list) free_list[nf] = id;
            if (d->stack) d->stack[d->top++] = id; /* free-list update (pushed in order) */
            ++nf;
        }
    }
    free(live);
    if (n_blocks) *n_blocks = nb;
    if (n_free) *n_free = nf;
    return violations;
}

int64_t kvo_verify(const kvo_geometry* g, uint64_t seed, const kvo_dst* d, int32_t new_stages,
                   const int32_t* nb, uint8_t* const* new_pools, int32_t n, const int32_t* req,
                   const int64_t* kv) {
    const uint64_t tb = kvo_token_bytes(g);
    const uint32_t words = (uint32_t)(tb / 2);
    const int32_t B = g->block_tokens;
    int64_t bad = 0;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t r = req[i];
        for (int32_t l = 0; l < g->num_layers; ++l) {
            const int32_t sn = kvo_stage_of_layer(new_stages, nb, l);
            const int32_t ll = l - kvo_stage_begin(new_stages, nb, sn);
            for (int64_t t = 0; t < kv[i]; ++t) {
                const int32_t blk = d->bt[(int64_t)r * d->max_blocks + t / B];
                if (blk < 0) {
                    bad += 2 * (int64_t)words;
                    continue;
                }
                for (int32_t k = 0; k < 2; ++k) {
                    const uint16_t* row = (const uint16_t*)(new_pools[sn] +
                                                            row_offset(g, d->num_blocks, ll, blk, k,
                                                                       (int32_t)(t % B)));
                    const uint64_t th = kvo_token_hash(seed, r, l, k, t);
                    for (uint32_t w = 0; w < words; ++w) bad += row[w] != kvo_word(th, w);
                }
            }
        }
    }
    return bad;
}

int32_t kvo_activation_owner(int32_t old_stages, const int32_t* ob, int32_t new_stages,
                             const int32_t* nb, int32_t from_old_stage) {
    /* A micro-batch in transit from old stage s carries the input of layer
     * ob[s] (engine.cpp:449-456, 483-488); that layer's new owner resumes it. */
    if (from_old_stage < 0 || from_old_stage + 1 >= old_stages) return -1;
    return kvo_stage_of_layer(new_stages, nb, ob[from_old_stage]);
}

int kvo_handoff_plan(int32_t old_stages, const int32_t* ob, int32_t new_stages, const int32_t* nb,
                     uint64_t row_bytes, int32_t n, const int32_t* after, const int32_t* tokens,
                     const uint64_t* arena_bytes, int32_t* new_stage, int32_t* resume_layer,
                     uint64_t* offset, uint64_t* bytes) {
    uint64_t bump[256];
    if (new_stages > 256) return -1;
    for (int32_t k = 0; k < new_stages; ++k) bump[k] = 0;
    for (int32_t i = 0; i < n; ++i) {
        if (after[i] >= old_stages) return -1; /* no such old stage */
        if (after[i] < 0 || after[i] + 1 == old_stages) {
            /* < 0: nothing computed yet, re-dispatch at the new head;
             * == K_old-1: the forward pass finished on the old pipeline,
             * not in flight any more (engine.cpp:449-456 completes it): no slot */
            new_stage[i] = after[i] < 0 ? 0 : -1;
            resume_layer[i] = after[i] < 0 ? 0 : -1;
            offset[i] = 0;
            bytes[i] = 0;
            continue;
        }
        const int32_t layer = ob[after[i]];
        const int32_t k = kvo_stage_of_layer(new_stages, nb, layer);
        const uint64_t b = (uint64_t)tokens[i] * row_bytes;
        const uint64_t off = (bump[k] + 255u) & ~(uint64_t)255u;
        if (off + b > arena_bytes[k]) return -1;
        new_stage[i] = k;
        resume_layer[i] = layer;
        offset[i] = off;
        bytes[i] = b;
        bump[k] = off + b;
    }
    return 0;
}

void kvo_weights_plan(int32_t num_layers, uint64_t layer_bytes, int32_t old_stages,
                      const int32_t* ob, int32_t new_stages, const int32_t* nb, int32_t* src_stage,
                      uint64_t* src_off, int32_t* dst_stage, uint64_t* dst_off) {
    for (int32_t l = 0; l < num_layers; ++l) {
        const int32_t so = kvo_stage_of_layer(old_stages, ob, l);
        const int32_t sn = kvo_stage_of_layer(new_stages, nb, l);
        src_stage[l] = so;
        dst_stage[l] = sn;
        src_off[l] = (uint64_t)(l - kvo_stage_begin(old_stages, ob, so)) * layer_bytes;
        dst_off[l] = (uint64_t)(l - kvo_stage_begin(new_stages, nb, sn)) * layer_bytes;
    }
}

double kvo_warm_start_ms(int32_t n, const double* stage_bytes, const uint8_t* cached,
                         double host_bw, double storage_bw) {
    /* cluster.cpp:525-536 */
    double total = 0.0;
    for (int32_t k = 0; k < n; ++k) {
        if (stage_bytes[k] <= 0.0) continue;
        total += stage_bytes[k] / (cached[k] ? host_bw : storage_bw);
    }
    return total;
}

void kvo_bm_init(int32_t* stack, int32_t capacity) {
    for (int32_t i = 0; i < capacity; ++i) stack[i] = capacity - 1 - i;
}

void kvo_abort(const kvo_geometry* g, kvo_dst* d) {
    const int64_t B = g->block_tokens;
    for (int32_t r = 0; r < d->max_requests; ++r) {
        const int64_t have = ceil_div(d->synced_hi[r], B);
        for (int64_t b = 0; b < have; ++b) {
            if (d->stack) d->stack[d->top++] = d->bt[(int64_t)r * d->max_blocks + b];
            d->bt[(int64_t)r * d->max_blocks + b] = -1;
        }
        d->synced_hi[r] = 0;
    }
    d->next_block = 0;
}
