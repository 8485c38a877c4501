// kvx_kernels.cuh -- sm_100a device code of the inflight-refactor KV transition.
//
// Kernels (launched on the transition's stream):
//   kvx_plan_kernel      one CTA: destination block allocation (block-wide
//                        exclusive scan of per-request new-block counts; bump
//                        rule or pops off the block manager's free stack),
//                        block-table rewrite, synced high-water marks, the
//                        per-block copy segments of the wave, and a bounds
//                        check of every segment.  Reads the wave entries
//                        straight from mapped pinned memory.  Restates the
//                        "which tokens move" half of engine.cpp:637-687.
//   kvx_bulk_kernel      THE mover (default): persistent, one elected thread
//                        per CTA streams (segment, layer) slabs global ->
//                        shared -> global through a cp.async.bulk ring with
//                        mbarrier tx counts (SASS UBLKCP / SYNCS); local HBM
//                        or NVLink-peer destinations; optional CTA split
//                        between peer and local layers.  Launched with PDL
//                        behind the plan kernel (griddepcontrol.wait).
//                        Pools of any layout (per-layer base, block / K-V /
//                        token / head strides); NVLink-peer sources (pull) too.
//   kvx_move_kernel      LSU mover (16-byte ld.global.nc / st.global, 8 in
//                        flight per thread); kvx_move256_kernel its 256-bit
//                        variant.  KVX_MOVE_IMPL=lsu|lsu256.
//   kvx_move_any_kernel  row mover: (K|V, token, head) rows through both pools'
//                        strides -- token-major <-> head-major (HND) transposes,
//                        and head-major tails beside the bulk mover.
//   kvx_copy_list_kernel bulk engine over a (src, dst, bytes) list: activation
//                        handoff and stage weight migration.
//   kvx_commit_kernel    one CTA: Eq. 10 check per live request
//                        (engine.cpp:707-713) with warp ballots, CSR
//                        compaction of live rows, free list of rows no longer
//                        live (scans); results written into mapped pinned
//                        memory.  Runs beside the last wave's mover (side
//                        stream): it needs the table, not the bytes.
//   kvx_bm_init_kernel   block-manager stack initialisation.
//   kvx_fill_kernel / kvx_verify_kernel   synthetic payload (tests + bench).
#pragma once
// Included by several translation units: non-template kernels have internal
// linkage (static), templates are instantiated where used.

#include <cstdint>
#include <cuda.h>  // CUtensorMap (the type only; no driver calls here)
#include <cuda_runtime.h>

namespace kvx {

struct Seg {  // one logical block of one request inside one wave
    int32_t src_blk;
    int32_t dst_blk;
    int32_t t0;  // first token inside the block
    int32_t t1;  // one past the last token
};

struct LayerPtr {  // layer l in the old / new pool (address of block b, K|V k, token t, head h:
                   //   base + b*bs + k*kv + t*ts + h*hs)
    char* src;
    char* dst;
    uint64_t src_bs, dst_bs;  // bytes between consecutive blocks (layout-dependent)
    uint64_t src_kv, dst_kv;  // bytes from a block's K rows to its V rows
    uint64_t src_ts, dst_ts;  // token stride
    uint64_t src_hs, dst_hs;  // head stride
    uint32_t run_tok;         // run copies: bytes per token of one run (token_bytes or head bytes)
    uint32_t nh;              // run copies: runs per K/V of a partial block (1 token-major, H head-major)
};

struct PoolAddr {  // one pool for the payload kernels: per-layer bases + strides
    char* const* layer;  // device array, one base per layer
    uint64_t blk_stride, kv_stride, tok_stride, head_stride;
    uint32_t head_bytes;
};

// ---------------------------------------------------------------- payload
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t token_hash(uint64_t seed, int32_t req, int32_t layer,
                                                        int32_t kv, int64_t tok) {
    uint64_t h = mix64(seed ^ (uint64_t)(uint32_t)req);
    h = mix64(h ^ (((uint64_t)(uint32_t)layer << 1) | (uint64_t)(kv & 1)));
    return mix64(h ^ (uint64_t)tok);
}
__host__ __device__ __forceinline__ uint32_t word(uint64_t th, uint32_t w) {
    return (uint32_t)(((th + (uint64_t)w * 0x9E3779B97F4A7C15ull) * 0xBF58476D1CE4E5B9ull) >> 48);
}
__device__ __forceinline__ uint4 pattern_vec(uint64_t th, uint32_t vec) {
    const uint32_t w = vec * 8u;
    uint4 v;
    v.x = word(th, w + 0) | (word(th, w + 1) << 16);
    v.y = word(th, w + 2) | (word(th, w + 3) << 16);
    v.z = word(th, w + 4) | (word(th, w + 5) << 16);
    v.w = word(th, w + 6) | (word(th, w + 7) << 16);
    return v;
}

// ------------------------------------------------------------ scan helper
// Block-wide exclusive scan of two int32 counters at once (1024 threads).
template <int kThreads>
__device__ __forceinline__ int2 block_exclusive_scan2(int2 v, int2* total) {
    static_assert(kThreads % 32 == 0 && kThreads <= 1024, "threads");
    __shared__ int2 warp_sums[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int2 inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int ax = __shfl_up_sync(0xffffffffu, inc.x, d);
        const int ay = __shfl_up_sync(0xffffffffu, inc.y, d);
        if (lane >= d) {
            inc.x += ax;
            inc.y += ay;
        }
    }
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int2 s = lane < kThreads / 32 ? warp_sums[lane] : make_int2(0, 0);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int ax = __shfl_up_sync(0xffffffffu, s.x, d);
            const int ay = __shfl_up_sync(0xffffffffu, s.y, d);
            if (lane >= d) {
                s.x += ax;
                s.y += ay;
            }
        }
        warp_sums[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const int2 before = wid > 0 ? warp_sums[wid - 1] : make_int2(0, 0);
    *total = warp_sums[kThreads / 32 - 1];
    __syncthreads();  // warp_sums reused by the next call
    return make_int2(before.x + inc.x - v.x, before.y + inc.y - v.y);
}

__device__ __forceinline__ int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// -------------------------------------------------------------- planning
constexpr int kPlanThreads = 1024;

// Wave entries are strictly ascending request ids (validated on the host),
// so rows never collide.  Destination rule: the new blocks of a request are
// logical blocks [ceil(synced_hi/B), ceil(hi/B)); their ids are the bump
// pointer plus the exclusive scan of the per-entry counts, in entry order.
static __global__ void __launch_bounds__(kPlanThreads, 1)
kvx_plan_kernel(const int32_t* __restrict__ req, const int64_t* __restrict__ lo,
                const int64_t* __restrict__ hi, int32_t n, const int32_t* __restrict__ src_bt,
                int32_t* __restrict__ dst_bt, int64_t* __restrict__ synced_hi, int32_t max_blocks,
                int32_t block_tokens, int32_t alloc_base, const int32_t* __restrict__ pop_stack,
                Seg* __restrict__ segs, int32_t src_cap, int32_t dst_cap, int32_t* __restrict__ err) {
    // let the mover (launched behind with programmatic stream serialization)
    // become resident now; it waits (griddepcontrol.wait) for this grid's
    // completion before it reads the segments
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int64_t B = block_tokens;
    int2 carry = make_int2(0, 0);
    for (int32_t base = 0; base < n; base += kPlanThreads) {
        const int32_t i = base + (int32_t)threadIdx.x;
        int32_t r = -1;
        int64_t l = 0, h = 0, s = 0;
        int2 cnt = make_int2(0, 0);  // (new blocks, segments)
        if (i < n) {
            r = req[i];
            l = lo[i];
            h = hi[i];
            s = synced_hi[r];
            if (h > l) {
                const int64_t have = cdiv(s, B), need = cdiv(h, B);
                cnt.x = need > have ? (int32_t)(need - have) : 0;
                cnt.y = (int32_t)(need - l / B);
            }
        }
        int2 tot;
        const int2 off = block_exclusive_scan2<kPlanThreads>(cnt, &tot);
        if (i < n && h > l) {
            int32_t* row = dst_bt + (int64_t)r * max_blocks;
            const int32_t* srow = src_bt + (int64_t)r * max_blocks;
            const int64_t have = cdiv(s, B);
            // bump pointer, or pops off the block manager's free stack
            // (alloc_base = its top): the j-th pop of the wave is stack[top-1-j]
            for (int32_t k = 0; k < cnt.x; ++k) {
                const int32_t j = carry.x + off.x + k;
                row[have + k] = pop_stack ? pop_stack[alloc_base - 1 - j] : alloc_base + j;
            }
            if (h > s) synced_hi[r] = h;
            const int64_t b0 = l / B;
            Seg* out = segs + carry.y + off.y;
            for (int32_t k = 0; k < cnt.y; ++k) {
                const int64_t b = b0 + k;
                const int64_t t0 = l > b * B ? l - b * B : 0;
                const int64_t t1 = h < (b + 1) * B ? h - b * B : B;
                Seg sg{srow[b], row[b], (int32_t)t0, (int32_t)t1};
                // bounds check on every segment (defence in depth behind the host
                // validation): an id outside its pool becomes an empty run, so the
                // mover never touches memory out of range; the error word reports it
                if (sg.src_blk < 0 || sg.src_blk >= src_cap || sg.dst_blk < 0 || sg.dst_blk >= dst_cap) {
                    *reinterpret_cast<volatile int32_t*>(err) = 1;  // idempotent; err is host-mapped
                    sg.t0 = sg.t1 = 0;
                }
                out[k] = sg;
            }
        }
        carry.x += tot.x;
        carry.y += tot.y;
    }
}

// Block-manager helper: stack[i] = capacity - 1 - i (pops yield 0, 1, 2, ...).
static __global__ void kvx_bm_init_kernel(int32_t* __restrict__ stack, int32_t capacity) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < capacity; i += gridDim.x * blockDim.x)
        stack[i] = capacity - 1 - i;
}

// Stream-ordered pop into a device array, LIFO (out[i] = stack[top-1-i], the
// order kvx_bm_pop and the plan kernel use).
static __global__ void kvx_bm_pop_kernel(const int32_t* __restrict__ stack, int32_t top, int32_t n,
                                         int32_t* __restrict__ out) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = stack[top - 1 - i];
}

// Stream-ordered push of device ids: stack[top+i] = ids[i].  An id outside
// [0, capacity) is not pushed (its slot gets -1) and raises the manager's
// error word, reported by the next host call on the manager.
static __global__ void kvx_bm_push_kernel(int32_t* __restrict__ stack, int32_t top, int32_t n,
                                          const int32_t* __restrict__ ids, int32_t capacity,
                                          int32_t* __restrict__ err) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int32_t v = ids[i];
        const bool ok = v >= 0 && v < capacity;
        stack[top + i] = ok ? v : -1;
        if (!ok) *reinterpret_cast<volatile int32_t*>(err) = 1;
    }
}

// Source-table rows replaced mid-transition (kvx_src_rows): table[req[i]] =
// rows[i], read straight from the pinned staging (zero-copy).
static __global__ void kvx_rows_kernel(const int32_t* __restrict__ req, const int32_t* __restrict__ rows, int32_t n,
                                       int32_t max_blocks, int32_t* __restrict__ table) {
    for (int32_t i = blockIdx.x; i < n; i += gridDim.x)
        for (int32_t b = threadIdx.x; b < max_blocks; b += blockDim.x)
            table[(int64_t)req[i] * max_blocks + b] = rows[(int64_t)i * max_blocks + b];
}

// ------------------------------------------------------------ LSU mover
constexpr int kMoveThreads = 512;
constexpr int kMoveUnroll = 8;

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream(uint4* p, const uint4& v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// CTA-cooperative copy of nvec 16-byte vectors.
__device__ __forceinline__ void cta_copy(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                         uint32_t nvec) {
    uint32_t i = threadIdx.x;
    const uint32_t step = kMoveThreads * kMoveUnroll;
    for (; i + (kMoveUnroll - 1) * kMoveThreads < nvec; i += step) {
        uint4 v[kMoveUnroll];
#pragma unroll
        for (int u = 0; u < kMoveUnroll; ++u) v[u] = ld_stream(src + i + u * kMoveThreads);
#pragma unroll
        for (int u = 0; u < kMoveUnroll; ++u) st_stream(dst + i + u * kMoveThreads, v[u]);
    }
    for (; i < nvec; i += kMoveThreads) st_stream(dst + i, ld_stream(src + i));
}

// 256-bit variant (sm_100: LDG/STG.256): half the memory instructions per
// byte; needs 32-byte-aligned runs (token_bytes % 32 == 0, checked on host).
struct alignas(32) V8 {
    uint32_t w[8];
};
__device__ __forceinline__ V8 ld_stream256(const V8* p) {
    V8 v;
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]),
                   "=r"(v.w[6]), "=r"(v.w[7])
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream256(V8* p, const V8& v) {
    asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]),
                 "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
                 : "memory");
}
__device__ __forceinline__ void cta_copy256(V8* __restrict__ dst, const V8* __restrict__ src, uint32_t n) {
    constexpr int kU = 4;
    uint32_t i = threadIdx.x;
    const uint32_t step = kMoveThreads * kU;
    for (; i + (kU - 1) * kMoveThreads < n; i += step) {
        V8 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = ld_stream256(src + i + u * kMoveThreads);
#pragma unroll
        for (int u = 0; u < kU; ++u) st_stream256(dst + i + u * kMoveThreads, v[u]);
    }
    for (; i < n; i += kMoveThreads) st_stream256(dst + i, ld_stream256(src + i));
}

static __global__ void __launch_bounds__(kMoveThreads)
kvx_move256_kernel(const Seg* __restrict__ segs, int32_t nseg, const LayerPtr* __restrict__ layers,
                   int32_t nlayers, uint64_t block_bytes, uint64_t token_bytes, int32_t block_tokens,
                   int32_t fence_system) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t units = (int64_t)nseg * nlayers;
    const uint64_t half = block_bytes >> 1;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int32_t layer = (int32_t)(u / nseg);
        const Seg sg = segs[u - (int64_t)layer * nseg];
        const LayerPtr lp = layers[layer];
        const char* src = lp.src + (uint64_t)sg.src_blk * lp.src_bs;
        char* dst = lp.dst + (uint64_t)sg.dst_blk * lp.dst_bs;
        if (sg.t0 == 0 && sg.t1 == block_tokens && lp.src_kv == half && lp.dst_kv == half) {
            cta_copy256(reinterpret_cast<V8*>(dst), reinterpret_cast<const V8*>(src), (uint32_t)(block_bytes >> 5));
        } else {  // K then V rows; per head for head-major pools
            const uint64_t off = (uint64_t)sg.t0 * lp.run_tok;
            const uint32_t n = (uint32_t)(((uint64_t)(sg.t1 - sg.t0) * lp.run_tok) >> 5);
            for (uint32_t r = 0; r < 2 * lp.nh; ++r) {
                const uint32_t kv = r / lp.nh, h = r % lp.nh;
                cta_copy256(reinterpret_cast<V8*>(dst + kv * lp.dst_kv + h * lp.dst_hs + off),
                            reinterpret_cast<const V8*>(src + kv * lp.src_kv + h * lp.src_hs + off), n);
            }
        }
    }
    if (fence_system) __threadfence_system();
}

// Work unit u -> (layer = u / nseg, segment = u % nseg): consecutive CTAs walk
// consecutive destination blocks of one layer (the dense rule makes them
// contiguous), sources are wherever the old block table points.
static __global__ void __launch_bounds__(kMoveThreads)
kvx_move_kernel(const Seg* __restrict__ segs, int32_t nseg, const LayerPtr* __restrict__ layers,
                int32_t nlayers, uint64_t block_bytes, uint64_t token_bytes, int32_t block_tokens,
                int32_t fence_system) {
    // launched with programmatic dependent launch behind the plan kernel:
    // wait until its segment list is complete and visible (no-op otherwise)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t units = (int64_t)nseg * nlayers;
    const uint64_t half = block_bytes >> 1;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int32_t layer = (int32_t)(u / nseg);
        const Seg sg = segs[u - (int64_t)layer * nseg];
        const LayerPtr lp = layers[layer];
        const char* src = lp.src + (uint64_t)sg.src_blk * lp.src_bs;
        char* dst = lp.dst + (uint64_t)sg.dst_blk * lp.dst_bs;
        if (sg.t0 == 0 && sg.t1 == block_tokens && lp.src_kv == half && lp.dst_kv == half) {
            cta_copy(reinterpret_cast<uint4*>(dst), reinterpret_cast<const uint4*>(src),
                     (uint32_t)(block_bytes >> 4));
        } else {  // K then V rows; per head for head-major pools
            const uint64_t off = (uint64_t)sg.t0 * lp.run_tok;
            const uint32_t nvec = (uint32_t)(((uint64_t)(sg.t1 - sg.t0) * lp.run_tok) >> 4);
            for (uint32_t r = 0; r < 2 * lp.nh; ++r) {
                const uint32_t kv = r / lp.nh, h = r % lp.nh;
                cta_copy(reinterpret_cast<uint4*>(dst + kv * lp.dst_kv + h * lp.dst_hs + off),
                         reinterpret_cast<const uint4*>(src + kv * lp.src_kv + h * lp.src_hs + off), nvec);
            }
        }
    }
    if (fence_system) __threadfence_system();  // peer (NVLink) stores visible before host sync
}

// --------------------------------------------- row-granular mover
// Copies (K|V, token, head) rows of head_bytes, addressed through both
// pools' strides -- any layout pair.  Used for moves between token-major
// (BLOCKS, KV_PLANES) and head-major (HEADS) pools (tails_only = 0), and for
// the partial blocks of head-major-to-head-major moves, whose 2*H short runs
// would starve the bulk mover's single issuing thread (tails_only = 1: full
// blocks are left to kvx_bulk_kernel; tails_only = 2: the partial blocks of a
// transposing wave whose whole blocks go to kvx_tmap_kernel).  Vectors of one row go to consecutive
// threads; rows are ordered tokens-inner when the source is head-major (its
// contiguous direction), heads-inner otherwise.  4 independent 16-byte loads
// in flight per thread.
// Unsigned 32-bit division by a divisor fixed for many dividends: one
// __umulhi + add + shifts (round-up magic, exact for every 32-bit n).
struct FastDiv {
    uint32_t d, m, l;
    __device__ __forceinline__ void init(uint32_t dv) {
        d = dv;
        l = 0;
        while (l < 32 && (1ull << l) < (uint64_t)dv) ++l;  // ceil(log2 d)
        m = (uint32_t)(((1ull << 32) * ((1ull << l) - dv)) / dv + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        if (d == 1) return n;
        const uint32_t t = __umulhi(m, n);
        return (t + ((n - t) >> 1)) >> (l - 1);
    }
};

static __global__ void __launch_bounds__(kMoveThreads)
kvx_move_any_kernel(const Seg* __restrict__ segs, int32_t nseg, const LayerPtr* __restrict__ layers,
                    int32_t nlayers, int32_t heads, uint32_t head_bytes, int32_t block_tokens,
                    int32_t tails_only, int32_t fence_system) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    constexpr int kU = 4;
    const int64_t units = (int64_t)nseg * nlayers;
    const uint32_t vph = head_bytes >> 4;  // 16-byte vectors per row
    const uint32_t H = (uint32_t)heads;
    // divisors fixed per kernel / per unit (FastDiv): token-granular transposing
    // waves 100 -> 87 us on C3's final wave; whole blocks go to kvx_tmap_kernel
    // (same box, profiles/r02af_ab_transposers_same_box.jsonl)
    FastDiv fv, fh, ft;
    fv.init(vph);
    fh.init(H);
    uint32_t ft_n = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int32_t layer = (int32_t)(u / nseg);
        const Seg sg = segs[u - (int64_t)layer * nseg];
        const LayerPtr lp = layers[layer];
        const bool full = sg.t0 == 0 && sg.t1 == block_tokens;
        if (tails_only == 1 && (lp.nh <= 1 || full)) continue;
        if (tails_only == 2 && full) continue;  // whole blocks: kvx_tmap_kernel
        const char* sb = lp.src + (uint64_t)sg.src_blk * lp.src_bs;
        char* db = lp.dst + (uint64_t)sg.dst_blk * lp.dst_bs;
        const uint32_t ntok = (uint32_t)(sg.t1 - sg.t0);
        if (ntok == 0) continue;  // emptied by the plan kernel's bounds check
        const uint32_t per_kv = ntok * H * vph;
        const bool tok_inner = lp.src_ts < lp.src_hs;  // head-major source (order barely matters:
                                                        // profiles/r01_row_sweep.jsonl)
        if (tok_inner && ntok != ft_n) {
            ft.init(ntok);
            ft_n = ntok;
        }
        const uint32_t total = 2 * per_kv;
        for (uint32_t base = threadIdx.x; base < total; base += kMoveThreads * kU) {
            uint4 v[kU];
            uint4* dp[kU];
#pragma unroll
            for (int k = 0; k < kU; ++k) {
                const uint32_t i = base + (uint32_t)k * kMoveThreads;
                dp[k] = nullptr;
                if (i < total) {
                    const uint32_t kv = i >= per_kv ? 1u : 0u, r = i - kv * per_kv;
                    const uint32_t row = fv.div(r), w = r - row * vph;
                    uint32_t h, t;
                    if (tok_inner) {
                        h = ft.div(row);
                        t = (uint32_t)sg.t0 + row - h * ntok;
                    } else {
                        const uint32_t tt = fh.div(row);
                        h = row - tt * H;
                        t = (uint32_t)sg.t0 + tt;
                    }
                    v[k] = ld_stream(reinterpret_cast<const uint4*>(sb + kv * lp.src_kv + t * lp.src_ts +
                                                                    h * lp.src_hs) + w);
                    dp[k] = reinterpret_cast<uint4*>(db + kv * lp.dst_kv + t * lp.dst_ts + h * lp.dst_hs) + w;
                }
            }
#pragma unroll
            for (int k = 0; k < kU; ++k)
                if (dp[k]) st_stream(dp[k], v[k]);
        }
    }
    if (fence_system) __threadfence_system();
}

// ------------------------------------------------------- TMA bulk mover
// One elected thread per CTA streams the CTA's (segment, layer) work through
// a kBulkStages-deep shared-memory ring with the bulk-copy engine:
//   cp.async.bulk global->shared (completes on an mbarrier with tx bytes),
//   cp.async.bulk shared->global (bulk_group; .read completion frees the slot).
// No registers carry payload; the SM's LSU pipe is idle.  Same work list and
// unit order as kvx_move_kernel.
constexpr int kBulkStages = 6;           // default ring depth
constexpr uint32_t kBulkChunk = 32768;   // default bytes per stage (16-byte multiple)
constexpr int kBulkThreads = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem)),
        "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem),
                 "r"(smem_u32(smem)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Copy descriptor of one (segment, layer) unit, resolved ahead of time by the
// CTA's helper lanes (kvx_bulk_kernel): the issuing lane then never waits on
// the dependent global loads of segs[] / layers[] -- one per unit, i.e. per
// 20 KiB of a token-granular wave -- between two bulk copies.
struct UnitDesc {
    const char* src;  // first run (K rows of the first head), offset applied
    char* dst;
    uint64_t src_kv, dst_kv, src_hs, dst_hs;
    uint32_t run_bytes;
    int32_t nrun;  // 0: nothing to move (empty segment / head-major tail)
    uint32_t nh;
    uint32_t pad;
};
constexpr int kDescBatch = 31;  // helper lanes 1..31 resolve one unit each per batch

__device__ __forceinline__ UnitDesc resolve_unit(const Seg* __restrict__ segs, const LayerPtr* __restrict__ layers,
                                                 int32_t nseg, int64_t u, uint64_t block_bytes,
                                                 int32_t block_tokens) {
    UnitDesc d{};
    if (u < 0) return d;
    const int32_t layer = (int32_t)(u / nseg);
    const Seg sg = segs[u - (int64_t)layer * nseg];
    const LayerPtr lp = layers[layer];
    const bool full = sg.t0 == 0 && sg.t1 == block_tokens;
    if (sg.t1 <= sg.t0) return d;      // emptied by the plan kernel's bounds check
    if (lp.nh > 1 && !full) return d;  // head-major tail: kvx_move_any_kernel(tails_only)
    const char* bs = lp.src + (uint64_t)sg.src_blk * lp.src_bs;
    char* bd = lp.dst + (uint64_t)sg.dst_blk * lp.dst_bs;
    const uint64_t half = block_bytes >> 1;
    d.src_kv = lp.src_kv;
    d.dst_kv = lp.dst_kv;
    d.src_hs = lp.src_hs;
    d.dst_hs = lp.dst_hs;
    if (full && lp.src_kv == half && lp.dst_kv == half) {
        d.nrun = 1;  // the whole block is one run on both sides (BLOCKS, HEADS)
        d.nh = 1;
        d.run_bytes = (uint32_t)block_bytes;
        d.src = bs;
        d.dst = bd;
    } else {  // K rows then V rows; per head for head-major pools
        const uint64_t off0 = (uint64_t)sg.t0 * lp.run_tok;
        d.nh = lp.nh;
        d.nrun = 2 * (int32_t)lp.nh;
        d.run_bytes = (uint32_t)((uint64_t)(sg.t1 - sg.t0) * lp.run_tok);
        d.src = bs + off0;
        d.dst = bd + off0;
    }
    return d;
}

// The issuing lane's side: walks the descriptors batch by batch (double
// buffered in shared memory; one __syncwarp hand-off per batch with the
// helpers, which resolve batch b+1 while batch b streams) and cuts each run
// into chunks of <= `chunk` bytes.
struct UnitIter {
    UnitDesc (*desc)[kDescBatch];
    int64_t my_units, nbatch;
    int64_t batch = -1;  // batch currently in `desc[batch & 1]`
    int pos = kDescBatch;
    int64_t seen = 0;    // units consumed so far
    uint32_t chunk;
    UnitDesc cur;
    int run = 0;
    const char* src;
    char* dst;
    uint64_t left = 0;

    __device__ bool load_unit() {
        for (;;) {
            if (seen >= my_units) return false;
            if (pos == kDescBatch) {  // next batch: meet the helpers
                ++batch;
                __syncwarp();
                pos = 0;
            }
            cur = desc[batch & 1][pos++];
            ++seen;
            if (cur.nrun == 0) continue;
            run = 0;
            src = cur.src;
            dst = cur.dst;
            left = cur.run_bytes;
            return true;
        }
    }
    __device__ bool next(const char** s, char** d, uint32_t* n) {
        while (left == 0) {
            if (++run < cur.nrun) {  // next (K|V, head) run of the unit
                const uint32_t kv = (uint32_t)run / cur.nh, h = (uint32_t)run % cur.nh;
                src = cur.src + kv * cur.src_kv + h * cur.src_hs;
                dst = cur.dst + kv * cur.dst_kv + h * cur.dst_hs;
                left = cur.run_bytes;
                continue;
            }
            if (!load_unit()) return false;
        }
        const uint32_t c = left > chunk ? chunk : (uint32_t)left;
        *s = src;
        *d = dst;
        *n = c;
        src += c;
        dst += c;
        left -= c;
        return true;
    }
};

// Generic single-thread bulk streaming loop over any chunk iterator with
// `bool next(const char**, char**, uint32_t*)`.
//   ring:  kStages slots of kChunk bytes; slot st completes on mbarrier st.
//   pack:  a slot takes up to kPack consecutive pieces (each <= kChunk) while
//          they fit, so short runs (a token's K or V row, a few KiB) do not
//          leave most of a slot empty -- the loads of a slot complete on its
//          mbarrier together (expect_tx = their sum), its stores form one
//          bulk group.
//   lag:   a slot is refilled once the store issued kLag slots earlier has
//          read shared memory (cp.async.bulk.wait_group.read kLag-1), so up to
//          kLag store groups drain while kStages - kLag slots load.
// kPack = 1, kLag = 2 is the slab configuration (one 64 KiB chunk per slot).
template <int kStages, uint32_t kChunk, int kLag = 2, int kPack = 1, class Iter>
__device__ __forceinline__ void bulk_stream(Iter& it, unsigned char* smem, uint64_t* bars) {
    static_assert(kLag >= 1 && kLag < kStages, "lag");
    static_assert(kPack >= 1, "pack");
    for (int i = 0; i < kStages; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    char* pend_dst[kStages][kPack];
    uint32_t pend_n[kStages][kPack];
    int pend_k[kStages];
    // one piece of look-ahead: the next piece is only taken into a slot if it fits
    const char* ns = nullptr;
    char* nd = nullptr;
    uint32_t nn = 0;
    bool have = it.next(&ns, &nd, &nn);
    auto fill = [&](int st) -> bool {
        if (!have) return false;
        const char* src[kPack];
        uint32_t used = 0, k = 0;
        while (have && k < (uint32_t)kPack && used + nn <= kChunk) {
            src[k] = ns;
            pend_dst[st][k] = nd;
            pend_n[st][k] = nn;
            used += nn;
            ++k;
            have = it.next(&ns, &nd, &nn);
        }
        pend_k[st] = (int)k;
        mbar_expect_tx(&bars[st], used);
        uint32_t off = 0;
        for (uint32_t q = 0; q < k; ++q) {
            bulk_g2s(smem + (size_t)st * kChunk + off, src[q], pend_n[st][q], &bars[st]);
            off += pend_n[st][q];
        }
        return true;
    };
    int64_t issued = 0, stored = 0;
    for (int st = 0; st < kStages; ++st) {  // prologue: fill the ring
        if (!fill(st)) break;
        ++issued;
    }
    while (stored < issued) {
        const int st = (int)(stored % kStages);
        const uint32_t parity = (uint32_t)((stored / kStages) & 1);
        mbar_wait(&bars[st], parity);
        uint32_t off = 0;
        for (int q = 0; q < pend_k[st]; ++q) {
            bulk_s2g(pend_dst[st][q], smem + (size_t)st * kChunk + off, pend_n[st][q]);
            off += pend_n[st][q];
        }
        bulk_commit();
        ++stored;
        // refill the slot stored kLag slots ago once its store has read smem
        if (have && stored >= kLag) {
            const int rs = (int)((stored - kLag) % kStages);
            bulk_wait_read<kLag - 1>();
            if (fill(rs)) ++issued;
        }
    }
    bulk_wait_all();
}

// The first n_peer layers of `layers` have a peer (NVLink) destination.  When
// a wave mixes them with local layers, CTAs [0, peer_ctas) stream only the
// peer units and the rest only the local ones, so the NVLink-bound and the
// HBM-bound traffic overlap instead of running layer after layer.
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// t_start / t_end (optional): the launch's own duration, first CTA start to
// last CTA end on %globaltimer (atomicMin / atomicMax) -- kvx_move_timings
// reads it, so no timing events sit in the stream on the stall path.
template <int kStages, uint32_t kChunk, int kLag = 2, int kPack = 1>
__global__ void __launch_bounds__(kBulkThreads)
kvx_bulk_kernel(const Seg* __restrict__ segs, int32_t nseg, const LayerPtr* __restrict__ layers,
                int32_t nlayers, uint64_t block_bytes, uint64_t token_bytes, int32_t block_tokens,
                int32_t n_peer, int32_t peer_ctas, unsigned long long* t_start, unsigned long long* t_end) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[kStages];
    __shared__ UnitDesc desc[2][kDescBatch];
    (void)token_bytes;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the plan kernel's segments
    if (t_start && threadIdx.x == 0) atomicMin(t_start, global_ns());
    // this CTA's units: u0, u0 + ustep, ... < units
    int64_t u0, ustep, units;
    const int64_t split = (int64_t)nseg * n_peer;
    if (peer_ctas > 0 && n_peer > 0 && n_peer < nlayers && (int)gridDim.x > peer_ctas) {
        if ((int)blockIdx.x < peer_ctas) {
            u0 = blockIdx.x;
            ustep = peer_ctas;
            units = split;
        } else {
            u0 = split + (blockIdx.x - peer_ctas);
            ustep = gridDim.x - peer_ctas;
            units = (int64_t)nseg * nlayers;
        }
    } else {
        u0 = blockIdx.x;
        ustep = gridDim.x;
        units = (int64_t)nseg * nlayers;
    }
    const int64_t my_units = u0 < units ? (units - u0 + ustep - 1) / ustep : 0;
    const int64_t nbatch = (my_units + kDescBatch - 1) / kDescBatch;
    if (nbatch == 0) return;
    const int lane = (int)threadIdx.x;
    if (lane != 0) {  // helpers: resolve batch b, publish it, go on with b + 1
        for (int64_t b = 0; b < nbatch; ++b) {
            const int64_t k = b * kDescBatch + (lane - 1);
            desc[b & 1][lane - 1] =
                resolve_unit(segs, layers, nseg, k < my_units ? u0 + k * ustep : -1, block_bytes, block_tokens);
            __syncwarp();  // batch b is visible to the issuing lane
        }
        return;
    }
    UnitIter it;
    it.desc = desc;
    it.my_units = my_units;
    it.nbatch = nbatch;
    it.chunk = kChunk;
    if (it.load_unit()) bulk_stream<kStages, kChunk, kLag, kPack>(it, smem, bars);
    if (t_end) atomicMax(t_end, global_ns());  // after bulk_wait_all: this CTA's stores landed
}

// ------------------------------------------- TMA tensor-map transposer
// Whole blocks between a token-major pool (per K|V plane [B][H][D]) and a
// head-major one ([H][B][D]).  The token-major side of every layer is
// described by a 5-D tensor map over (D, B, H, K|V, block) -- dims ordered
// head-outer with the pool's real strides -- so one box (D, B, hc) lands in
// shared memory as a head-major tile [hc][B][D]: the bulk engine does the
// transpose, no thread touches the payload.  The head-major side is a plain
// contiguous range of hc head planes.
//   t2h (token-major -> head-major): tensor load, 1-D bulk store
//   h2t (head-major -> token-major): 1-D bulk load, tensor store
// A box that runs past the last head is zero-filled on load (and only the
// valid heads are stored) or clipped on store.  Partial blocks stay with the
// row mover (kvx_move_any_kernel, tails_only = 2).  Same ring discipline as
// bulk_stream: kStages slots, refill once the store kLag slots back has read
// its slot.
__device__ __forceinline__ void tmap_g2s(void* smem, const CUtensorMap* map, int32_t c2, int32_t c3, int32_t c4,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(smem_u32(smem)),
        "l"(map), "r"(0), "r"(0), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmap_s2g(const CUtensorMap* map, int32_t c2, int32_t c3, int32_t c4, const void* smem) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                     map),
                 "r"(0), "r"(0), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(smem))
                 : "memory");
}

template <int kStages, int kLag>
__global__ void __launch_bounds__(32)
kvx_tmap_kernel(const Seg* __restrict__ segs, int32_t nseg, const LayerPtr* __restrict__ layers, int32_t nlayers,
                const CUtensorMap* __restrict__ maps, int32_t heads, int32_t hc, uint32_t head_plane,
                int32_t block_tokens, int32_t t2h) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[kStages];
    if (threadIdx.x != 0) return;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t slot = (uint32_t)hc * head_plane;  // bytes of one full box
    const int32_t nchunk = (heads + hc - 1) / hc;
    const int64_t pieces_per_unit = 2 * (int64_t)nchunk;
    const int64_t units = (int64_t)nseg * nlayers;
    // walk (unit, K|V, head chunk) of this CTA's units; full blocks only
    int64_t u = blockIdx.x;
    int64_t p = 0;  // piece within the unit
    struct Piece {
        const CUtensorMap* map;
        const char* hm_src;  // head-major side (h2t: load from; t2h: store to)
        char* hm_dst;
        int32_t c2, c3, c4;
        uint32_t bytes;  // valid head-plane bytes
    };
    Piece cur{};
    bool unit_ok = false;
    LayerPtr lp{};
    Seg sg{};
    int32_t layer = 0;
    auto next = [&](Piece* out) -> bool {
        for (;;) {
            if (u >= units) return false;
            if (!unit_ok || p == pieces_per_unit) {
                if (unit_ok) u += gridDim.x;
                p = 0;
                unit_ok = false;
                if (u >= units) return false;
                layer = (int32_t)(u / nseg);
                sg = segs[u - (int64_t)layer * nseg];
                lp = layers[layer];
                if (!(sg.t0 == 0 && sg.t1 == block_tokens)) {  // partial: the row mover's
                    u += gridDim.x;
                    continue;
                }
                unit_ok = true;
            }
            const int32_t kv = (int32_t)(p / nchunk), ch = (int32_t)(p % nchunk);
            ++p;
            const int32_t h0 = ch * hc;
            const int32_t nh = heads - h0 < hc ? heads - h0 : hc;
            out->map = maps + layer;
            out->c2 = h0;
            out->c3 = kv;
            out->c4 = t2h ? sg.src_blk : sg.dst_blk;
            out->bytes = (uint32_t)nh * head_plane;
            if (t2h) {
                out->hm_dst = lp.dst + (uint64_t)sg.dst_blk * lp.dst_bs + kv * lp.dst_kv + (uint64_t)h0 * lp.dst_hs;
                out->hm_src = nullptr;
            } else {
                out->hm_src = lp.src + (uint64_t)sg.src_blk * lp.src_bs + kv * lp.src_kv + (uint64_t)h0 * lp.src_hs;
                out->hm_dst = nullptr;
            }
            return true;
        }
    };
    for (int i = 0; i < kStages; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    Piece pend[kStages];
    bool have = next(&cur);
    auto fill = [&](int st) -> bool {
        if (!have) return false;
        pend[st] = cur;
        unsigned char* s = smem + (size_t)st * slot;
        if (t2h) {
            mbar_expect_tx(&bars[st], slot);  // the whole box arrives (heads past the end zero-filled)
            tmap_g2s(s, cur.map, cur.c2, cur.c3, cur.c4, &bars[st]);
        } else {
            mbar_expect_tx(&bars[st], cur.bytes);
            bulk_g2s(s, cur.hm_src, cur.bytes, &bars[st]);
        }
        have = next(&cur);
        return true;
    };
    int64_t issued = 0, stored = 0;
    for (int st = 0; st < kStages; ++st) {
        if (!fill(st)) break;
        ++issued;
    }
    while (stored < issued) {
        const int st = (int)(stored % kStages);
        mbar_wait(&bars[st], (uint32_t)((stored / kStages) & 1));
        const Piece& pc = pend[st];
        unsigned char* s = smem + (size_t)st * slot;
        if (t2h)
            bulk_s2g(pc.hm_dst, s, pc.bytes);
        else
            tmap_s2g(pc.map, pc.c2, pc.c3, pc.c4, s);  // heads past the end are clipped
        bulk_commit();
        ++stored;
        if (have && stored >= kLag) {
            bulk_wait_read<kLag - 1>();
            if (fill((int)((stored - kLag) % kStages))) ++issued;
        }
    }
    bulk_wait_all();
}

// ------------------------------------------------- generic copy list
// Activation handoff (and any batched device copy): a list of (src, dst,
// bytes) pieces, 16-byte aligned, streamed by the same bulk engine loop.
struct Piece {
    const char* src;
    char* dst;
    uint64_t bytes;
};

struct PieceIter {
    const Piece* p;
    int64_t n, i, step;
    const char* src;
    char* dst;
    uint64_t left;
    uint32_t chunk;
    __device__ bool next(const char** s, char** d, uint32_t* c) {
        while (left == 0) {
            i += step;
            if (i >= n) return false;
            src = p[i].src;
            dst = p[i].dst;
            left = p[i].bytes;
        }
        const uint32_t k = left > chunk ? chunk : (uint32_t)left;
        *s = src;
        *d = dst;
        *c = k;
        src += k;
        dst += k;
        left -= k;
        return true;
    }
};

template <int kStages, uint32_t kChunk>
__global__ void __launch_bounds__(kBulkThreads)
kvx_copy_list_kernel(const Piece* __restrict__ pieces, int64_t n) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[kStages];
    if (threadIdx.x != 0 || (int64_t)blockIdx.x >= n) return;
    PieceIter it;
    it.p = pieces;
    it.n = n;
    it.step = gridDim.x;
    it.i = (int64_t)blockIdx.x - it.step;
    it.left = 0;
    it.chunk = kChunk;
    bulk_stream<kStages, kChunk>(it, smem, bars);
}

// ------------------------------------------------------------- commit
constexpr int kCommitThreads = 1024;

// Phase A (this kernel, one CTA): live flags, Eq. 10 violations, CSR row
// pointers and free-list offsets; phase B writes the blocks (same kernel,
// after the scans).  live_flag is a scratch [max_requests] array.
static __global__ void __launch_bounds__(kCommitThreads, 1)
kvx_commit_kernel(const int32_t* __restrict__ req, const int64_t* __restrict__ kv, int32_t n,
                  const int32_t* __restrict__ dst_bt, const int64_t* __restrict__ synced_hi,
                  uint8_t* __restrict__ live_flag, int32_t max_requests, int32_t max_blocks,
                  int32_t block_tokens, int32_t* __restrict__ row_ptr,
                  int32_t* __restrict__ blocks, int32_t* __restrict__ free_list,
                  int64_t* __restrict__ out /* [0]=violations [1]=n_blocks [2]=n_free */,
                  int32_t* __restrict__ free_list_dev /* optional device copy (block-manager push) */,
                  const int32_t* __restrict__ err = nullptr /* plan-kernel error word -> out[3] */) {
    __shared__ unsigned long long s_viol;
    if (threadIdx.x == 0) s_viol = 0;
    for (int32_t r = threadIdx.x; r < max_requests; r += kCommitThreads) live_flag[r] = 0;
    __syncthreads();
    for (int32_t i = threadIdx.x; i < n; i += kCommitThreads) live_flag[req[i]] = 1;
    __syncthreads();
    const int64_t B = block_tokens;

    // Live rows: violation ballot + CSR of the allocated blocks.
    int2 carry = make_int2(0, 0);
    for (int32_t base = 0; base < n; base += kCommitThreads) {
        const int32_t i = base + (int32_t)threadIdx.x;
        int32_t nb = 0;
        bool bad = false;
        int32_t r = -1;
        if (i < n) {
            r = req[i];
            const int64_t s = synced_hi[r];
            bad = s != kv[i];  // engine.cpp:712
            nb = (int32_t)cdiv(s, B);
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, bad);
        if ((threadIdx.x & 31) == 0 && ballot) atomicAdd(&s_viol, (unsigned long long)__popc(ballot));
        int2 tot;
        const int2 off = block_exclusive_scan2<kCommitThreads>(make_int2(nb, 0), &tot);
        if (i < n) {
            const int32_t o = carry.x + off.x;
            if (row_ptr) row_ptr[i] = o;
            if (blocks)
                for (int32_t k = 0; k < nb; ++k) blocks[o + k] = dst_bt[(int64_t)r * max_blocks + k];
        }
        carry.x += tot.x;
    }
    if (threadIdx.x == 0 && row_ptr) row_ptr[n] = carry.x;
    const int32_t n_blocks = carry.x;

    // Dead rows (allocated but no longer live): ballot-compacted free list.
    carry = make_int2(0, 0);
    for (int32_t base = 0; base < max_requests; base += kCommitThreads) {
        const int32_t r = base + (int32_t)threadIdx.x;
        int32_t nb = 0;
        if (r < max_requests && !live_flag[r]) nb = (int32_t)cdiv(synced_hi[r], B);
        int2 tot;
        const int2 off = block_exclusive_scan2<kCommitThreads>(make_int2(nb, 0), &tot);
        if (nb > 0 && (free_list || free_list_dev))
            for (int32_t k = 0; k < nb; ++k) {
                const int32_t id = dst_bt[(int64_t)r * max_blocks + k];
                if (free_list) free_list[carry.x + off.x + k] = id;
                if (free_list_dev) free_list_dev[carry.x + off.x + k] = id;
            }
        carry.x += tot.x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        out[0] = (int64_t)s_viol;
        out[1] = n_blocks;
        out[2] = carry.x;
        out[3] = err ? (int64_t)*err : 0;
    }
}

// ---------------------------------------------------- payload kernels
// grid = (entries, max logical blocks); one CTA per (request, logical block),
// looping over the pool's layers and the block's K/V token rows.
// from == nullptr: tokens [0, tokens[i]); else [from[i], tokens[i]) (decode appends).
static __global__ void __launch_bounds__(256)
kvx_fill_kernel(PoolAddr pa, int32_t first_layer,
                int32_t num_layers, const int32_t* __restrict__ req,
                const int64_t* __restrict__ tokens, const int32_t* __restrict__ bt,
                int32_t max_blocks, int32_t block_tokens, uint64_t token_bytes, uint64_t seed,
                const int64_t* __restrict__ from = nullptr) {
    const int32_t i = blockIdx.x;
    const int32_t r = req[i];
    const uint32_t vecs = (uint32_t)(token_bytes >> 4);
    for (int32_t b = blockIdx.y; (int64_t)b * block_tokens < tokens[i]; b += gridDim.y) {  // grid.y <= 65535
        int64_t t_begin = (int64_t)b * block_tokens;
        const int64_t t_end = min(tokens[i], t_begin + block_tokens);
        if (from) {
            if (t_end <= from[i]) continue;
            t_begin = max(t_begin, from[i]);
        }
        const int32_t blk = bt[(int64_t)r * max_blocks + b];
        const int32_t rows = (int32_t)(t_end - t_begin);
        const int32_t row0 = (int32_t)(t_begin - (int64_t)b * block_tokens);  // first row inside the block
        for (int32_t l = 0; l < num_layers; ++l) {
            char* slab = pa.layer[l] + (uint64_t)blk * pa.blk_stride;
            for (int32_t kvr = 0; kvr < 2 * rows; ++kvr) {
                const int32_t kvi = kvr / rows, t = kvr % rows;
                const uint64_t th = token_hash(seed, r, first_layer + l, kvi, t_begin + t);
                char* row = slab + (uint64_t)kvi * pa.kv_stride + (uint64_t)(row0 + t) * pa.tok_stride;
                const uint32_t vph = pa.head_bytes >> 4;  // vector v of the token lies in head v / vph
                for (uint32_t v = threadIdx.x; v < vecs; v += blockDim.x)
                    *reinterpret_cast<uint4*>(row + (uint64_t)(v / vph) * pa.head_stride + (v % vph) * 16u) =
                        pattern_vec(th, v);
            }
        }
    }
}

static __global__ void __launch_bounds__(256)
kvx_verify_kernel(PoolAddr pa, int32_t first_layer,
                  int32_t num_layers, const int32_t* __restrict__ req,
                  const int64_t* __restrict__ tokens, const int32_t* __restrict__ bt,
                  int32_t max_blocks, int32_t block_tokens, uint64_t token_bytes, uint64_t seed,
                  unsigned long long* __restrict__ mismatches) {
    const int32_t i = blockIdx.x;
    const int32_t r = req[i];
    const uint32_t vecs = (uint32_t)(token_bytes >> 4);
    unsigned long long bad = 0;
    for (int32_t b = blockIdx.y; (int64_t)b * block_tokens < tokens[i]; b += gridDim.y) {  // grid.y <= 65535
        const int64_t t_begin = (int64_t)b * block_tokens;
        const int64_t t_end = min(tokens[i], t_begin + block_tokens);
        const int32_t blk = bt[(int64_t)r * max_blocks + b];
        const int32_t rows = (int32_t)(t_end - t_begin);
        if (blk < 0) {
            bad += threadIdx.x == 0 ? (unsigned long long)num_layers * 2 * rows * vecs * 8 : 0;
            continue;
        }
        for (int32_t l = 0; l < num_layers; ++l) {
            const char* slab = pa.layer[l] + (uint64_t)blk * pa.blk_stride;
            for (int32_t kvr = 0; kvr < 2 * rows; ++kvr) {
                const int32_t kvi = kvr / rows, t = kvr % rows;
                const uint64_t th = token_hash(seed, r, first_layer + l, kvi, t_begin + t);
                const char* row = slab + (uint64_t)kvi * pa.kv_stride + (uint64_t)t * pa.tok_stride;
                const uint32_t vph = pa.head_bytes >> 4;
                for (uint32_t v = threadIdx.x; v < vecs; v += blockDim.x) {
                    const uint4 want = pattern_vec(th, v);
                    const uint4 got =
                        *reinterpret_cast<const uint4*>(row + (uint64_t)(v / vph) * pa.head_stride + (v % vph) * 16u);
                    const uint32_t d[4] = {want.x ^ got.x, want.y ^ got.y, want.z ^ got.z, want.w ^ got.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) bad += ((d[q] & 0xffffu) != 0) + ((d[q] >> 16) != 0);
                }
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_down_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(mismatches, bad);
}

}  // namespace kvx
