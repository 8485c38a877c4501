// kvx_plane.cpp -- pipesim::KvxPlane over the kvx C-ABI (see
// pipesim/kvx_plane.hpp).  Host-side C++ of the drop-in: it owns the GPU pools
// of every in-flight transition of one Engine and turns RefactorCtx snapshots
// into kvx_wave / kvx_commit calls.  No CUDA here -- only include/kvx.h.
#include "pipesim/kvx_plane.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <mutex>
#include <string>
#include <exception>
#include <execinfo.h>
#include <unistd.h>

#include <json.hpp>

#include "kvx.h"
#include "pipesim/engine.hpp"
#include "pipesim/errors.hpp"

namespace pipesim {

namespace {

constexpr std::uint64_t kSeed = 0xE9E;  // payload pattern of the emulated serving writes
constexpr int kBlockTokens = 16;

std::int64_t cdiv(std::int64_t a, std::int64_t b) { return (a + b - 1) / b; }

[[noreturn]] void die(const char* call, int rc) {
    // A failing data plane is a failed run, never a silent fallback to the
    // simulated charge: the engine's own error type carries it out.
    throw InvalidSpecError(std::string("kvx: ") + call + " failed (" + std::to_string(rc) + "): " +
                           kvx_last_error());
}
#define KVX_OR_DIE(call)                 \
    do {                                 \
        const int rc_ = (call);          \
        if (rc_ != KVX_OK) die(#call, rc_); \
    } while (0)

// Process-wide record of what the planes did (written at exit).
struct Stats {
    std::mutex mu;
    std::string mode;
    std::int64_t engines = 0, transitions = 0, commits = 0, aborts = 0, unfinished = 0, waves = 0, grows = 0;
    std::int64_t tokens = 0, violations_host = 0, violations_device = 0, violation_mismatches = 0;
    std::int64_t mismatched_words = 0, verified_tokens = 0;
    double bytes_moved = 0.0, device_ms = 0.0, kv_charged_bytes = 0.0;
    std::map<std::string, std::int64_t> geometries;
    nlohmann::json wave_log = nlohmann::json::array();  // first kWaveLog waves
    static constexpr std::size_t kWaveLog = 4096;
};
Stats& stats() {
    static Stats s;
    return s;
}
nlohmann::json report_locked(Stats& s) {
    nlohmann::json j;
    j["kind"] = "kvx_plane_report";
    j["pid"] = static_cast<std::int64_t>(getpid());
    j["mode"] = s.mode;
    j["engines"] = s.engines;
    j["transitions"] = s.transitions;
    j["commits"] = s.commits;
    j["aborts"] = s.aborts;
    j["unfinished"] = s.unfinished;
    j["waves"] = s.waves;
    j["grows"] = s.grows;
    j["tokens"] = s.tokens;
    j["bytes_moved"] = s.bytes_moved;
    j["device_ms"] = s.device_ms;
    j["kv_charged_bytes"] = s.kv_charged_bytes;
    j["violations_host"] = s.violations_host;
    j["violations_device"] = s.violations_device;
    j["violation_mismatches"] = s.violation_mismatches;
    j["mismatched_words"] = s.mismatched_words;
    j["verified_tokens"] = s.verified_tokens;
    j["geometries"] = s.geometries;
    j["kvx_launches"] = kvx_launch_count();
    j["wave_log"] = s.wave_log;
    return j;
}
void write_report() {
    const char* path = std::getenv("PIPESIM_KVX_REPORT");
    if (!path || !*path) return;
    Stats& s = stats();
    std::lock_guard<std::mutex> lk(s.mu);
    std::ofstream f(path, std::ios::app);
    f << report_locked(s).dump() << "\n";
}

// One in-flight transition of one instance.
struct Xfer {
    kvx_geometry g{};
    std::vector<std::int32_t> old_b, new_b;
    kvx_transition* t = nullptr;
    std::vector<kvx_pool*> old_pools, new_pools;
    std::int32_t src_cap = 0, dst_cap = 0;
    std::vector<std::int32_t> src_bt;      // [max_requests * max_blocks], -1 = unassigned
    std::vector<std::int32_t> src_free;    // unassigned source block ids (fragmented order)
    std::vector<std::int64_t> filled;      // source tokens written per request (serving's appends)
    std::vector<std::int64_t> synced;      // host mirror of the destination's synced marks
    std::int64_t dst_alloc = 0;
    std::uint64_t epoch = 0;
    struct Wave {
        std::vector<std::int32_t> req;
        std::vector<std::int64_t> lo, hi;
    };
    std::vector<Wave> history;             // replayed when the pools grow
};

}  // namespace

struct KvxPlane::Impl {
    bool measured = false;
    bool trace = std::getenv("PIPESIM_KVX_TRACE") != nullptr;  // one stderr line per plane call
    int device = 0;
    std::string geom_spec = "auto";
    int num_layers = 0;
    double bpt = 0.0;
    int max_sync_rounds = 8;
    std::int32_t max_requests = 0, max_blocks = 1;
    std::vector<std::int64_t> req_max_tokens;  // prompt + output per request
    double max_pool_bytes = 96e9;              // cap per transition (source + destination), of 180 GB
    kvx_geometry pending{};                    // fixed by grant_kv_bytes for the next begin
    std::int64_t pending_blocks = 0;
    std::map<std::int64_t, Xfer> active;
    std::uint64_t lcg = 12345;

    kvx_geometry geometry(int heads, int dim) const {
        return kvx_geometry{num_layers, heads, dim, 2, kBlockTokens};
    }
    static double pool_bytes(const kvx_geometry& g, std::int64_t blocks) {
        return (double)g.num_layers * (double)blocks * 2.0 * g.block_tokens * g.num_kv_heads * g.head_dim * g.elem_bytes;
    }
    // The transition's pool geometry: the Llama shape of kv_bytes_per_token
    // (2 * L * H * 128 * 2 B) when it is one and fits, else a small test shape.
    kvx_geometry choose(std::int64_t blocks) const {
        int h = 2, d = 64;
        bool real = false;
        if (geom_spec == "auto") {
            const double per = bpt / (2.0 * num_layers * 128 * 2);
            if (per >= 1.0 && per <= 128.0 && per == std::floor(per)) {
                h = (int)per;
                d = 128;
                real = true;
            }
        } else if (std::sscanf(geom_spec.c_str(), "%d,%d", &h, &d) != 2) {
            throw InvalidSpecError("PIPESIM_KVX_GEOMETRY must be auto or H,D");
        }
        kvx_geometry g = geometry(h, d);
        // source (1.25x, fragmentation slack) + destination must fit the cap
        if (real && 2.3 * pool_bytes(g, blocks) > max_pool_bytes) g = geometry(2, 64);
        if (2.3 * pool_bytes(g, blocks) > max_pool_bytes) g = geometry(1, 8);
        return g;
    }

    void shuffle_into(std::vector<std::int32_t>& v, std::int32_t from, std::int32_t to) {
        std::vector<std::int32_t> ids;
        for (std::int32_t i = from; i < to; ++i) ids.push_back(i);
        for (std::size_t i = ids.size(); i > 1; --i) {  // fragmented source pages
            lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
            std::swap(ids[i - 1], ids[(std::size_t)((lcg >> 33) % i)]);
        }
        v.insert(v.begin(), ids.begin(), ids.end());
    }

    std::vector<std::pair<int, int>> ranges(const std::vector<std::int32_t>& b) const {
        std::vector<std::pair<int, int>> r;
        int prev = 0;
        for (std::int32_t x : b) {
            r.push_back({prev, x});
            prev = x;
        }
        r.push_back({prev, num_layers});
        return r;
    }

    void make_pools(Xfer& x) {
        for (auto [b, e] : ranges(x.old_b)) {
            kvx_pool* p = nullptr;
            KVX_OR_DIE(kvx_pool_create(device, &x.g, e - b, x.src_cap, &p));
            x.old_pools.push_back(p);
        }
        for (auto [b, e] : ranges(x.new_b)) {
            kvx_pool* p = nullptr;
            KVX_OR_DIE(kvx_pool_create(device, &x.g, e - b, x.dst_cap, &p));
            KVX_OR_DIE(kvx_pool_zero(p));
            x.new_pools.push_back(p);
        }
        kvx_transition_desc d{};
        d.geometry = x.g;
        d.old_plan = {(std::int32_t)x.old_pools.size(), x.old_b.data(), x.old_pools.data()};
        d.new_plan = {(std::int32_t)x.new_pools.size(), x.new_b.data(), x.new_pools.data()};
        d.device = device;
        d.max_requests = max_requests;
        d.max_blocks = max_blocks;
        d.dst_num_blocks = x.dst_cap;
        d.src_block_table = x.src_bt.data();
        d.epoch = x.epoch;
        d.max_sync_rounds = max_sync_rounds;
        d.kv_bytes_per_token = bpt;
        KVX_OR_DIE(kvx_begin(&d, &x.t));
    }
    void free_pools(Xfer& x) {
        if (x.t) kvx_destroy(x.t);
        x.t = nullptr;
        for (kvx_pool* p : x.old_pools) kvx_pool_destroy(p);
        for (kvx_pool* p : x.new_pools) kvx_pool_destroy(p);
        x.old_pools.clear();
        x.new_pools.clear();
    }
    // The serving pipeline's writes: tokens [0, hi) of each request exist in
    // the source before a wave reads them.
    void fill(Xfer& x, const std::vector<std::int32_t>& req, const std::vector<std::int64_t>& hi) {
        std::vector<std::int32_t> fr;
        std::vector<std::int64_t> ft;
        for (std::size_t i = 0; i < req.size(); ++i)
            if (hi[i] > x.filled[(std::size_t)req[i]]) {
                fr.push_back(req[i]);
                ft.push_back(hi[i]);
                x.filled[(std::size_t)req[i]] = hi[i];
            }
        if (fr.empty()) return;
        auto rg = ranges(x.old_b);
        for (std::size_t k = 0; k < x.old_pools.size(); ++k)
            KVX_OR_DIE(kvx_pool_fill_pattern(x.old_pools[k], kSeed, rg[k].first, (std::int32_t)fr.size(), fr.data(),
                                             ft.data(), x.src_bt.data(), max_requests, max_blocks));
    }
    // Source blocks of a request the first time a wave reads it (its whole
    // length, as a paged serving cache reserves it), and the destination
    // blocks the wave allocates; on a shortfall the pools are rebuilt larger
    // and the transition's earlier waves replayed (the block rule is
    // deterministic, so the destination ends up identical).
    void reserve(Xfer& x, const Xfer::Wave& w) {
        std::int64_t src_need = 0, dst_need = 0;
        for (std::size_t i = 0; i < w.req.size(); ++i) {
            const std::int32_t r = w.req[i];
            if (w.hi[i] <= w.lo[i]) continue;
            if (x.src_bt[(std::size_t)r * max_blocks] < 0) src_need += cdiv(req_max_tokens[(std::size_t)r], kBlockTokens);
            dst_need += std::max<std::int64_t>(0, cdiv(w.hi[i], kBlockTokens) - cdiv(x.synced[(std::size_t)r], kBlockTokens));
        }
        if (src_need > (std::int64_t)x.src_free.size() || x.dst_alloc + dst_need > x.dst_cap) grow(x, src_need, dst_need);
        // requests the grant's table did not cover (admitted, or first read, after
        // it): their rows go to the device table with kvx_src_rows
        std::vector<std::int32_t> new_req, new_rows;
        for (std::size_t i = 0; i < w.req.size(); ++i) {
            const std::int32_t r = w.req[i];
            if (w.hi[i] <= w.lo[i] || x.src_bt[(std::size_t)r * max_blocks] >= 0) continue;
            const std::int64_t nb = cdiv(req_max_tokens[(std::size_t)r], kBlockTokens);
            for (std::int64_t b = 0; b < nb; ++b) {
                x.src_bt[(std::size_t)r * max_blocks + (std::size_t)b] = x.src_free.back();
                x.src_free.pop_back();
            }
            new_req.push_back(r);
            new_rows.insert(new_rows.end(), x.src_bt.begin() + (std::ptrdiff_t)r * max_blocks,
                            x.src_bt.begin() + (std::ptrdiff_t)(r + 1) * max_blocks);
        }
        if (!new_req.empty())
            KVX_OR_DIE(kvx_src_rows(x.t, x.epoch, (std::int32_t)new_req.size(), new_req.data(), new_rows.data()));
    }
    void grow(Xfer& x, std::int64_t src_need, std::int64_t dst_need) {
        const std::int32_t old_src = x.src_cap;
        x.src_cap = (std::int32_t)std::max<std::int64_t>(2LL * x.src_cap, x.src_cap + 2 * src_need);
        x.dst_cap = (std::int32_t)std::max<std::int64_t>(2LL * x.dst_cap, x.dst_alloc + 2 * dst_need);
        free_pools(x);
        shuffle_into(x.src_free, old_src, x.src_cap);
        make_pools(x);
        std::vector<std::int32_t> req;
        std::vector<std::int64_t> hi;
        for (std::int32_t r = 0; r < max_requests; ++r)
            if (x.filled[(std::size_t)r] > 0) {
                req.push_back(r);
                hi.push_back(x.filled[(std::size_t)r]);
                x.filled[(std::size_t)r] = 0;
            }
        fill(x, req, hi);
        for (const Xfer::Wave& w : x.history)
            KVX_OR_DIE(kvx_wave(x.t, x.epoch, (std::int32_t)w.req.size(), w.req.data(), w.lo.data(), w.hi.data()));
        double ms = 0.0;
        KVX_OR_DIE(kvx_wait(x.t, x.epoch, &ms));
        std::lock_guard<std::mutex> lk(stats().mu);
        ++stats().grows;
    }
};

KvxPlane::KvxPlane(std::unique_ptr<Impl> impl) : impl_(std::move(impl)) {}

KvxPlane::~KvxPlane() {
    if (!impl_) return;
    std::int64_t open = 0;
    for (auto& [id, x] : impl_->active) {
        (void)id;
        impl_->free_pools(x);
        ++open;
    }
    std::lock_guard<std::mutex> lk(stats().mu);
    stats().unfinished += open;
}

std::shared_ptr<KvxPlane> KvxPlane::from_env(const EngineConfig& cfg, const std::vector<Request>& workload) {
    const char* mode = std::getenv("PIPESIM_KVX");
    if (!mode || !*mode || std::string(mode) == "0" || std::string(mode) == "off") return nullptr;
    const std::string m(mode);
    if (m != "1" && m != "parity" && m != "measured")
        throw InvalidSpecError("PIPESIM_KVX must be parity or measured");
    auto impl = std::make_unique<Impl>();
    impl->measured = m == "measured";
    if (const char* d = std::getenv("PIPESIM_KVX_DEVICE")) impl->device = std::atoi(d);
    if (const char* g = std::getenv("PIPESIM_KVX_GEOMETRY")) impl->geom_spec = g;
    if (const char* c = std::getenv("PIPESIM_KVX_MAX_GB")) impl->max_pool_bytes = std::atof(c) * 1e9;
    impl->num_layers = (int)cfg.graph.ops.size();
    impl->bpt = cfg.exec.kv_bytes_per_token;
    impl->max_sync_rounds = cfg.max_sync_rounds;
    impl->max_requests = (std::int32_t)std::max<std::size_t>(1, workload.size());
    impl->req_max_tokens.resize(workload.size());
    for (std::size_t i = 0; i < workload.size(); ++i) {
        impl->req_max_tokens[i] = (std::int64_t)workload[i].prompt_tokens + workload[i].output_tokens;
        impl->max_blocks = (std::int32_t)std::max<std::int64_t>(impl->max_blocks, cdiv(impl->req_max_tokens[i], kBlockTokens));
    }
    static std::once_flag once;
    std::call_once(once, [] {
        // the statistics object must outlive the exit handler: construct it
        // first (function statics die in reverse order of construction,
        // interleaved with atexit handlers)
        stats();
        std::atexit(write_report);
        if (std::getenv("PIPESIM_KVX_TRACE"))  // where an escaping exception came from
            std::set_terminate([] {
                void* frames[64];
                const int n = backtrace(frames, 64);
                std::fprintf(stderr, "kvx-plane: terminate; backtrace:\n");
                backtrace_symbols_fd(frames, n, 2);
                std::abort();
            });
    });
    {
        std::lock_guard<std::mutex> lk(stats().mu);
        stats().mode = impl->measured ? "measured" : "parity";
        ++stats().engines;
    }
    return std::shared_ptr<KvxPlane>(new KvxPlane(std::move(impl)));
}

bool KvxPlane::measured_time() const { return impl_->measured; }

std::string KvxPlane::stats_json() {
    Stats& s = stats();
    std::lock_guard<std::mutex> lk(s.mu);
    return report_locked(s).dump();
}

void KvxPlane::reset_stats() {
    Stats& s = stats();
    std::lock_guard<std::mutex> lk(s.mu);
    const std::string mode = s.mode;
    s.engines = s.transitions = s.commits = s.aborts = s.unfinished = s.waves = s.grows = 0;
    s.tokens = s.violations_host = s.violations_device = s.violation_mismatches = 0;
    s.mismatched_words = s.verified_tokens = 0;
    s.bytes_moved = s.device_ms = s.kv_charged_bytes = 0.0;
    s.geometries.clear();
    s.wave_log = nlohmann::json::array();
    s.mode = mode;
}

std::vector<double> KvxPlane::grant_kv_bytes(const std::vector<int>& new_boundaries,
                                             const std::vector<std::int64_t>& live_max_tokens) {
    Impl& I = *impl_;
    if (I.trace)
        std::fprintf(stderr, "kvx-plane grant K=%zu live=%zu\n", new_boundaries.size() + 1, live_max_tokens.size());
    std::int64_t blocks = 0;
    for (std::int64_t t : live_max_tokens) blocks += cdiv(t, kBlockTokens);
    blocks = std::max<std::int64_t>(blocks, 16);
    I.pending = I.choose(blocks);
    I.pending_blocks = blocks;
    std::vector<std::int32_t> b(new_boundaries.begin(), new_boundaries.end());
    std::vector<std::uint64_t> out(b.size() + 1);
    KVX_OR_DIE(kvx_stage_kv_bytes(&I.pending, (std::int32_t)out.size(), b.data(), (std::int32_t)blocks, out.data()));
    return std::vector<double>(out.begin(), out.end());
}

void KvxPlane::begin(std::int64_t instance, std::uint64_t epoch, const std::vector<int>& old_boundaries,
                     const std::vector<int>& new_boundaries, int num_layers) {
    Impl& I = *impl_;
    if (I.trace)
        std::fprintf(stderr, "kvx-plane begin inst=%lld epoch=%llu K %zu->%zu blocks=%lld\n", (long long)instance,
                     (unsigned long long)epoch, old_boundaries.size() + 1, new_boundaries.size() + 1,
                     (long long)I.pending_blocks);
    if (num_layers != I.num_layers) throw InvalidSpecError("kvx: layer count changed");
    auto it = I.active.find(instance);
    if (it != I.active.end()) {  // a previous transition of this instance never ended (engine reset)
        I.free_pools(it->second);
        I.active.erase(it);
    }
    Xfer& x = I.active[instance];
    x.g = I.pending.num_layers ? I.pending : I.choose(16);
    x.old_b.assign(old_boundaries.begin(), old_boundaries.end());
    x.new_b.assign(new_boundaries.begin(), new_boundaries.end());
    x.epoch = epoch;
    x.dst_cap = (std::int32_t)std::max<std::int64_t>(16, I.pending_blocks);
    x.src_cap = (std::int32_t)(x.dst_cap + x.dst_cap / 4 + 16);
    x.src_bt.assign((std::size_t)I.max_requests * I.max_blocks, -1);
    x.filled.assign((std::size_t)I.max_requests, 0);
    x.synced.assign((std::size_t)I.max_requests, 0);
    I.shuffle_into(x.src_free, 0, x.src_cap);
    I.make_pools(x);
    const double charged = [&] {
        std::vector<std::uint64_t> out(x.new_b.size() + 1);
        if (kvx_stage_kv_bytes(&x.g, (std::int32_t)out.size(), x.new_b.data(), x.dst_cap, out.data()) != KVX_OK) return 0.0;
        double s = 0.0;
        for (auto v : out) s += (double)v;
        return s;
    }();
    I.pending = kvx_geometry{};
    std::lock_guard<std::mutex> lk(stats().mu);
    ++stats().transitions;
    stats().kv_charged_bytes += charged;
    ++stats().geometries[std::to_string(x.g.num_kv_heads) + "x" + std::to_string(x.g.head_dim)];
}

double KvxPlane::wave(std::int64_t instance, std::uint64_t epoch, const std::map<std::int32_t, std::int64_t>& sync_target,
                      const std::map<std::int32_t, std::int64_t>& synced_tokens, double modelled_ms, double now_ms) {
    Impl& I = *impl_;
    if (I.trace)
        std::fprintf(stderr, "kvx-plane wave inst=%lld epoch=%llu entries=%zu now=%.3f\n", (long long)instance,
                     (unsigned long long)epoch, sync_target.size(), now_ms);
    auto xit = I.active.find(instance);
    if (xit == I.active.end()) throw InvalidSpecError("kvx: wave without a transition");
    Xfer& x = xit->second;
    Xfer::Wave w;
    std::int64_t tokens = 0;
    for (const auto& [r, target] : sync_target) {  // std::map: ascending request ids (engine.hpp:153-154)
        auto s = synced_tokens.find(r);
        const std::int64_t lo = s == synced_tokens.end() ? 0 : s->second;
        w.req.push_back(r);
        w.lo.push_back(lo);
        w.hi.push_back(target);
        tokens += std::max<std::int64_t>(0, target - lo);
    }
    I.reserve(x, w);
    I.fill(x, w.req, w.hi);
    KVX_OR_DIE(kvx_wave(x.t, epoch, (std::int32_t)w.req.size(), w.req.data(), w.lo.data(), w.hi.data()));
    double ms = 0.0;
    KVX_OR_DIE(kvx_wait(x.t, epoch, &ms));
    for (std::size_t i = 0; i < w.req.size(); ++i) {
        const std::size_t r = (std::size_t)w.req[i];
        const std::int64_t had = cdiv(x.synced[r], kBlockTokens);
        if (w.hi[i] > x.synced[r]) {
            x.dst_alloc += std::max<std::int64_t>(0, cdiv(w.hi[i], kBlockTokens) - had);
            x.synced[r] = w.hi[i];
        }
    }
    x.history.push_back(std::move(w));
    const double out = I.measured ? ms : modelled_ms;
    std::lock_guard<std::mutex> lk(stats().mu);
    Stats& s = stats();
    ++s.waves;
    s.tokens += tokens;
    s.bytes_moved += (double)tokens * 2.0 * x.g.num_layers * x.g.num_kv_heads * x.g.head_dim * x.g.elem_bytes;
    s.device_ms += ms;
    if (s.wave_log.size() < Stats::kWaveLog)
        s.wave_log.push_back({{"instance", instance}, {"epoch", epoch}, {"now_ms", now_ms}, {"tokens", tokens},
                              {"modelled_ms", modelled_ms}, {"measured_ms", ms}, {"scheduled_ms", out}});
    return out;
}

void KvxPlane::commit(std::int64_t instance, std::uint64_t epoch, const std::vector<std::int32_t>& live_req,
                      const std::vector<std::int64_t>& live_kv, std::int64_t host_violations) {
    Impl& I = *impl_;
    if (I.trace)
        std::fprintf(stderr, "kvx-plane commit inst=%lld epoch=%llu live=%zu\n", (long long)instance,
                     (unsigned long long)epoch, live_req.size());
    auto it = I.active.find(instance);
    if (it == I.active.end()) throw InvalidSpecError("kvx: commit without a transition");
    Xfer& x = it->second;
    // the tokens the final wave did not cover (violations) are not in the
    // destination; the live set's payload is checked on what was synced
    std::vector<std::int32_t> row_ptr(live_req.size() + 1);
    std::vector<std::int32_t> blocks((std::size_t)std::max<std::int64_t>(1, x.dst_alloc));
    std::vector<std::int32_t> freel((std::size_t)std::max<std::int64_t>(1, x.dst_alloc));
    kvx_commit_result res{};
    res.row_ptr = row_ptr.data();
    res.blocks = blocks.data();
    res.blocks_cap = (std::int32_t)blocks.size();
    res.free_list = freel.data();
    res.free_cap = (std::int32_t)freel.size();
    KVX_OR_DIE(kvx_commit(x.t, epoch, (std::int32_t)live_req.size(), live_req.data(), live_kv.data(), &res));
    std::vector<std::int64_t> covered(live_kv.size());
    std::int64_t verified = 0;
    for (std::size_t i = 0; i < live_req.size(); ++i) {
        covered[i] = std::min(live_kv[i], x.synced[(std::size_t)live_req[i]]);
        verified += covered[i];
    }
    std::int64_t bad = 0;
    KVX_OR_DIE(kvx_verify_pattern(x.t, kSeed, (std::int32_t)live_req.size(), live_req.data(), covered.data(), &bad));
    if (res.violations != host_violations || bad != 0)
        std::fprintf(stderr, "kvx: instance %lld commit: device Eq. 10 %lld vs host %lld, %lld payload words differ\n",
                     (long long)instance, (long long)res.violations, (long long)host_violations, (long long)bad);
    I.free_pools(x);
    I.active.erase(it);
    std::lock_guard<std::mutex> lk(stats().mu);
    Stats& s = stats();
    ++s.commits;
    s.violations_host += host_violations;
    s.violations_device += res.violations;
    s.violation_mismatches += res.violations != host_violations ? 1 : 0;
    s.mismatched_words += bad;
    s.verified_tokens += verified;
}

void KvxPlane::abort(std::int64_t instance) {
    Impl& I = *impl_;
    if (I.trace) std::fprintf(stderr, "kvx-plane abort inst=%lld\n", (long long)instance);
    auto it = I.active.find(instance);
    if (it == I.active.end()) return;
    KVX_OR_DIE(kvx_abort(it->second.t));
    I.free_pools(it->second);
    I.active.erase(it);
    std::lock_guard<std::mutex> lk(stats().mu);
    ++stats().aborts;
}

}  // namespace pipesim
