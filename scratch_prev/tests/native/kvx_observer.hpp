// kvx_observer.hpp -- the reference engine driving the B200 data plane
// (TEST INFRASTRUCTURE shared by engine_kvx.cpp and test_kvx_engine.cpp).
//
// An observer attached through the reference's public trace hook
// (engine.hpp:119) calls the kvx C-ABI exactly where the UNMODIFIED engine
// charges simulated KV movement:
//   new RefactorCtx + wave 0   (engine.cpp:633-647)  -> kvx_begin + kvx_wave
//   delta wave                 (engine.cpp:665-674)  -> kvx_wave
//   final wave                 (engine.cpp:680-687)  -> kvx_wave
//   RefactorCommit             (engine.cpp:697-713)  -> kvx_commit (Eq. 10 on device)
//   abort_refactor             (engine.cpp:759-772)  -> kvx_abort
// RefactorCtx is read through `private`->`public` in the including TU (see
// extract_waves.cpp); the serving pipeline's decode appends are emulated by
// writing the payload before any wave reads it (engine.cpp:494-499).
#pragma once

#include <any>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <queue>
#include <string>
#include <vector>

#include <json.hpp>

#include "pipesim/cluster.hpp"
#include "pipesim/controller.hpp"
#include "pipesim/metrics.hpp"
#include "pipesim/modelgraph.hpp"
#include "pipesim/workload.hpp"

#define private public
#include "pipesim/engine.hpp"
#undef private

#include "kvx.h"
#include "scenarios.hpp"  // oracle/scenarios.hpp

using namespace pipesim;
using json = nlohmann::json;


namespace kvxobs {

using namespace pipesim;
using json = nlohmann::json;


constexpr uint64_t kSeed = 0xE9E;

#define CHECK_KVX(call)                                                                     \
    do {                                                                                    \
        int rc_ = (call);                                                                   \
        if (rc_ != KVX_OK) {                                                                \
            std::fprintf(stderr, "%s failed: %d %s\n", #call, rc_, kvx_last_error());       \
            std::exit(2);                                                                   \
        }                                                                                   \
    } while (0)

struct Live {
    std::vector<int32_t> req;
    std::vector<int64_t> kv;
};

struct Xfer {  // one transition's data-plane state
    kvx_transition* t = nullptr;
    std::vector<kvx_pool*> old_pools, new_pools;
    std::vector<int32_t> old_b, new_b;
    std::vector<int64_t> filled;  // source tokens written per request
    uint64_t epoch = 0;
    int rounds = -1;
    bool commit_scheduled = false;
    int waves = 0;
    int64_t tokens = 0;
    Live commit_live;
    bool have_commit_live = false;
    json wave_times = json::array();
};

struct Observer {
    Engine* e = nullptr;
    kvx_geometry g{};
    int32_t max_requests = 0, max_blocks = 0, src_blocks = 0, dst_blocks = 0;
    std::vector<int32_t> src_bt;  // fragmented source block table
    std::map<int64_t, Xfer> active;
    int64_t commits = 0, aborts = 0, violations_ref = 0;
    int64_t dev_violations = 0, mismatched_words = 0, transitions = 0;
    double measured_ms = 0.0, measured_bytes = 0.0;  // KV waves on the GPU (reference-accounted bytes)
    std::vector<json> lines;
    bool print_lines = true;
    int64_t tokens_moved = 0;

    std::vector<int32_t> bounds(int plan) {
        return e->cfg_.granularities.plans[(size_t)plan].plan.boundaries;
    }
    std::vector<std::pair<int, int>> ranges(const std::vector<int32_t>& b) {
        std::vector<std::pair<int, int>> r;
        int prev = 0;
        for (int32_t x : b) {
            r.push_back({prev, x});
            prev = x;
        }
        r.push_back({prev, g.num_layers});
        return r;
    }

    void fill_source(Xfer& x, const std::vector<int32_t>& req, const std::vector<int64_t>& hi) {
        std::vector<int32_t> fr;
        std::vector<int64_t> ft;
        for (size_t i = 0; i < req.size(); ++i)
            if (hi[i] > x.filled[(size_t)req[i]]) {
                fr.push_back(req[i]);
                ft.push_back(hi[i]);
                x.filled[(size_t)req[i]] = hi[i];
            }
        if (fr.empty()) return;
        auto rg = ranges(x.old_b);
        for (size_t k = 0; k < x.old_pools.size(); ++k)
            CHECK_KVX(kvx_pool_fill_pattern(x.old_pools[k], kSeed, rg[k].first, (int32_t)fr.size(),
                                            fr.data(), ft.data(), src_bt.data(), max_requests,
                                            max_blocks));
    }

    void begin(int64_t id, Engine::InstanceRt& inst) {
        Xfer x;
        x.epoch = inst.epoch;
        x.old_b = bounds(inst.plan_index);
        x.new_b = bounds(inst.refactor->target_plan);
        x.filled.assign((size_t)max_requests, 0);
        for (auto [b, en] : ranges(x.old_b)) {
            kvx_pool* p = nullptr;
            CHECK_KVX(kvx_pool_create(0, &g, en - b, src_blocks, &p));
            CHECK_KVX(kvx_pool_zero(p));
            x.old_pools.push_back(p);
        }
        for (auto [b, en] : ranges(x.new_b)) {
            kvx_pool* p = nullptr;
            CHECK_KVX(kvx_pool_create(0, &g, en - b, dst_blocks, &p));
            CHECK_KVX(kvx_pool_zero(p));
            x.new_pools.push_back(p);
        }
        kvx_transition_desc d{};
        d.geometry = g;
        d.old_plan = {(int32_t)x.old_pools.size(), x.old_b.data(), x.old_pools.data()};
        d.new_plan = {(int32_t)x.new_pools.size(), x.new_b.data(), x.new_pools.data()};
        d.device = 0;
        d.max_requests = max_requests;
        d.max_blocks = max_blocks;
        d.dst_num_blocks = dst_blocks;
        d.src_block_table = src_bt.data();
        d.epoch = inst.epoch;
        d.max_sync_rounds = e->cfg_.max_sync_rounds;
        d.kv_bytes_per_token = e->cfg_.exec.kv_bytes_per_token;
        CHECK_KVX(kvx_begin(&d, &x.t));
        active.emplace(id, std::move(x));
    }

    void wave(Xfer& x, const Engine::RefactorCtx& ctx) {
        std::vector<int32_t> req;
        std::vector<int64_t> lo, hi;
        for (const auto& [r, target] : ctx.sync_target) {  // std::map: ascending request ids
            auto it = ctx.synced_tokens.find(r);
            req.push_back(r);
            lo.push_back(it == ctx.synced_tokens.end() ? 0 : it->second);
            hi.push_back(target);
            x.tokens += std::max<int64_t>(0, target - lo.back());
        }
        fill_source(x, req, hi);  // decode appends of the serving pipeline
        int64_t tok = 0;
        for (size_t i = 0; i < req.size(); ++i) tok += std::max<int64_t>(0, hi[i] - lo[i]);
        CHECK_KVX(kvx_wave(x.t, x.epoch, (int32_t)req.size(), req.data(), lo.data(), hi.data()));
        // measured-time mode: the B200 time of this wave beside the reference's
        // modelled sync_ms = tokens * kv_bytes_per_token / kv_bw() (engine.cpp:644,670,683)
        double ms = 0.0;
        CHECK_KVX(kvx_wait(x.t, x.epoch, &ms));
        const double bw = e->cfg_.kv_sync_bw_bytes_per_ms > 0.0 ? e->cfg_.kv_sync_bw_bytes_per_ms
                                                                : e->cfg_.inter_stage_bw_bytes_per_ms;
        if (tok > 0) {
            measured_ms += ms;
            measured_bytes += (double)tok * e->cfg_.exec.kv_bytes_per_token;
        }
        json w;
        w["tokens"] = tok;
        w["modelled_ms"] = (double)tok * e->cfg_.exec.kv_bytes_per_token / bw;
        w["measured_ms"] = ms;
        x.wave_times.push_back(w);
        ++x.waves;
    }

    void end(int64_t id, bool committed, int64_t ref_violations) {
        Xfer& x = active.at(id);
        json j;
        j["instance"] = id;
        j["waves"] = x.waves;
        j["tokens"] = x.tokens;
        j["old_stages"] = x.old_pools.size();
        j["new_stages"] = x.new_pools.size();
        j["wave_times"] = x.wave_times;
        if (committed) {
            if (!x.have_commit_live) {
                std::fprintf(stderr, "commit without a captured live set\n");
                std::exit(3);
            }
            Live& lv = x.commit_live;
            std::vector<int32_t> row_ptr(lv.req.size() + 1);
            std::vector<int32_t> blocks((size_t)max_requests * max_blocks + 1);
            std::vector<int32_t> freel((size_t)max_requests * max_blocks + 1);
            kvx_commit_result res{};
            res.row_ptr = row_ptr.data();
            res.blocks = blocks.data();
            res.blocks_cap = (int32_t)blocks.size();
            res.free_list = freel.data();
            res.free_cap = (int32_t)freel.size();
            CHECK_KVX(kvx_commit(x.t, x.epoch, (int32_t)lv.req.size(), lv.req.data(), lv.kv.data(), &res));
            int64_t bad = 0;
            CHECK_KVX(kvx_verify_pattern(x.t, kSeed, (int32_t)lv.req.size(), lv.req.data(), lv.kv.data(), &bad));
            j["kind"] = "commit";
            j["violations_device"] = res.violations;
            j["violations_reference"] = ref_violations;
            j["mismatched_words"] = bad;
            j["live"] = lv.req.size();
            j["blocks"] = res.n_blocks;
            j["freed"] = res.n_free;
            dev_violations += res.violations;
            mismatched_words += bad;
            if (res.violations != ref_violations) {
                std::fprintf(stderr, "Eq. 10 disagreement: device %lld reference %lld\n",
                             (long long)res.violations, (long long)ref_violations);
                std::exit(4);
            }
        } else {
            CHECK_KVX(kvx_abort(x.t));
            uint64_t ep = 0;
            CHECK_KVX(kvx_epoch(x.t, &ep));
            j["kind"] = "abort";
            j["epoch_after"] = ep;
        }
        if (print_lines) std::printf("%s\n", j.dump().c_str());
        lines.push_back(j);
        tokens_moved += x.tokens;
        kvx_destroy(x.t);
        for (kvx_pool* p : x.old_pools) kvx_pool_destroy(p);
        for (kvx_pool* p : x.new_pools) kvx_pool_destroy(p);
        active.erase(id);
        ++transitions;
    }

    void observe() {
        const EngineResult& res = e->result_;
        for (const auto& ip : e->instances_) {
            auto& inst = *ip;
            auto it = active.find(inst.id);
            if (it != active.end() && (!inst.refactor || inst.epoch != it->second.epoch)) {
                const bool committed = res.refactor_commits > commits;
                const int64_t dv = res.kv_violations - violations_ref;
                commits = res.refactor_commits;
                aborts = res.refactor_aborts;
                violations_ref = res.kv_violations;
                end(inst.id, committed, dv);
                it = active.end();
            }
            if (!inst.refactor) continue;
            if (it == active.end()) {
                begin(inst.id, inst);
                it = active.find(inst.id);
            }
            Xfer& x = it->second;
            const auto& ctx = *inst.refactor;
            if (ctx.rounds != x.rounds || ctx.commit_scheduled != x.commit_scheduled) {
                x.rounds = ctx.rounds;
                x.commit_scheduled = ctx.commit_scheduled;
                wave(x, ctx);
            }
        }
    }

    void before(const SimEvent& ev) {
        observe();
        if (ev.kind != EventKind::RefactorCommit) return;
        auto& inst = *e->instances_[(size_t)ev.instance_id];
        if (inst.state != Engine::InstState::Refactoring || !inst.refactor) return;
        if (ev.aux != (int64_t)inst.epoch) return;
        Xfer& x = active.at(inst.id);
        x.commit_live = {};
        for (size_t i = 0; i < e->reqs_.size(); ++i) {
            const auto& rt = e->reqs_[i];
            if (rt.done || rt.home != inst.id) continue;
            x.commit_live.req.push_back((int32_t)i);
            x.commit_live.kv.push_back(rt.kv_tokens);
        }
        // the final wave's tokens exist in the source before the data plane commits
        fill_source(x, x.commit_live.req, x.commit_live.kv);
        x.have_commit_live = true;
    }
};

// Barrier -> commit stall per transition of a plain engine run (no data
// plane), read through the same trace hook: the barrier is the handler that
// sets RefactorCtx::barrier (engine.cpp:676), the commit the RefactorCommit
// dispatch that ends the ctx (engine.cpp:690-757).
struct StallProbe {
    Engine* e = nullptr;
    std::map<int64_t, double> barrier_at;
    std::map<int64_t, bool> had_ctx;
    std::vector<double> stalls;
    double prev_ms = 0.0, commit_ev_ms = -1.0;
    void before(const SimEvent& ev) {
        for (const auto& ip : e->instances_) {
            auto& inst = *ip;
            if (inst.refactor && inst.refactor->barrier && !barrier_at.count(inst.id)) barrier_at[inst.id] = prev_ms;
            if (!inst.refactor && had_ctx[inst.id] && barrier_at.count(inst.id)) {
                if (commit_ev_ms >= 0) stalls.push_back(commit_ev_ms - barrier_at[inst.id]);
                barrier_at.erase(inst.id);
            }
            had_ctx[inst.id] = (bool)inst.refactor;
        }
        if (ev.kind == EventKind::RefactorCommit) commit_ev_ms = ev.time_ms;
        prev_ms = ev.time_ms;
    }
};

inline json plain_run(const scen::Scenario& sc, double kv_bw) {
    scen::Built b = scen::build(sc);
    b.ec.kv_sync_bw_bytes_per_ms = kv_bw;
    Engine engine(b.ec, b.cluster, sc.reqs);
    for (auto [t, k] : sc.forced) engine.force_refactor_at(t, "m0", k);
    for (double t : sc.revocations) engine.revoke_grant_at(t, "m0");
    StallProbe pr;
    pr.e = &engine;
    engine.set_trace_sink([&pr](const SimEvent& ev) { pr.before(ev); });
    EngineResult r = engine.run();
    pr.before(SimEvent{engine.now_ms_, 0, EventKind::Arrival, -1, -1, -1, -1});
    double lat = 0.0;
    for (const auto& rec : r.records) lat += rec.finish_ms - rec.arrival_ms;
    json j;
    j["kv_sync_bw_bytes_per_ms"] = kv_bw;
    j["stall_ms"] = pr.stalls;
    j["mean_latency_ms"] = r.records.empty() ? 0.0 : lat / (double)r.records.size();
    j["duration_ms"] = r.duration_ms;
    j["refactor_commits"] = r.refactor_commits;
    return j;
}

inline std::vector<Request> steady(int n, double gap, int prompt, int output) {
    std::vector<Request> v;
    for (int i = 0; i < n; ++i) {
        Request r;
        r.id = i;
        r.arrival_ms = gap * (i + 1);
        r.prompt_tokens = prompt;
        r.output_tokens = output;
        r.model_id = "m0";
        r.slo_deadline_ms = 1.0e9;
        v.push_back(r);
    }
    return v;
}


// Runs one scenario through the unmodified engine with the kvx data plane
// attached (the body of engine_kvx's main, reused by test_kvx_engine.cpp).
struct RunOut {
    EngineResult res;
    std::unique_ptr<Observer> obs;
};

inline RunOut run_with_kvx(const scen::Scenario& sc, int heads, int dim, bool print_lines,
                           bool with_refactors = true) {
    scen::Built built = scen::build(sc);
    const std::vector<Request>& reqs = sc.reqs;
    Engine engine(built.ec, built.cluster, reqs);
    if (with_refactors) {
        for (auto [t, k] : sc.forced) engine.force_refactor_at(t, "m0", k);
        for (double t : sc.revocations) engine.revoke_grant_at(t, "m0");
    }
    RunOut out;
    out.obs = std::make_unique<Observer>();
    Observer& obs = *out.obs;
    obs.print_lines = print_lines;
    obs.e = &engine;
    obs.g = kvx_geometry{sc.num_ops, heads, dim, 2, 16};
    obs.max_requests = (int32_t)reqs.size();
    int32_t total = 0;
    for (const auto& r : reqs) {
        obs.max_blocks = std::max(obs.max_blocks, (r.prompt_tokens + r.output_tokens + 15) / 16);
        total += (r.prompt_tokens + r.output_tokens + 15) / 16;
    }
    obs.src_blocks = total + total / 4 + 1;
    obs.dst_blocks = total;
    // Fragmented source pages: a fixed pseudo-random permutation of the pool.
    std::vector<int32_t> perm((size_t)obs.src_blocks);
    for (int32_t i = 0; i < obs.src_blocks; ++i) perm[(size_t)i] = i;
    uint64_t s = 12345;
    for (int32_t i = obs.src_blocks - 1; i > 0; --i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        std::swap(perm[(size_t)i], perm[(size_t)((s >> 33) % (uint64_t)(i + 1))]);
    }
    obs.src_bt.assign((size_t)obs.max_requests * obs.max_blocks, -1);
    int32_t k = 0;
    for (size_t r = 0; r < reqs.size(); ++r)
        for (int32_t b = 0; b < (reqs[r].prompt_tokens + reqs[r].output_tokens + 15) / 16; ++b)
            obs.src_bt[r * (size_t)obs.max_blocks + (size_t)b] = perm[(size_t)k++];
    engine.set_trace_sink([&obs](const SimEvent& ev) { obs.before(ev); });
    out.res = engine.run();
    obs.observe();
    obs.e = nullptr;
    return out;
}

inline const scen::Scenario* find_scenario(const std::vector<scen::Scenario>& all, const std::string& name) {
    for (const auto& sc : all)
        if (sc.name == name) return &sc;
    return nullptr;
}

}  // namespace kvxobs
