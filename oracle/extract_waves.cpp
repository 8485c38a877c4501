// Golden-vector extractor for the inflight-refactor KV transition.
//
// TEST INFRASTRUCTURE ONLY.  Links the UNMODIFIED reference library
// (oracle/_ref/libpipesim.a, built from /root/reference/proj/src by
// oracle/Makefile) and runs forced-refactor scenarios through the reference's
// public Engine API (force_refactor_at / revoke_grant_at / set_trace_sink,
// /root/reference/proj/include/pipesim/engine.hpp:109-119).
//
// The reference keeps its transition state (RefactorCtx, engine.hpp:149-158)
// private.  To read it we compile THIS translation unit with `private` mapped
// to `public` around the include; GCC does not reorder members across access
// specifiers, so the object layout is the one libpipesim.a was built with.
// Nothing is written through these members -- the observer is read-only.
//
// The trace sink runs *before* each handler (engine.cpp:243-245), so each
// observation sees the state the previous handler left behind.  A wave is
// identified by (epoch, rounds, commit_scheduled): begin_refactor issues wave 0
// (engine.cpp:637-647), every delta wave bumps `rounds` (engine.cpp:665-674),
// the post-barrier final wave sets `commit_scheduled` (engine.cpp:680-687).
// Per wave we record, for every snapshotted request, the interval
// [synced_before, target) -- exactly the tokens the reference charges in
// kv_synced_bytes.  Commit records carry the live (req, kv_tokens) set the
// Eq. 10 check of engine.cpp:704-713 runs over, and the violation count the
// reference produced.
//
// Usage: extract_waves <out_dir>   (writes <scenario>.jsonl per scenario)
#include <any>
#include <cstdio>
#include <deque>
#include <fstream>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <queue>
#include <string>
#include <vector>

#include <json.hpp>

// Every header engine.hpp pulls in is included first (and is #pragma once),
// so the access-specifier remap below touches engine.hpp alone.
#include "pipesim/cluster.hpp"
#include "pipesim/controller.hpp"
#include "pipesim/metrics.hpp"
#include "pipesim/modelgraph.hpp"
#include "pipesim/workload.hpp"

#define private public
#include "pipesim/engine.hpp"
#undef private
#include "pipesim/cluster.hpp"
#include "pipesim/modelgraph.hpp"
#include "pipesim/rng.hpp"
#include "pipesim/workload.hpp"

using namespace pipesim;
using json = nlohmann::json;

namespace {

struct Scenario {
    std::string name;
    std::string note;
    int num_ops = 32;
    int ops_per_group = 2;
    double op_param_bytes = 0.5e9;
    double act_bytes = 2.0e6;
    std::vector<int> stage_counts;
    int static_stages = 4;
    int max_batch_factor = 32;
    double kv_bytes_per_token = 1.0e5;
    double kv_sync_bw = 0.0;  // 0 = inter-stage bw (engine.cpp:87-90)
    double inter_stage_bw = 1.0e7;
    double batch_max_wait_ms = 0.0;
    int max_sync_rounds = 8;
    SyntheticClusterSpec cluster;
    std::vector<Request> reqs;
    std::vector<std::pair<double, int>> forced;  // (t_ms, target stages)
    std::vector<double> revocations;
};

std::vector<Request> steady(int n, double gap_ms, int prompt, int output) {
    std::vector<Request> v;
    for (int i = 0; i < n; ++i) {
        Request r;
        r.id = i;
        r.arrival_ms = gap_ms * (i + 1);
        r.prompt_tokens = prompt;
        r.output_tokens = output;
        r.model_id = "m0";
        r.slo_deadline_ms = 1.0e9;
        v.push_back(r);
    }
    return v;
}

// Fixture of test_engine.cpp:23-55 (32-op uniform chain, kv 1e5 B/token,
// 2x4x4 synthetic cluster).
Scenario engine_fixture(const std::vector<int>& counts, int static_stages) {
    Scenario s;
    s.stage_counts = counts;
    s.static_stages = static_stages;
    s.cluster.racks = 2;
    s.cluster.servers_per_rack = 4;
    s.cluster.gpus_per_server = 4;
    s.cluster.gpu_memory_bytes = 16.0e9;
    s.cluster.storage_bw_bytes_per_ms = 1.0e6;
    s.cluster.host_bw_bytes_per_ms = 1.0e7;
    return s;
}

// Llama-shaped chain: one op per decoder layer; kv bytes/token =
// 2 (K,V) * layers * kv_heads * head_dim * 2 B (fp16).
Scenario llama(int layers, int kv_heads, double params_total) {
    Scenario s;
    s.num_ops = layers;
    s.ops_per_group = 1;
    s.op_param_bytes = params_total / layers;
    s.act_bytes = 2.0e6;
    s.kv_bytes_per_token = 2.0 * layers * kv_heads * 128 * 2;
    s.kv_sync_bw = 900.0e6;  // NVLink 5, bytes per ms
    s.inter_stage_bw = 50.0e6;
    s.max_batch_factor = 32;
    s.batch_max_wait_ms = 0.0;
    s.cluster.racks = 2;
    s.cluster.servers_per_rack = 8;
    s.cluster.gpus_per_server = 8;
    s.cluster.gpu_memory_bytes = 180.0e9;
    s.cluster.storage_bw_bytes_per_ms = 50.0e6;
    s.cluster.host_bw_bytes_per_ms = 200.0e6;
    return s;
}

std::vector<Scenario> scenarios() {
    std::vector<Scenario> out;
    {  // test_engine.cpp:194-205
        Scenario s = engine_fixture({4, 8}, 4);
        s.name = "engine_zero_inflight";
        s.note = "test_engine.cpp:194-205 forced 4->8 after all requests finished";
        s.reqs = steady(3, 5.0, 64, 3);
        s.forced = {{5000.0, 8}};
        out.push_back(s);
    }
    {  // test_engine.cpp:207-238
        Scenario s = engine_fixture({4, 16}, 4);
        s.name = "engine_mid_decode";
        s.note = "test_engine.cpp:207-238 forced 4->16 at 200 ms mid-decode";
        for (int i = 0; i < 30; ++i) {
            Request r;
            r.id = i;
            r.arrival_ms = 1.0 + 0.01 * i;
            r.prompt_tokens = 100;
            r.output_tokens = 20;
            r.model_id = "m0";
            r.slo_deadline_ms = 1.0e9;
            s.reqs.push_back(r);
        }
        s.forced = {{200.0, 16}};
        out.push_back(s);
    }
    {  // test_engine.cpp:240-249
        Scenario s = engine_fixture({4, 16}, 16);
        s.name = "engine_consolidate";
        s.note = "test_engine.cpp:240-249 forced 16->4 at 150 ms";
        s.reqs = steady(40, 4.0, 100, 10);
        s.forced = {{150.0, 4}};
        out.push_back(s);
    }
    {  // test_engine.cpp:251-263
        Scenario s = engine_fixture({4, 16}, 4);
        s.name = "engine_revoke";
        s.note = "test_engine.cpp:251-263 forced 4->16 at 100 ms, grant revoked at 110 ms";
        s.reqs = steady(40, 4.0, 100, 10);
        s.forced = {{100.0, 16}};
        s.revocations = {110.0};
        out.push_back(s);
    }
    {  // acceptance_main.cpp:631-689
        Scenario s = engine_fixture({4, 16}, 4);
        s.name = "criterion12";
        s.note = "acceptance_main.cpp:631-689 forced 4->16 at 400 ms and 16->4 at 8000 ms";
        s.max_batch_factor = 8;
        s.batch_max_wait_ms = 5.0;
        s.cluster.servers_per_rack = 8;
        s.cluster.storage_bw_bytes_per_ms = SyntheticClusterSpec{}.storage_bw_bytes_per_ms;
        s.cluster.host_bw_bytes_per_ms = SyntheticClusterSpec{}.host_bw_bytes_per_ms;
        for (int i = 0; i < 100; ++i) {
            Request r;
            r.id = i;
            r.arrival_ms = 1.0 + 0.05 * i;
            r.prompt_tokens = 120;
            r.output_tokens = 24;
            r.model_id = "m0";
            r.slo_deadline_ms = 1.0e9;
            s.reqs.push_back(r);
        }
        s.forced = {{400.0, 16}, {8000.0, 4}};
        out.push_back(s);
    }
    {  // BASELINE config 1: Llama-2-7B shape, 4->2 merge, 256 blocks of 16 tokens
        Scenario s = llama(32, 32, 13.5e9);
        s.name = "llama7b_4to2";
        s.note = "BASELINE C1: 32 layers, 32 KV heads, 4->2 merge, 16 requests x 256 tokens";
        s.stage_counts = {2, 4};
        s.static_stages = 4;
        s.reqs = steady(16, 0.01, 248, 24);
        s.forced = {{400.0, 2}};
        out.push_back(s);
    }
    {  // BASELINE config 2: 7B, 2->8 split, 1024 live requests
        Scenario s = llama(32, 32, 13.5e9);
        s.name = "llama7b_2to8";
        s.note = "BASELINE C2: 32 layers, 32 KV heads, 2->8 split, 1024 requests x 128 tokens";
        s.stage_counts = {2, 8};
        s.static_stages = 2;
        s.reqs = steady(1024, 0.001, 128, 16);
        s.forced = {{1500.0, 8}};
        out.push_back(s);
    }
    {  // BASELINE config 3: 13B, 8->4 merge, ~20k live tokens
        Scenario s = llama(40, 40, 26.0e9);
        s.name = "llama13b_8to4";
        s.note = "BASELINE C3: 40 layers, 40 KV heads, 8->4 merge, 256 requests, prompts U[16,144]";
        s.stage_counts = {4, 8};
        s.static_stages = 8;
        Rng rng(0);
        for (int i = 0; i < 256; ++i) {
            Request r;
            r.id = i;
            r.arrival_ms = 1.0 + 0.001 * i;
            r.prompt_tokens = 16 + static_cast<int>(rng.next_u64() % 129);
            r.output_tokens = 64;
            r.model_id = "m0";
            r.slo_deadline_ms = 1.0e9;
            s.reqs.push_back(r);
        }
        s.forced = {{4000.0, 4}};
        out.push_back(s);
    }
    {  // BASELINE config 4 neighbour: 70B GQA shape; same-K re-placement has no
       // reference path (engine.cpp:562), so pin the 80-layer 8->2 and 2->8 moves.
        Scenario s = llama(80, 8, 138.0e9);
        s.name = "llama70b_8to2to8";
        s.note = "BASELINE C4 neighbour: 80 layers, 8 KV heads, 8->2 then 2->8";
        s.stage_counts = {2, 8};
        s.static_stages = 8;
        s.reqs = steady(64, 0.05, 1000, 64);
        s.forced = {{100.0, 2}, {2500.0, 8}};
        out.push_back(s);
    }
    {  // BASELINE config 5: bursty mixed-length trace, repeated refactors
        Scenario s = llama(40, 40, 26.0e9);
        s.name = "bursty_repeated";
        s.note = "BASELINE C5: gamma arrivals CV=4, mixed lengths, forced 8->4->8->4";
        s.stage_counts = {4, 8};
        s.static_stages = 8;
        ArrivalSpec as;
        as.mean_rate = 400.0;
        as.target_cv = 4.0;
        as.duration_s = 2.0;
        as.seed = 7;
        s.reqs = generate_arrivals(as);
        Rng rng(11);
        for (auto& r : s.reqs) {
            r.prompt_tokens = 8 + static_cast<int>(rng.next_u64() % 500);
            r.output_tokens = 4 + static_cast<int>(rng.next_u64() % 60);
            r.slo_deadline_ms = 1.0e9;
        }
        s.forced = {{300.0, 4}, {1500.0, 8}, {3000.0, 4}};
        out.push_back(s);
    }
    return out;
}

json plan_json(const Engine& e, int plan_index) {
    const auto& gp = e.cfg_.granularities.plans[static_cast<std::size_t>(plan_index)];
    json j;
    j["stages"] = gp.config.stages;
    j["boundaries"] = gp.plan.boundaries;
    return j;
}

struct InstSeen {
    bool active = false;
    std::uint64_t epoch = 0;
    int rounds = -1;
    bool commit_scheduled = false;
    int wave = -1;
    bool barrier = false;
    bool commit_pending = false;
    int old_plan = -1;
};

struct Observer {
    Engine* e = nullptr;
    std::ofstream* out = nullptr;
    std::map<std::int64_t, InstSeen> seen;
    std::int64_t commits = 0, aborts = 0, violations = 0;
    double bytes = 0.0;

    void emit(const json& j) { (*out) << j.dump() << "\n"; }

    // Per-server parameter loads of the new stages, as begin_refactor
    // computed them (engine.cpp:621-631): each stage's op range, bytes and
    // whether the server's host cache covers it (cluster.cpp:176-195), plus
    // the reference's warm_start_latency_ms (cluster.cpp:525-536).
    json param_loads(const Engine::InstanceRt& inst, const Engine::RefactorCtx& ctx) {
        const auto loads = e->stage_loads(ctx.target_plan);
        const std::string& model = e->models_[(size_t)inst.model].name;
        std::map<int, std::vector<StageLoad>> per_server;
        for (size_t k = 0; k < ctx.new_gpus.size(); ++k)
            per_server[e->hrg_.gpu(ctx.new_gpus[k]).server_id].push_back(loads[k]);
        json arr = json::array();
        for (const auto& [server, ls] : per_server) {
            json st = json::array();
            for (const auto& l : ls)
                st.push_back({l.begin_op, l.end_op, l.bytes,
                              e->affinity_.cache_covers(server, model, l.begin_op, l.end_op)});
            json j;
            j["server"] = server;
            j["stages"] = st;
            j["host_bw"] = e->hrg_.server(server).host_bw_bytes_per_ms;
            j["storage_bw"] = e->hrg_.storage_bw_bytes_per_ms;
            j["latency_ms"] = warm_start_latency_ms(e->hrg_, e->affinity_, server, model, ls);
            arr.push_back(j);
        }
        return arr;
    }

    // The in-flight micro-batches the barrier leaves to drain
    // (engine.cpp:142-149,449-464): computing in a stage, queued at a stage
    // inbound, or in transit between stages.  `after` = the last old stage
    // whose output the batch holds (-1: none yet); `act_bytes` = the
    // reference's modelled hop size scale_activation(plan, after, units)
    // (modelgraph.cpp:220-233, engine.cpp:136-140).  Tokens per unit: the
    // prompt for a prefill pass, 1 for a decode pass.
    json microbatches(const Engine::InstanceRt& inst) {
        const auto& plan = e->cfg_.granularities.plans[(size_t)inst.plan_index].plan;
        json arr = json::array();
        auto add = [&](const Engine::MicroBatch& b, const char* where, int after) {
            json units = json::array();
            for (const auto& u : b.units) {
                const auto& rt = e->reqs_[(size_t)u.req];
                units.push_back({u.req, u.pass, u.pass == 0 ? rt.prompt_tokens : 1});
            }
            json j;
            j["batch"] = b.id;
            j["where"] = where;
            j["after"] = after;
            j["units"] = units;
            j["act_bytes"] = after >= 0 ? scale_activation(plan, after, (int)b.units.size(),
                                                           e->cfg_.exec.batch_scaling)
                                        : 0.0;
            arr.push_back(j);
        };
        for (size_t s = 0; s < inst.stages.size(); ++s) {
            const auto& st = inst.stages[s];
            if (st.current) add(*st.current, "current", (int)s - 1);
            for (const auto& b : st.inbound) add(b, "inbound", (int)s - 1);
        }
        for (const auto& [id, b] : inst.in_transit) add(b, "transit", b.transit_from);
        return arr;
    }

    void observe(double t_ms) {
        const EngineResult& res = e->result_;
        for (const auto& ip : e->instances_) {
            auto& inst = *ip;
            InstSeen& s = seen[inst.id];
            if (s.active && (!inst.refactor || inst.epoch != s.epoch)) {
                // The transition ended in the previous handler.
                json j;
                j["instance"] = inst.id;
                j["t_ms"] = t_ms;
                if (res.refactor_commits > commits) {
                    j["kind"] = "commit";
                    j["violations"] = res.kv_violations - violations;
                } else if (res.refactor_aborts > aborts) {
                    j["kind"] = "abort";
                } else {
                    j["kind"] = "end_unknown";
                }
                j["kv_synced_bytes_total"] = res.kv_synced_bytes;
                emit(j);
                commits = res.refactor_commits;
                aborts = res.refactor_aborts;
                violations = res.kv_violations;
                s = InstSeen{};
            }
            if (!inst.refactor) continue;
            const auto& ctx = *inst.refactor;
            if (!s.active) {
                s.active = true;
                s.epoch = inst.epoch;
                s.old_plan = inst.plan_index;
                json j;
                j["kind"] = "begin";
                j["instance"] = inst.id;
                j["t_ms"] = t_ms;
                j["epoch"] = inst.epoch;
                j["old"] = plan_json(*e, inst.plan_index);
                j["new"] = plan_json(*e, ctx.target_plan);
                j["new_gpus"] = ctx.new_gpus;
                j["load_ready_ms"] = ctx.load_ready_ms;
                j["begin_ms"] = begin_ms[inst.id];  // now_ms of begin_refactor
                j["param_loads"] = param_loads(inst, ctx);
                emit(j);
            }
            if (ctx.barrier && !s.barrier) {
                // engine.cpp:676 fell in the previous handler: record the live
                // set and in-flight batches the barrier decision saw (the
                // handler does not change them), so a replay can reproduce
                // the delta-vs-barrier choice of engine.cpp:665-678.
                s.barrier = true;
                json live = json::array();
                for (std::size_t i = 0; i < e->reqs_.size(); ++i) {
                    const auto& rt = e->reqs_[i];
                    if (rt.done || rt.home != inst.id) continue;
                    live.push_back({static_cast<std::int64_t>(i), rt.kv_tokens});
                }
                json j;
                j["kind"] = "barrier";
                j["instance"] = inst.id;
                j["t_ms"] = t_ms;
                j["epoch"] = inst.epoch;
                j["rounds"] = ctx.rounds;
                j["inflight_batches"] = inst.inflight_batches;
                j["live"] = live;
                j["microbatches"] = microbatches(inst);
                emit(j);
            }
            if (ctx.rounds != s.rounds || ctx.commit_scheduled != s.commit_scheduled) {
                // A new snapshot wave was issued by the previous handler.
                s.rounds = ctx.rounds;
                s.commit_scheduled = ctx.commit_scheduled;
                ++s.wave;
                json entries = json::array();
                std::int64_t tokens = 0;
                for (const auto& [req, target] : ctx.sync_target) {
                    auto it = ctx.synced_tokens.find(req);
                    const std::int64_t lo = it == ctx.synced_tokens.end() ? 0 : it->second;
                    entries.push_back({req, lo, target});
                    tokens += std::max<std::int64_t>(0, target - lo);
                }
                json j;
                j["kind"] = "wave";
                j["instance"] = inst.id;
                j["t_ms"] = t_ms;
                j["epoch"] = inst.epoch;
                j["wave"] = s.wave;
                j["rounds"] = ctx.rounds;
                j["final"] = ctx.commit_scheduled;
                j["barrier"] = ctx.barrier;
                j["entries"] = entries;
                j["tokens"] = tokens;
                j["kv_synced_bytes_total"] = res.kv_synced_bytes;
                emit(j);
            }
        }
    }

    std::map<std::int64_t, double> begin_ms;  // time of the last RefactorBegin per instance

    void before(const SimEvent& ev) {
        observe(ev.time_ms);
        if (ev.kind == EventKind::RefactorBegin) begin_ms[ev.instance_id] = ev.time_ms;
        if (ev.kind == EventKind::RefactorCommit) {
            auto& inst = *e->instances_[static_cast<std::size_t>(ev.instance_id)];
            if (inst.state != Engine::InstState::Refactoring || !inst.refactor) return;
            if (ev.aux != static_cast<std::int64_t>(inst.epoch)) return;
            // State the Eq. 10 check (engine.cpp:704-713) is about to run over.
            json live = json::array();
            for (std::size_t i = 0; i < e->reqs_.size(); ++i) {
                const auto& rt = e->reqs_[i];
                if (rt.done || rt.home != inst.id) continue;
                live.push_back({static_cast<std::int64_t>(i), rt.kv_tokens});
            }
            json synced = json::array();
            for (const auto& [req, tokens] : inst.refactor->synced_tokens) synced.push_back({req, tokens});
            json j;
            j["kind"] = "commit_state";
            j["instance"] = inst.id;
            j["t_ms"] = ev.time_ms;
            j["epoch"] = inst.epoch;
            j["live"] = live;
            j["synced_before_final"] = synced;
            emit(j);
        }
    }
};

void run(const Scenario& s, const std::string& dir) {
    CompGraph g = make_uniform_chain(s.num_ops, 1.0, s.op_param_bytes, s.act_bytes, s.ops_per_group);
    PartitionParams pp;
    pp.bandwidth_bytes_per_ms = s.inter_stage_bw;
    pp.gpu_memory_bytes = s.cluster.gpu_memory_bytes;
    EngineConfig ec;
    ec.graph = g;
    ec.granularities = enumerate_granularities(g, s.stage_counts, pp, s.max_batch_factor);
    ec.exec.batch_exponent = 0.8;
    ec.exec.stage_efficiency_exponent = 1.0;
    ec.exec.kv_bytes_per_token = s.kv_bytes_per_token;
    ec.exec.batch_max_wait_ms = s.batch_max_wait_ms;
    ec.exec.batch_scaling = {0.1, 1};
    ec.inter_stage_bw_bytes_per_ms = s.inter_stage_bw;
    ec.kv_sync_bw_bytes_per_ms = s.kv_sync_bw;
    ec.max_sync_rounds = s.max_sync_rounds;
    ec.policy.adaptive = false;
    ec.policy.static_stages = s.static_stages;
    ec.policy.initial_instances = 1;
    ec.default_slo_ms = 1.0e9;
    ec.seed = 1;
    Hrg cluster = make_synthetic_cluster(s.cluster);
    ec.storage_bw_bytes_per_ms = s.cluster.storage_bw_bytes_per_ms;

    Engine engine(ec, cluster, s.reqs);
    for (const auto& [t, k] : s.forced) engine.force_refactor_at(t, "m0", k);
    for (double t : s.revocations) engine.revoke_grant_at(t, "m0");

    std::ofstream out(dir + "/" + s.name + ".jsonl");
    Observer obs;
    obs.e = &engine;
    obs.out = &out;
    {
        json h;
        h["kind"] = "scenario";
        h["name"] = s.name;
        h["note"] = s.note;
        h["num_layers"] = s.num_ops;
        h["kv_bytes_per_token"] = s.kv_bytes_per_token;
        h["max_sync_rounds"] = s.max_sync_rounds;
        h["num_requests"] = s.reqs.size();
        h["stage_counts"] = s.stage_counts;
        json forced = json::array();
        for (const auto& [t, k] : s.forced) forced.push_back({t, k});
        h["forced"] = forced;
        h["revocations"] = s.revocations;
        obs.emit(h);
    }
    engine.set_trace_sink([&obs](const SimEvent& ev) { obs.before(ev); });
    EngineResult res = engine.run();
    obs.observe(engine.now_ms_);
    json r;
    r["kind"] = "result";
    r["refactor_commits"] = res.refactor_commits;
    r["refactor_aborts"] = res.refactor_aborts;
    r["refactor_holds"] = res.refactor_holds;
    r["kv_violations"] = res.kv_violations;
    r["kv_synced_bytes"] = res.kv_synced_bytes;
    r["events_dispatched"] = res.events_dispatched;
    r["memory_conserved"] = res.memory_conserved;
    r["anti_colocation_ok"] = res.anti_colocation_ok;
    obs.emit(r);
    std::printf("%-22s commits=%lld aborts=%lld holds=%lld violations=%lld kv_bytes=%.6g\n",
                s.name.c_str(), static_cast<long long>(res.refactor_commits),
                static_cast<long long>(res.refactor_aborts),
                static_cast<long long>(res.refactor_holds),
                static_cast<long long>(res.kv_violations), res.kv_synced_bytes);
}

}  // namespace

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : ".";
    const std::string only = argc > 2 ? argv[2] : "";
    for (const auto& s : scenarios()) {
        if (!only.empty() && s.name != only) continue;
        run(s, dir);
    }
    return 0;
}
