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
#include <algorithm>
#include <any>
#include <chrono>
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
#include "pipesim/config.hpp"
#include "pipesim/experiment.hpp"
#include "scenarios.hpp"

using namespace pipesim;
using scen::Scenario;
using scen::scenarios;
using json = nlohmann::json;

namespace {

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
                j["barrier_ms"] = prev_dispatch_ms;  // time of the handler that set it
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
    double prev_dispatch_ms = 0.0;            // event time of the handler that just ran

    void before(const SimEvent& ev) {
        observe(ev.time_ms);
        prev_dispatch_ms = ev.time_ms;
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

void run_engine(Engine& engine, const Scenario& s, const std::string& dir);

void run(const Scenario& s, const std::string& dir) {
    scen::Built b = scen::build(s);
    EngineConfig& ec = b.ec;
    Hrg& cluster = b.cluster;

    Engine engine(ec, cluster, s.reqs);
    for (const auto& [t, k] : s.forced) engine.force_refactor_at(t, "m0", k);
    for (double t : s.revocations) engine.revoke_grant_at(t, "m0");
    run_engine(engine, s, dir);
}

// BASELINE config 5 as the reference runs it: the adaptive FlexPipe policy
// (controller Alg. 1, controller.cpp:55) decides every refactor on a gamma
// trace, built through the public experiment API (experiment.hpp:37-47) from
// the reference's own configs/flexpipe-demo.json, shortened.
void run_adaptive(double cv, double duration_s, const std::string& dir) {
    ExperimentConfig cfg = load_config("/root/reference/proj/configs/flexpipe-demo.json");
    cfg.workload.spec.target_cv = cv;
    cfg.workload.spec.duration_s = duration_s;
    cfg.output_dir = "/tmp/pipesim-adaptive";
    // A livelier controller than the demo's (hysteresis 0.5, cooldown 30 s,
    // sigma 20 -- with which g* never leaves 4), so the trace sees
    // controller-chosen refactors; the decisions remain the reference's own.
    cfg.ctrl.hysteresis_margin = 0.02;
    cfg.ctrl.refactor_cooldown_ms = 8000.0;
    cfg.ctrl.sensitivity_sigma = 1.0;  // CV match sharp enough to move g* with the window CV
    ExperimentSetup setup = build_setup(cfg);
    const auto profiles = calibrate_profiles(cfg);
    Scenario s;
    char name[64];
    std::snprintf(name, sizeof(name), "adaptive_cv%g", cv);
    s.name = name;
    s.note = "BASELINE C5: adaptive policy (controller Alg. 1) on configs/flexpipe-demo.json, gamma CV " +
             std::to_string(cv) + ", " + std::to_string((int)duration_s) + " s";
    s.num_ops = (int)setup.engine.graph.ops.size();
    s.kv_bytes_per_token = setup.engine.exec.kv_bytes_per_token;
    s.max_sync_rounds = setup.engine.max_sync_rounds;
    s.reqs = setup.requests;
    for (const auto& gp : setup.granularities.plans) s.stage_counts.push_back(gp.config.stages);
    Engine engine(setup.engine, setup.cluster, setup.requests);
    engine.set_profiles(profiles);
    run_engine(engine, s, dir);
}

void run_engine(Engine& engine, const Scenario& s, const std::string& dir) {

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

// --time <scenario> <reps>: wall time of the reference's own transition
// handlers (SURVEY App. A probe 3), attributed by trace-sink deltas: the sink
// runs right before each handler (engine.cpp:243-245), so a handler's cost is
// the time to the next dispatch.  Medians over reps; JSON on stdout.
int time_handlers(const std::string& name, int reps) {
    std::map<std::string, std::vector<double>> us;
    std::vector<double> run_ms;
    for (const auto& s : scenarios()) {
        if (s.name != name) continue;
        for (int rep = 0; rep < reps; ++rep) {
            scen::Built b = scen::build(s);
            Engine engine(b.ec, b.cluster, s.reqs);
            for (const auto& [t, k] : s.forced) engine.force_refactor_at(t, "m0", k);
            for (double t : s.revocations) engine.revoke_grant_at(t, "m0");
            std::string pending;
            auto t_prev = std::chrono::steady_clock::now();
            engine.set_trace_sink([&](const SimEvent& ev) {
                const auto now = std::chrono::steady_clock::now();
                if (!pending.empty())
                    us[pending].push_back(std::chrono::duration<double, std::micro>(now - t_prev).count());
                pending.clear();
                if (ev.kind == EventKind::RefactorBegin || ev.kind == EventKind::KvSyncComplete ||
                    ev.kind == EventKind::RefactorCommit)
                    pending = to_string(ev.kind);
                t_prev = std::chrono::steady_clock::now();
            });
            const auto t0 = std::chrono::steady_clock::now();
            engine.run();
            run_ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        }
    }
    auto med = [](std::vector<double> v) {
        if (v.empty()) return 0.0;
        std::sort(v.begin(), v.end());
        return v[v.size() / 2];
    };
    json j;
    j["scenario"] = name;
    j["reps"] = reps;
    for (const auto& [k, v] : us) j[k + "_us"] = med(v);
    j["engine_run_ms"] = med(run_ms);
    std::printf("%s\n", j.dump().c_str());
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 2 && std::string(argv[1]) == "--time")
        return time_handlers(argv[2], argc > 3 ? std::atoi(argv[3]) : 5);
    const std::string dir = argc > 1 ? argv[1] : ".";
    const std::string only = argc > 2 ? argv[2] : "";
    for (const auto& s : scenarios()) {
        if (!only.empty() && s.name != only) continue;
        run(s, dir);
    }
    for (double cv : {1.0, 4.0, 7.0}) {
        char name[64];
        std::snprintf(name, sizeof(name), "adaptive_cv%g", cv);
        if (!only.empty() && only != name) continue;
        run_adaptive(cv, 600.0, dir);
    }
    return 0;
}
