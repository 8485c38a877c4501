// engine_patched_run.cpp -- one golden scenario through the PATCHED reference
// engine (integration/engine_kvx.patch) with the kvx data plane in the mode
// PIPESIM_KVX selects (parity | measured | unset = the reference).  Prints one
// JSON line: the engine's outcome and, per transition, the simulated times of
// its waves and commit -- in measured mode these are the B200's.
// Usage: engine_patched_run <scenario>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include <json.hpp>

#include "pipesim/engine.hpp"
#include "pipesim/kvx_plane.hpp"
#include "scenarios.hpp"  // oracle/scenarios.hpp

using namespace pipesim;
using json = nlohmann::json;

int main(int argc, char** argv) {
    const std::string name = argc > 1 ? argv[1] : "llama13b_8to4";
    const scen::Scenario* sc = nullptr;
    static const auto all = scen::scenarios();
    for (const auto& s : all)
        if (s.name == name) sc = &s;
    if (!sc) {
        std::fprintf(stderr, "unknown scenario %s\n", name.c_str());
        return 1;
    }
    scen::Built b = scen::build(*sc);
    Engine engine(b.ec, b.cluster, sc->reqs);
    for (auto [t, k] : sc->forced) engine.force_refactor_at(t, "m0", k);
    for (double t : sc->revocations) engine.revoke_grant_at(t, "m0");
    std::map<std::int64_t, std::vector<double>> syncs, commits, begins;
    engine.set_trace_sink([&](const SimEvent& ev) {
        if (ev.kind == EventKind::KvSyncComplete) syncs[ev.instance_id].push_back(ev.time_ms);
        if (ev.kind == EventKind::RefactorCommit) commits[ev.instance_id].push_back(ev.time_ms);
    });
    EngineResult r = engine.run();
    double lat = 0.0;
    for (const auto& rec : r.records) lat += rec.finish_ms - rec.arrival_ms;
    json out;
    const char* mode = std::getenv("PIPESIM_KVX");
    out["scenario"] = name;
    out["mode"] = mode ? mode : "off";
    out["refactor_commits"] = r.refactor_commits;
    out["refactor_holds"] = r.refactor_holds;
    out["kv_violations"] = r.kv_violations;
    out["kv_synced_bytes"] = r.kv_synced_bytes;
    out["duration_ms"] = r.duration_ms;
    out["mean_latency_ms"] = r.records.empty() ? 0.0 : lat / (double)r.records.size();
    out["kv_sync_complete_ms"] = syncs;
    out["refactor_commit_ms"] = commits;
    if (mode) {
        json st = json::parse(KvxPlane::stats_json());
        json waves = json::array();
        for (const auto& w : st["wave_log"])
            waves.push_back({{"instance", w["instance"]}, {"issued_ms", w["now_ms"]}, {"tokens", w["tokens"]},
                             {"modelled_ms", w["modelled_ms"]}, {"measured_ms", w["measured_ms"]},
                             {"scheduled_ms", w["scheduled_ms"]}});
        out["waves"] = waves;
        out["mismatched_words"] = st["mismatched_words"];
        out["violations_device"] = st["violations_device"];
        out["geometries"] = st["geometries"];
    }
    std::printf("%s\n", out.dump().c_str());
    return 0;
}
