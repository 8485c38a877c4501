// test_kvx_patched.cpp -- the PATCHED reference engine (integration/
// engine_kvx.patch: its own transition handlers call the kvx data plane)
// in the reference's doctest style.  Built against the patched headers and
// libpipesim_kvx.a by integration/Makefile; needs a GPU.
//   - parity mode: the engine's golden outcomes are unchanged with real KV
//     moving (criterion 12: 2 commits, kv_synced_bytes 2.42e9, Eq. 10 == 0
//     on host and device, every live word equal to the payload);
//   - measured-time mode: every KvSyncComplete is scheduled at the measured
//     device completion of its wave (engine.cpp:646,672), the commit at
//     max(final wave measured, load_ready) (:686);
//   - a KV shortfall at the grant is a refactor hold (engine.cpp:592-593).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cstdlib>
#include <map>
#include <vector>

#include <json.hpp>

#include "pipesim/engine.hpp"
#include "pipesim/kvx_plane.hpp"
#include "scenarios.hpp"  // oracle/scenarios.hpp

using namespace pipesim;
using json = nlohmann::json;

namespace {
const scen::Scenario& scenario(const char* name) {
    static const auto all = scen::scenarios();
    for (const auto& s : all)
        if (s.name == name) return s;
    FAIL("unknown scenario");
    return all.front();
}

struct Run {
    EngineResult res;
    json stats;
    std::vector<SimEvent> events;
};

Run run(const scen::Scenario& sc, const char* mode, double gpu_memory_bytes = 0.0) {
    setenv("PIPESIM_KVX", mode, 1);
    KvxPlane::reset_stats();
    scen::Scenario s = sc;
    if (gpu_memory_bytes > 0.0) s.cluster.gpu_memory_bytes = gpu_memory_bytes;
    scen::Built b = scen::build(s);
    Engine engine(b.ec, b.cluster, s.reqs);
    for (auto [t, k] : s.forced) engine.force_refactor_at(t, "m0", k);
    for (double t : s.revocations) engine.revoke_grant_at(t, "m0");
    Run r;
    engine.set_trace_sink([&r](const SimEvent& ev) { r.events.push_back(ev); });
    r.res = engine.run();
    r.stats = json::parse(KvxPlane::stats_json());
    unsetenv("PIPESIM_KVX");
    return r;
}
}  // namespace

TEST_CASE("patched engine, parity mode: criterion 12 unchanged with real KV moving") {
    // acceptance_main.cpp:631-689 via oracle/scenarios.hpp ("criterion12")
    Run r = run(scenario("criterion12"), "parity");
    CHECK(r.res.refactor_commits == 2);
    CHECK(r.res.refactor_aborts == 0);
    CHECK(r.res.kv_violations == 0);
    CHECK(r.res.kv_synced_bytes == doctest::Approx(2.42e9));
    CHECK(r.stats["commits"] == 2);
    CHECK(r.stats["transitions"] == 2);
    CHECK(r.stats["violations_device"] == 0);
    CHECK(r.stats["violation_mismatches"] == 0);
    CHECK(r.stats["mismatched_words"] == 0);
    CHECK(r.stats["verified_tokens"].get<std::int64_t>() > 0);
    CHECK(r.stats["tokens"].get<double>() * 1.0e5 == doctest::Approx(r.res.kv_synced_bytes));
    CHECK(r.res.memory_conserved);
}

TEST_CASE("patched engine, parity mode: revocation aborts on the device") {  // test_engine.cpp:251-263
    Run r = run(scenario("engine_revoke"), "parity");
    CHECK(r.res.refactor_aborts == 1);
    CHECK(r.res.refactor_commits == 0);
    CHECK(r.stats["aborts"] == 1);
    CHECK(r.stats["commits"] == 0);
    CHECK(r.res.memory_conserved);
}

TEST_CASE("patched engine, measured-time mode: events at the measured completion") {
    Run r = run(scenario("criterion12"), "measured");
    CHECK(r.res.refactor_commits == 2);
    CHECK(r.res.kv_violations == 0);
    CHECK(r.stats["mismatched_words"] == 0);
    CHECK(r.stats["violation_mismatches"] == 0);
    std::map<std::int64_t, std::vector<double>> syncs, commits;  // per instance: dispatch times
    for (const SimEvent& ev : r.events) {
        if (ev.kind == EventKind::KvSyncComplete) syncs[ev.instance_id].push_back(ev.time_ms);
        if (ev.kind == EventKind::RefactorCommit) commits[ev.instance_id].push_back(ev.time_ms);
    }
    const auto& log = r.stats["wave_log"];
    REQUIRE(log.size() >= 4);
    int at_measured = 0, moved = 0;
    for (const auto& w : log) {
        const double due = w["now_ms"].get<double>() + w["scheduled_ms"].get<double>();
        CHECK(w["scheduled_ms"].get<double>() == w["measured_ms"].get<double>());
        const std::int64_t inst = w["instance"].get<std::int64_t>();
        bool found = false;
        for (double t : syncs[inst]) found = found || t == due;         // delta / wave 0 (:646,672)
        for (double t : commits[inst]) found = found || t >= due;       // final: max(due, load_ready) (:686)
        CHECK(found);
        at_measured += found;
        moved += w["tokens"].get<std::int64_t>() > 0;
    }
    CHECK(at_measured == (int)log.size());
    CHECK(moved >= 2);
}

TEST_CASE("patched engine: a KV shortfall at the grant is a refactor hold") {
    // C3 (13B, 8->4) at its real KV geometry: a 4-stage grant needs 6.5 GB of
    // parameters + 7.95 GB of KV per GPU (10 layers x 2,426 blocks x 320 KiB,
    // every live request at its full length).  With 10 GB GPUs the reference
    // (which charges parameters only, cluster.cpp:75-82) commits into memory
    // it does not have; the patched engine holds instead.
    const auto& c3 = scenario("llama13b_8to4");
    Run tight = run(c3, "parity", 10.0e9);
    CHECK(tight.res.refactor_commits == 0);
    CHECK(tight.res.refactor_holds >= 1);
    CHECK(tight.stats["transitions"] == 0);
    Run roomy = run(c3, "parity", 16.0e9);
    CHECK(roomy.res.refactor_commits == 1);
    CHECK(roomy.res.refactor_holds == 0);
    CHECK(roomy.stats["geometries"].contains("40x128"));  // the real 13B shape moved
    CHECK(roomy.stats["kv_charged_bytes"].get<double>() > 4.0 * 7.9e9);
    CHECK(roomy.stats["mismatched_words"] == 0);
    CHECK(roomy.res.memory_conserved);
}
