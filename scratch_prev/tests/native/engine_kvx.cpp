// engine_kvx.cpp -- CLI over kvx_observer.hpp: runs a golden scenario through
// the UNMODIFIED reference engine with the kvx data plane attached, prints one
// JSON line per transition and a summary (incl. measured-time mode).
// Usage: engine_kvx <scenario> [auto | heads dim]
#include "kvx_observer.hpp"

using namespace kvxobs;

int main(int argc, char** argv) {
    std::string name = argc > 1 ? argv[1] : "criterion12";
    if (name == "consolidate") name = "engine_consolidate";  // test_engine.cpp:240-249
    if (name == "revoke") name = "engine_revoke";            // test_engine.cpp:251-263
    const auto all = scen::scenarios();
    const scen::Scenario* sp = find_scenario(all, name);
    if (!sp) {
        std::fprintf(stderr, "unknown scenario %s\n", name.c_str());
        return 1;
    }
    const scen::Scenario& sc = *sp;
    // KV geometry: "auto" = the model shape whose bytes/token equals the
    // scenario's kv_bytes_per_token (Llama presets); else heads x dim given.
    int heads = 2, dim = 64;
    if (argc > 2 && std::string(argv[2]) == "auto") {
        const double per = sc.kv_bytes_per_token / (2.0 * sc.num_ops * 128 * 2);
        if (per == (double)(int)per && per >= 1.0) {
            heads = (int)per;
            dim = 128;
        }
    } else if (argc > 3) {
        heads = std::atoi(argv[2]);
        dim = std::atoi(argv[3]);
    }
    scen::Built built = scen::build(sc);
    RunOut run = run_with_kvx(sc, heads, dim, /*print_lines=*/true);
    const EngineResult& res = run.res;
    Observer& obs = *run.obs;
    json sum;
    sum["kind"] = "summary";
    sum["scenario"] = name;
    sum["refactor_commits"] = res.refactor_commits;
    sum["refactor_aborts"] = res.refactor_aborts;
    sum["kv_violations_reference"] = res.kv_violations;
    sum["kv_violations_device"] = obs.dev_violations;
    sum["mismatched_words"] = obs.mismatched_words;
    sum["transitions"] = obs.transitions;
    sum["kv_synced_bytes_reference"] = res.kv_synced_bytes;
    sum["kvx_launches"] = kvx_launch_count();
    sum["geometry"] = {sc.num_ops, heads, dim};
    // measured-time mode: feed the B200-measured KV wave
    // bandwidth back into the unmodified engine through its own knob
    // (EngineConfig::kv_sync_bw_bytes_per_ms, engine.cpp:87-90) and report
    // the simulated stall / latency under the modelled and measured speeds.
    if (obs.measured_ms > 0.0 && obs.measured_bytes > 0.0) {
        const double modelled_bw = built.ec.kv_sync_bw_bytes_per_ms > 0.0 ? built.ec.kv_sync_bw_bytes_per_ms
                                                                         : built.ec.inter_stage_bw_bytes_per_ms;
        json cal;
        cal["modelled"] = plain_run(sc, modelled_bw);
        cal["measured"] = plain_run(sc, obs.measured_bytes / obs.measured_ms);
        sum["measured_time_mode"] = cal;
    }
    std::printf("%s\n", sum.dump().c_str());
    return (obs.mismatched_words == 0 && obs.dev_violations == res.kv_violations) ? 0 : 5;
}
