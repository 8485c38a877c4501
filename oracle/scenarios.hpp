// scenarios.hpp -- the forced-refactor scenarios the goldens are extracted
// from (TEST INFRASTRUCTURE).  Shared by oracle/extract_waves.cpp (golden
// vectors) and tests/native/engine_kvx.cpp (the reference engine driving the
// kvx data plane), so both run byte-identical reference engines.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "pipesim/cluster.hpp"
#include "pipesim/modelgraph.hpp"
#include "pipesim/rng.hpp"
#include "pipesim/workload.hpp"

namespace scen {

using namespace pipesim;

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

inline std::vector<Request> steady(int n, double gap_ms, int prompt, int output) {
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
inline Scenario engine_fixture(const std::vector<int>& counts, int static_stages) {
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
inline Scenario llama(int layers, int kv_heads, double params_total) {
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

inline std::vector<Scenario> scenarios() {
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
    {  // delta-wave rounds: a slow KV link (kv_sync_bw, engine.cpp:87-90) keeps
       // decode ahead of every wave, so delta waves repeat (engine.cpp:665-674)
       // until the max_sync_rounds cap (engine.hpp:75) forces the barrier.
        Scenario s = engine_fixture({4, 8}, 4);
        s.name = "delta_rounds_cap";
        s.note = "slow KV link: 5 delta waves until max_sync_rounds=5 forces the barrier";
        s.kv_sync_bw = 2.0e4;  // bytes per ms
        s.max_sync_rounds = 5;
        s.reqs = steady(24, 2.0, 40, 200);
        s.forced = {{150.0, 8}};
        out.push_back(s);
    }
    {
        Scenario s = engine_fixture({4, 8}, 4);
        s.name = "delta_rounds_converge";
        s.note = "moderate KV link: delta waves shrink (990, 34, 1 tokens) until one finds nothing new";
        s.kv_sync_bw = 5.0e5;
        s.reqs = steady(24, 2.0, 40, 60);
        s.forced = {{600.0, 8}};
        out.push_back(s);
    }
    {
        // EngineConfig::max_sync_rounds = 0 is a valid setting: wave 0 goes
        // straight to the barrier (engine.cpp:666 never issues a delta wave).
        Scenario s = engine_fixture({4, 8}, 4);
        s.name = "delta_rounds_zero";
        s.note = "max_sync_rounds=0: wave 0, then the barrier at once (no delta wave)";
        s.kv_sync_bw = 2.0e4;
        s.max_sync_rounds = 0;
        s.reqs = steady(24, 2.0, 40, 200);
        s.forced = {{150.0, 8}};
        out.push_back(s);
    }
    return out;
}


// EngineConfig + cluster of a scenario, as run() in extract_waves.cpp builds them.
struct Built {
    EngineConfig ec;
    Hrg cluster;
};

inline Built build(const Scenario& s) {
    CompGraph g = make_uniform_chain(s.num_ops, 1.0, s.op_param_bytes, s.act_bytes, s.ops_per_group);
    PartitionParams pp;
    pp.bandwidth_bytes_per_ms = s.inter_stage_bw;
    pp.gpu_memory_bytes = s.cluster.gpu_memory_bytes;
    Built b;
    EngineConfig& ec = b.ec;
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
    b.cluster = make_synthetic_cluster(s.cluster);
    ec.storage_bw_bytes_per_ms = s.cluster.storage_bw_bytes_per_ms;
    return b;
}

}  // namespace scen
