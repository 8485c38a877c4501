// test_kvx_engine.cpp -- the refactor tests of the reference's own suite
// (/root/reference/proj/tests/test_engine.cpp:194-263, acceptance criterion 12
// at acceptance_main.cpp:631-689), restated with the kvx data plane attached:
// the same scenarios, the same assertions the reference makes about its
// simulated transition, plus the data-plane ones -- the device's Eq. 10 count
// equals the reference's and every live destination word equals the payload.
// doctest-style (oracle/shim/doctest.h) so they read like the reference's tests.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include "kvx_observer.hpp"

using namespace kvxobs;

namespace {
const std::vector<scen::Scenario>& all() {
    static const auto v = scen::scenarios();
    return v;
}
RunOut run(const char* name, bool refactors = true) {
    const scen::Scenario* sc = find_scenario(all(), name);
    REQUIRE(sc != nullptr);
    return run_with_kvx(*sc, 2, 64, /*print_lines=*/false, refactors);
}
int count_kind(const RunOut& r, const char* kind) {
    int n = 0;
    for (const auto& l : r.obs->lines) n += l["kind"] == kind;
    return n;
}
void check_tokens_preserved(const RunOut& forced, const RunOut& base) {
    REQUIRE(forced.res.records.size() == base.res.records.size());
    for (std::size_t i = 0; i < forced.res.records.size(); ++i) {
        CHECK(forced.res.records[i].outcome == RequestOutcome::Completed);
        CHECK(forced.res.records[i].tokens_generated == base.res.records[i].tokens_generated);
    }
}
}  // namespace

TEST_CASE("engine+kvx: forced refactor with zero in-flight moves no KV") {  // test_engine.cpp:194-205
    auto r = run("engine_zero_inflight");
    CHECK(r.res.refactor_commits == 1);
    CHECK(r.res.kv_violations == 0);
    CHECK(r.obs->dev_violations == 0);
    CHECK(r.obs->tokens_moved == 0);
    CHECK(r.res.kv_synced_bytes == doctest::Approx(0.0));
    CHECK(r.res.memory_conserved);
    CHECK(r.res.anti_colocation_ok);
}

TEST_CASE("engine+kvx: refactor mid-decode keeps tokens and KV consistent") {  // test_engine.cpp:207-238
    auto base = run("engine_mid_decode", false);
    auto r = run("engine_mid_decode");
    CHECK(r.res.refactor_commits == 1);
    CHECK(r.res.kv_violations == 0);
    CHECK(r.obs->dev_violations == r.res.kv_violations);
    CHECK(r.res.kv_synced_bytes > 0.0);
    CHECK(r.obs->tokens_moved > 0);
    CHECK(r.obs->mismatched_words == 0);
    check_tokens_preserved(r, base);
    CHECK(r.res.memory_conserved);
    CHECK(r.res.anti_colocation_ok);
}

TEST_CASE("engine+kvx: consolidation back to coarse also commits cleanly") {  // test_engine.cpp:240-249
    auto r = run("engine_consolidate");
    CHECK(r.res.refactor_commits == 1);
    CHECK(r.res.kv_violations == 0);
    CHECK(r.obs->dev_violations == 0);
    CHECK(r.obs->mismatched_words == 0);
    for (const auto& rec : r.res.records) CHECK(rec.outcome == RequestOutcome::Completed);
}

TEST_CASE("engine+kvx: revoked grant aborts the transition, old pipeline survives") {  // test_engine.cpp:251-263
    auto r = run("engine_revoke");
    CHECK(r.res.refactor_aborts == 1);
    CHECK(r.res.refactor_commits == 0);
    CHECK(count_kind(r, "abort") == 1);
    CHECK(count_kind(r, "commit") == 0);
    for (const auto& rec : r.res.records) CHECK(rec.outcome == RequestOutcome::Completed);
    CHECK(r.res.memory_conserved);
    CHECK(r.res.anti_colocation_ok);
}

TEST_CASE("engine+kvx: mid-decode refactor correctness (acceptance criterion 12)") {  // acceptance_main.cpp:631-689
    auto base = run("criterion12", false);
    auto r = run("criterion12");
    CHECK(r.res.refactor_commits == 2);
    CHECK(r.res.kv_violations == 0);
    CHECK(r.obs->dev_violations == 0);
    CHECK(r.obs->mismatched_words == 0);
    CHECK(r.res.kv_synced_bytes == doctest::Approx(2.42e9));
    CHECK(count_kind(r, "commit") == 2);
    check_tokens_preserved(r, base);
}

TEST_CASE("engine+kvx: delta waves up to max_sync_rounds, then the barrier") {  // engine.cpp:665-676
    auto r = run("delta_rounds_cap");
    CHECK(r.res.refactor_commits == 1);
    REQUIRE(r.obs->lines.size() == 1);
    CHECK(r.obs->lines[0]["waves"] == 7);  // wave 0 + 5 delta waves + final
    CHECK(r.obs->dev_violations == 0);
    CHECK(r.obs->mismatched_words == 0);
}
