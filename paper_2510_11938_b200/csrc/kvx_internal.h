// kvx_internal.h -- shared between the data plane (kvx_*.cu) and kvx_ctl.cpp
// (control-plane mirror).  Not part of the public ABI.
#pragma once

#include <cstdint>
#include <vector>

#include "kvx.h"

namespace kvx {

// RefactorCtx (/root/reference/proj/include/pipesim/engine.hpp:149-158),
// with the std::map<int32,int64> pair replaced by dense per-request arrays
// (absent == 0, as every reader in engine.cpp:540-542,711 treats it).
struct CtlState {
    bool began = false;
    std::vector<int64_t> synced;    // synced_tokens
    std::vector<int64_t> target;    // sync_target
    std::vector<uint8_t> in_target; // key present in sync_target
    std::vector<int32_t> target_keys;
    int32_t rounds = 0;
    bool barrier = false;
    bool commit_scheduled = false;
    int32_t waves = 0;
    int32_t max_sync_rounds = 8;    // EngineConfig::max_sync_rounds (engine.hpp:75)
    double kv_bytes_per_token = 0.0;
    double kv_synced_bytes = 0.0;
    int64_t last_wave_tokens = 0;
    int64_t host_violations = 0;    // Eq. 10 on the mirror, checked against the device at collect
    bool handoff = false;           // in-flight batches are handed off, not drained

    void init(int32_t max_requests, int32_t max_rounds, double bpt) {
        synced.assign((size_t)max_requests, 0);
        target.assign((size_t)max_requests, 0);
        in_target.assign((size_t)max_requests, 0);
        target_keys.clear();
        // kept as given: 0 is valid (wave 0, then the barrier; engine.cpp:666),
        // and a negative cap behaves like 0 there too.  The default of 8
        // (engine.hpp:75) lives in the callers (kvx.py, the engine's config).
        max_sync_rounds = max_rounds;
        kv_bytes_per_token = bpt;
    }
};

CtlState& ctl_of(kvx_transition* t);
const CtlState& ctl_of(const kvx_transition* t);
uint64_t epoch_of(const kvx_transition* t);
int set_error(int code, const char* msg);

}  // namespace kvx
