// pipesim/kvx_plane.hpp -- the B200 KV data plane behind pipesim's refactor
// handlers.
//
// integration/engine_kvx.patch adds a `std::shared_ptr<KvxPlane> kvx_` to
// pipesim::Engine and calls it exactly where the reference charges simulated
// KV movement today:
//   begin_refactor  grant (engine.cpp:566-619)  -> grant_kv_bytes: the new
//                   stages' KV is charged with their parameters, so a KV
//                   shortfall is a refactor hold (:592-593)
//                   wave 0 (:637-647)            -> begin + wave
//   on_kv_sync_complete delta (:665-674), final (:680-687) -> wave
//   on_refactor_commit Eq. 10 (:697-713)        -> commit (device check beside
//                   the host loop, payload verified)
//   abort_refactor  (:759-772)                   -> abort
// Every call goes through the kvx C-ABI (include/kvx.h).  The plane owns the
// GPU pools of each in-flight transition and writes the serving pipeline's
// KV payload before a wave reads it (the decode appends of engine.cpp:494-499
// that the simulator only counts).
//
// Enabled per process by the environment (the Engine constructor asks):
//   PIPESIM_KVX=parity     kvx live; the engine keeps its modelled timing, so
//                          the reference's own tests and goldens hold unchanged
//   PIPESIM_KVX=measured   measured-time mode: KvSyncComplete and
//                          RefactorCommit are scheduled at the MEASURED device
//                          completion of each wave (engine.cpp:646,672,686)
//   PIPESIM_KVX_GEOMETRY   "auto" (default: the Llama shape whose bytes/token
//                          equals kv_bytes_per_token, else 2 heads x 64) or
//                          "H,D"
//   PIPESIM_KVX_DEVICE     CUDA device (default 0)
//   PIPESIM_KVX_MAX_GB     cap on one transition's pools, source + destination
//                          (default 96); above it the plane moves a smaller
//                          test geometry (2 x 64, then 1 x 8) -- and charges that
//   PIPESIM_KVX_REPORT     file that receives one JSON line per process at exit:
//                          transitions, waves, bytes, device vs host Eq. 10
//                          counts, mismatched payload words, the wave log
// Unset PIPESIM_KVX: from_env returns null and the engine is the reference.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace pipesim {

struct EngineConfig;
struct Request;

class KvxPlane {
public:
    static std::shared_ptr<KvxPlane> from_env(const EngineConfig& cfg, const std::vector<Request>& workload);
    ~KvxPlane();

    bool measured_time() const;
    /// Device KV bytes each new stage's GPU must hold for this grant: the
    /// destination pools sized for the instance's live requests at their full
    /// length (kvx_stage_kv_bytes).  Fixes the transition's pool geometry.
    std::vector<double> grant_kv_bytes(const std::vector<int>& new_boundaries,
                                       const std::vector<std::int64_t>& live_max_tokens);
    void begin(std::int64_t instance, std::uint64_t epoch, const std::vector<int>& old_boundaries,
               const std::vector<int>& new_boundaries, int num_layers);
    /// One wave over RefactorCtx's snapshot: tokens [synced, target) of every
    /// targeted request.  Returns the wave's duration for the engine's
    /// schedule: the measured device time in measured mode, else modelled_ms.
    double wave(std::int64_t instance, std::uint64_t epoch, const std::map<std::int32_t, std::int64_t>& sync_target,
                const std::map<std::int32_t, std::int64_t>& synced_tokens, double modelled_ms, double now_ms);
    /// Commit on the device (Eq. 10 + compaction) for the live (req, kv)
    /// set, checked against the host loop's count and the payload.
    void commit(std::int64_t instance, std::uint64_t epoch, const std::vector<std::int32_t>& live_req,
                const std::vector<std::int64_t>& live_kv, std::int64_t host_violations);
    void abort(std::int64_t instance);

    /// What every plane of this process did so far (the PIPESIM_KVX_REPORT
    /// line), as JSON; reset_stats() zeroes it (tests).
    static std::string stats_json();
    static void reset_stats();

    struct Impl;

private:
    explicit KvxPlane(std::unique_ptr<Impl> impl);
    std::unique_ptr<Impl> impl_;
};

}  // namespace pipesim
