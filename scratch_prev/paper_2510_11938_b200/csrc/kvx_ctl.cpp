// kvx_ctl.cpp -- the reference's RefactorCtx state machine, restated on the
// library side of the C-ABI (include/kvx.h, kvx_ctl_*).  Each handler follows
// /root/reference/proj/src/engine.cpp line for line in SEMANTICS (not code):
//   kvx_ctl_begin          engine.cpp:633-647  (snapshot, wave 0, accounting)
//   kvx_ctl_sync_complete  engine.cpp:651-688  (apply, delta / barrier / final)
//   kvx_ctl_commit         engine.cpp:697-713  (final apply, Eq. 10)
// and issues the device waves through kvx_wave / kvx_commit.
#include <algorithm>
#include <vector>

#include "kvx.h"
#include "kvx_internal.h"

namespace {

using kvx::CtlState;

bool live_ok(const kvx_transition* t, int32_t n, const int32_t* req, const int64_t* kv) {
    const CtlState& c = kvx::ctl_of(t);
    if (n < 0 || (n > 0 && (!req || !kv))) return false;
    for (int32_t i = 0; i < n; ++i) {
        if (req[i] < 0 || (size_t)req[i] >= c.synced.size()) return false;
        if (i > 0 && req[i - 1] >= req[i]) return false;
        if (kv[i] < 0) return false;
    }
    return true;
}

// kv_tokens_unsynced (engine.cpp:534-546) over the live homed set.
int64_t unsynced(const CtlState& c, int32_t n, const int32_t* req, const int64_t* kv) {
    int64_t total = 0;
    for (int32_t i = 0; i < n; ++i) total += std::max<int64_t>(0, kv[i] - c.synced[(size_t)req[i]]);
    return total;
}

// snapshot_sync_targets (engine.cpp:548-556) + the device wave over
// [synced, target) of every snapshotted request.
// The mirror is updated only once kvx_wave accepted the wave, so a refused
// wave (e.g. KVX_ENOSPC -> hold / abort) leaves no target behind that a later
// apply() would count as synced.
int snapshot_and_issue(kvx_transition* t, int32_t n, const int32_t* req, const int64_t* kv) {
    CtlState& c = kvx::ctl_of(t);
    std::vector<int64_t> lo((size_t)n), hi((size_t)n);
    for (int32_t i = 0; i < n; ++i) {
        const size_t r = (size_t)req[i];
        lo[(size_t)i] = c.synced[r];
        hi[(size_t)i] = std::max(kv[i], c.synced[r]);
    }
    const int rc = kvx_wave(t, kvx::epoch_of(t), n, req, lo.data(), hi.data());
    if (rc != KVX_OK) return rc;
    for (int32_t k : c.target_keys) c.in_target[(size_t)k] = 0;
    c.target_keys.clear();
    for (int32_t i = 0; i < n; ++i) {
        const size_t r = (size_t)req[i];
        c.target[r] = kv[i];
        c.in_target[r] = 1;
        c.target_keys.push_back(req[i]);
    }
    ++c.waves;
    return KVX_OK;
}

// engine.cpp:657-662 / 697-702
void apply(CtlState& c) {
    for (int32_t k : c.target_keys) {
        const size_t r = (size_t)k;
        c.synced[r] = std::max(c.synced[r], c.target[r]);
        c.in_target[r] = 0;
    }
    c.target_keys.clear();
}

}  // namespace

extern "C" {

int kvx_ctl_begin(kvx_transition* t, int32_t n, const int32_t* req, const int64_t* kv,
                  int64_t* tokens_out) {
    if (!t) return kvx::set_error(KVX_EINVAL, "transition is null");
    CtlState& c = kvx::ctl_of(t);
    if (c.began) return kvx::set_error(KVX_ESTATE, "kvx_ctl_begin called twice");
    if (!live_ok(t, n, req, kv)) return kvx::set_error(KVX_EINVAL, "bad live set");
    int64_t tokens = 0;
    for (int32_t i = 0; i < n; ++i) tokens += kv[i];
    const int rc = snapshot_and_issue(t, n, req, kv);
    if (rc != KVX_OK) return rc;
    c.began = true;
    c.kv_synced_bytes += (double)tokens * c.kv_bytes_per_token;  // engine.cpp:645
    c.last_wave_tokens = tokens;
    if (tokens_out) *tokens_out = tokens;
    return KVX_OK;
}

int kvx_ctl_sync_complete(kvx_transition* t, uint64_t epoch, int32_t n, const int32_t* req,
                          const int64_t* kv, int32_t inflight_batches, int32_t* action_out,
                          int64_t* tokens_out) {
    if (!t) return kvx::set_error(KVX_EINVAL, "transition is null");
    if (epoch != kvx::epoch_of(t)) return kvx::set_error(KVX_ESTALE, "stale epoch");  // engine.cpp:654
    CtlState& c = kvx::ctl_of(t);
    if (!c.began) return kvx::set_error(KVX_ESTATE, "kvx_ctl_begin not called");
    if (!live_ok(t, n, req, kv)) return kvx::set_error(KVX_EINVAL, "bad live set");
    if (tokens_out) *tokens_out = 0;
    apply(c);
    if (!c.barrier) {
        const int64_t delta = unsynced(c, n, req, kv);
        if (delta > 0 && c.rounds < c.max_sync_rounds) {
            const int rc = snapshot_and_issue(t, n, req, kv);
            if (rc != KVX_OK) return rc;
            ++c.rounds;
            c.kv_synced_bytes += (double)delta * c.kv_bytes_per_token;  // engine.cpp:671
            c.last_wave_tokens = delta;
            if (tokens_out) *tokens_out = delta;
            if (action_out) *action_out = KVX_ACT_DELTA;
            return KVX_OK;
        }
        c.barrier = true;  // engine.cpp:676
    }
    // engine.cpp:678 -- unless the in-flight micro-batches are handed off to
    // the new pipeline (kvx_handoff) instead of drained on the old one
    if (c.commit_scheduled || (inflight_batches > 0 && !c.handoff)) {
        if (action_out) *action_out = KVX_ACT_BARRIER_WAIT;
        return KVX_OK;
    }
    const int64_t final_delta = unsynced(c, n, req, kv);
    const int rc = snapshot_and_issue(t, n, req, kv);
    if (rc != KVX_OK) return rc;
    c.kv_synced_bytes += (double)final_delta * c.kv_bytes_per_token;  // engine.cpp:684
    c.commit_scheduled = true;
    c.last_wave_tokens = final_delta;
    if (tokens_out) *tokens_out = final_delta;
    if (action_out) *action_out = KVX_ACT_FINAL;
    return KVX_OK;
}

int kvx_ctl_commit_async(kvx_transition* t, uint64_t epoch, int32_t n, const int32_t* req,
                         const int64_t* kv) {
    if (!t) return kvx::set_error(KVX_EINVAL, "transition is null");
    if (epoch != kvx::epoch_of(t)) return kvx::set_error(KVX_ESTALE, "stale epoch");  // engine.cpp:693
    CtlState& c = kvx::ctl_of(t);
    if (!c.began) return kvx::set_error(KVX_ESTATE, "kvx_ctl_begin not called");
    if (!live_ok(t, n, req, kv)) return kvx::set_error(KVX_EINVAL, "bad live set");
    apply(c);  // engine.cpp:697-702
    int64_t host_violations = 0;  // engine.cpp:707-713
    for (int32_t i = 0; i < n; ++i)
        if (c.synced[(size_t)req[i]] != kv[i]) ++host_violations;
    const int rc = kvx_commit_async(t, epoch, n, req, kv);
    if (rc != KVX_OK) return rc;
    c.host_violations = host_violations;
    return KVX_OK;
}

int kvx_ctl_commit_collect(kvx_transition* t, kvx_commit_result* out) {
    if (!t) return kvx::set_error(KVX_EINVAL, "transition is null");
    CtlState& c = kvx::ctl_of(t);
    kvx_commit_result local{};
    kvx_commit_result* res = out ? out : &local;
    const int rc = kvx_commit_collect(t, res);
    if (rc != KVX_OK) return rc;
    if (res->violations != c.host_violations)
        return kvx::set_error(KVX_ECUDA, "device Eq. 10 check disagrees with the control mirror");
    return KVX_OK;
}

int kvx_ctl_commit(kvx_transition* t, uint64_t epoch, int32_t n, const int32_t* req,
                   const int64_t* kv, kvx_commit_result* out) {
    const int rc = kvx_ctl_commit_async(t, epoch, n, req, kv);
    if (rc != KVX_OK) return rc;
    return kvx_ctl_commit_collect(t, out);
}

int kvx_ctl_set_handoff(kvx_transition* t, int32_t enable) {
    if (!t) return kvx::set_error(KVX_EINVAL, "transition is null");
    kvx::ctl_of(t).handoff = enable != 0;
    return KVX_OK;
}

int kvx_ctl_state_get(const kvx_transition* t, kvx_ctl_state* out) {
    if (!t || !out) return kvx::set_error(KVX_EINVAL, "null argument");
    const CtlState& c = kvx::ctl_of(t);
    out->rounds = c.rounds;
    out->barrier = c.barrier ? 1 : 0;
    out->commit_scheduled = c.commit_scheduled ? 1 : 0;
    out->waves = c.waves;
    out->kv_synced_bytes = c.kv_synced_bytes;
    out->last_wave_tokens = c.last_wave_tokens;
    return KVX_OK;
}

}  // extern "C"
