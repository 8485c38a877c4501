"""Oracle control plane vs the reference's own transitions (CPU).

The golden vectors come from the UNMODIFIED reference engine
(oracle/extract_waves.cpp over /root/reference/proj/src); the oracle's
restatement of RefactorCtx (oracle/kvx_oracle.c, engine.cpp:534-713) must
reproduce every wave interval, every delta/barrier/final decision, the exact
double-precision kv_synced_bytes accumulator and the Eq. 10 violation count.
"""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import workload as W
from tests.replay import replay

NAMES = W.golden_names()


def test_goldens_present():
    assert {"criterion12", "engine_mid_decode", "engine_consolidate", "engine_revoke",
            "engine_zero_inflight", "llama13b_8to4", "llama7b_4to2", "llama7b_2to8",
            "llama70b_8to2to8", "bursty_repeated"} <= set(NAMES)


@pytest.mark.parametrize("name", NAMES)
def test_control_plane_matches_reference(name):
    """Replays every transition in the reference's own global event order
    (instances refactor concurrently in the adaptive goldens), one shared
    EngineResult::kv_synced_bytes accumulator, bit-exact after every wave."""
    scn = W.load_golden(name)
    acc = np.zeros(1, np.float64)  # EngineResult::kv_synced_bytes, shared across transitions
    commits = aborts = violations = 0
    gens, ctxs = {}, {}

    def shim(ctx):
        class Shim:
            def begin(self, req, kv):
                return ctx.begin(req, kv)

            def on_sync_complete(self, req, kv, inflight):
                return ctx.on_sync_complete(req, kv, inflight)
        return Shim()

    for ti, kind, ev in scn.timeline:
        t = scn.transitions[ti]
        if ti not in gens:
            ctxs[ti] = O.ControlCtx(scn.num_requests, scn.max_sync_rounds, scn.kv_bytes_per_token, acc)
            gens[ti] = replay(shim(ctxs[ti]), t)
        if kind == "wave":
            w, _, _ = next(gens[ti])       # consumes the barriers before this wave
            assert w is ev
            assert acc[0] == w.kv_synced_bytes_total  # bit-exact, engine.cpp:645,671,684
        elif kind == "commit":
            ctxs[ti].apply()               # engine.cpp:697-702
            v = ctxs[ti].violations(t.live_req, t.live_kv)
            assert v == t.violations
            violations += v
            commits += 1
            assert acc[0] == t.kv_synced_bytes_total
        elif kind == "abort":
            aborts += 1
    assert acc[0] == scn.result["kv_synced_bytes"]
    assert commits == scn.result["refactor_commits"]
    assert aborts == scn.result["refactor_aborts"]
    assert violations == scn.result["kv_violations"]


def test_adaptive_goldens_refactor_under_the_controller():
    """BASELINE C5: the reference's own controller (Alg. 1) decides the
    refactors on gamma traces; more burstiness, more refactors."""
    n = {cv: W.load_golden(f"adaptive_cv{cv}").result["refactor_commits"] for cv in (1, 4, 7)}
    assert n[1] == 0 and n[4] >= 1 and n[7] > n[4]


def test_known_answers_spec():
    """zero in-flight -> zero KV bytes; 100 valid tokens ->
    sync bytes = 100 * bytes_per_token."""
    scn = W.load_golden("engine_zero_inflight")
    assert scn.result["kv_synced_bytes"] == 0.0
    acc = np.zeros(1)
    ctx = O.ControlCtx(8, 8, 1.0e5, acc)
    tok, lo, hi = ctx.begin(np.array([3]), np.array([100]))
    assert tok == 100 and acc[0] == 100 * 1.0e5


def test_criterion12_wave_plan():
    """refactor 1 moves 100 x [0,120) in its final wave; refactor 2
    moves 100 x [0,121) in wave 0 and 100 x [121,122) in the final wave."""
    scn = W.load_golden("criterion12")
    t1, t2 = scn.transitions
    assert t1.waves[0].tokens == 0 and t1.waves[-1].tokens == 12000
    assert (t2.waves[0].hi == 121).all() and (t2.waves[-1].lo == 121).all()
    assert (t2.waves[-1].hi == 122).all()
    assert scn.result["kv_synced_bytes"] == 2.42e9


def test_violation_detected_when_tokens_missing():
    acc = np.zeros(1)
    ctx = O.ControlCtx(4, 8, 1.0, acc)
    ctx.begin(np.array([0, 1]), np.array([10, 20]))
    ctx.apply()
    assert ctx.violations(np.array([0, 1]), np.array([10, 21])) == 1


def test_delta_rounds_capped():
    """max_sync_rounds (engine.hpp:75) bounds delta waves, then the barrier falls."""
    acc = np.zeros(1)
    ctx = O.ControlCtx(2, 2, 1.0, acc)
    kv = 10
    ctx.begin(np.array([0]), np.array([kv]))
    acts = []
    for _ in range(4):
        kv += 1
        act, tok, lo, hi = ctx.on_sync_complete(np.array([0]), np.array([kv]), 3)
        acts.append(act)
    assert acts == [O.ACT_DELTA, O.ACT_DELTA, O.ACT_BARRIER_WAIT, O.ACT_BARRIER_WAIT]
    act, tok, lo, hi = ctx.on_sync_complete(np.array([0]), np.array([kv]), 0)
    assert act == O.ACT_FINAL and tok == kv - 12 and lo[0] == 12 and hi[0] == kv


def test_delta_round_cap_and_convergence_pinned():
    """engine.cpp:665-676: delta waves repeat while delta > 0 and rounds <
    max_sync_rounds; the cap (5 here) or an empty delta drops the barrier."""
    cap = W.load_golden("delta_rounds_cap").transitions[0]
    assert [w.rounds for w in cap.waves] == [0, 1, 2, 3, 4, 5, 5] and cap.waves[-1].final
    assert [e.rounds for e in cap.events if isinstance(e, W.Barrier)] == [5]
    conv = W.load_golden("delta_rounds_converge").transitions[0]
    assert [w.tokens for w in conv.waves][:3] == [990, 34, 1]
    assert [e.rounds for e in conv.events if isinstance(e, W.Barrier)] == [2]


def test_zero_sync_rounds_pinned():
    """EngineConfig::max_sync_rounds = 0 (engine.cpp:666): the reference
    issues wave 0 and then goes straight to the barrier, no delta wave.  The
    oracle keeps 0 as given (the product used to turn <= 0 into 8)."""
    t = W.load_golden("delta_rounds_zero").transitions[0]
    assert len(t.waves) == 2 and t.waves[-1].final and t.waves[0].rounds == 0
    assert [e.rounds for e in t.events if isinstance(e, W.Barrier)] == [0]
