"""Replays a golden transition (tests/golden, from the unmodified reference
engine) through any object with the RefactorCtx handler shape:

    begin(req, kv) -> tokens, lo, hi
    on_sync_complete(req, kv, inflight) -> action, tokens, lo, hi

and checks every decision and interval against the reference's.
"""
import numpy as np

from paper_2510_11938_b200.workload import Barrier, Wave

ACT_DELTA, ACT_BARRIER_WAIT, ACT_FINAL = 0, 1, 2


def replay(ctl, t, check_intervals=True):
    """Yields (wave, lo, hi) for each wave the replay issued; asserts parity."""
    ev = list(t.events)
    w0 = ev.pop(0)
    assert isinstance(w0, Wave) and w0.index == 0
    tok, lo, hi = ctl.begin(w0.req, w0.hi)
    assert tok == int(w0.hi.sum()) == w0.tokens + int(w0.lo.sum())
    if check_intervals:
        np.testing.assert_array_equal(lo, w0.lo)
        np.testing.assert_array_equal(hi, w0.hi)
    yield w0, lo, hi
    while ev:
        e = ev.pop(0)
        if isinstance(e, Barrier):
            act, tok, lo, hi = ctl.on_sync_complete(e.req, e.kv, e.inflight_batches)
            if e.inflight_batches > 0:
                assert act == ACT_BARRIER_WAIT, (act, e.inflight_batches)
                continue
            # Quiescent at the barrier: the final wave is issued in the same handler.
            assert act == ACT_FINAL
            w = ev.pop(0)
            assert isinstance(w, Wave) and w.final
        else:
            w = e
            if w.final:
                act, tok, lo, hi = ctl.on_sync_complete(w.req, w.hi, 0)
                assert act == ACT_FINAL
            else:
                act, tok, lo, hi = ctl.on_sync_complete(w.req, w.hi, 1)
                assert act == ACT_DELTA
        assert tok == w.tokens
        if check_intervals:
            np.testing.assert_array_equal(lo, w.lo)
            np.testing.assert_array_equal(hi, w.hi)
        yield w, lo, hi
