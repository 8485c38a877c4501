"""Stage-boundary activation handoff: the oracle plan over the in-flight
micro-batches the reference leaves at each barrier (tests/golden)."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import workload as W


def barriers():
    for name in W.golden_names():
        scn = W.load_golden(name)
        for ti, t in enumerate(scn.transitions):
            for e in t.events:
                if isinstance(e, W.Barrier) and e.microbatches:
                    yield name, ti, t, e


CASES = list(barriers())


def test_every_reference_barrier_has_its_inflight_set():
    assert len(CASES) >= 10
    # the barrier's in-flight count (engine.cpp:678) is exactly the batches we see
    for name, ti, t, b in CASES:
        assert len(b.microbatches) == b.inflight_batches


@pytest.mark.parametrize("name,ti,t,b", CASES, ids=[f"{c[0]}-{c[1]}" for c in CASES])
def test_plan_routes_to_owner_of_resume_layer(name, ti, t, b):
    row = 512
    after = [m.after for m in b.microbatches]
    tokens = [m.tokens for m in b.microbatches]
    cap = [1 << 40] * (len(t.new_boundaries) + 1)
    rc, ns, rl, off, by = O.handoff_plan(t.old_boundaries, t.new_boundaries, row, after, tokens, cap)
    assert rc == 0
    for i, m in enumerate(b.microbatches):
        if m.after < 0:
            assert (ns[i], rl[i], by[i]) == (0, 0, 0)
            continue
        assert rl[i] == t.old_boundaries[m.after]                     # resumes at the next old stage's first layer
        assert ns[i] == O.activation_owner(t.old_boundaries, t.new_boundaries, m.after)
        assert by[i] == m.tokens * row
        assert off[i] % 256 == 0
        assert m.act_bytes > 0                                         # the reference charges a hop for it
    # arenas: disjoint, packed in batch order
    for k in set(ns.tolist()):
        idx = [i for i in range(len(ns)) if ns[i] == k and by[i] > 0]
        ends = [int(off[i] + by[i]) for i in idx]
        starts = [int(off[i]) for i in idx]
        assert all(starts[j + 1] >= ends[j] for j in range(len(idx) - 1))


def test_arena_overflow_rejected():
    rc, *_ = O.handoff_plan([2], [1, 3], 256, [0], [10], [0, 100, 0])
    assert rc == -1


def test_finished_and_out_of_range_stages():
    """after_stage == K_old-1: the batch finished the old pipeline (engine.cpp:456-458
    completes it), so it is not in flight and gets no slot; after_stage >= K_old has
    no old stage and is rejected."""
    rc, ns, rl, off, by = O.handoff_plan([2], [1, 3], 256, [-1, 0, 1], [4, 4, 4], [1 << 20] * 3)
    assert rc == 0
    assert (ns[0], rl[0], by[0]) == (0, 0, 0)      # re-dispatched at the new head
    assert (ns[1], rl[1], by[1]) == (1, 2, 1024)   # resumes at layer 2, owned by new stage 1
    assert (ns[2], rl[2], by[2]) == (-1, -1, 0)    # done: no slot
    rc, *_ = O.handoff_plan([2], [1, 3], 256, [2], [4], [1 << 20] * 3)
    assert rc == -1
