"""Property tests of the oracle data plane (CPU, hypothesis): invariants of
the destination block rule and of byte placement that hold for ANY plan pair,
request set and wave sequence -- independent of the reference goldens, which
pin the specific cases (test_golden_control, test_oracle_dataplane).

  * bump rule: the ids a transition hands out are exactly 0..K-1, in wave
    order then ascending request id, K = sum ceil(final / B);
  * no destination block is shared by two (request, logical block) pairs;
  * every synced token's K and V rows equal the payload (kvo_verify), and
    blocks never handed out stay untouched (zero);
  * re-syncing an overlap is idempotent (bytes and tables unchanged);
  * commit: Eq. 10 counts exactly the live requests not fully synced; the
    CSR rows are the live requests' table rows; the free list is the dropped
    requests' blocks in ascending request order.
"""
import numpy as np
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import pyoracle as O
from paper_2510_11938_b200 import workload as W

B = 16


@st.composite
def transitions(draw):
    L = draw(st.integers(2, 10))
    cuts = lambda: sorted(draw(st.sets(st.integers(1, L - 1), max_size=min(L - 1, 4))))  # noqa: E731
    ob, nb = cuts(), cuts()
    n = draw(st.integers(1, 10))
    final = np.array(draw(st.lists(st.integers(0, 70), min_size=n, max_size=n)), np.int64)
    n_waves = draw(st.integers(1, 4))
    waves, synced = [], np.zeros(n, np.int64)
    for w in range(n_waves):
        last = w == n_waves - 1
        target = final.copy() if last else np.minimum(
            final, synced + np.array(draw(st.lists(st.integers(0, 40), min_size=n, max_size=n))))
        pick = np.array(draw(st.lists(st.booleans(), min_size=n, max_size=n)))
        req = np.nonzero((target > synced) | (pick & (not last)))[0].astype(np.int32)
        back = np.array(draw(st.lists(st.integers(0, 20), min_size=len(req), max_size=len(req))), np.int64)
        lo = np.maximum(0, synced[req] - back)          # overlaps re-synced (idempotent)
        hi = np.maximum(target[req], synced[req])
        waves.append((req, lo, hi))
        synced[req] = hi
    alive = np.array(draw(st.lists(st.booleans(), min_size=n, max_size=n)))
    seed = draw(st.integers(0, 2**31))
    return L, ob, nb, final, waves, alive, seed


def new_ids_of(bt_before, bt_after):
    """Ids newly written into the table, in (request, logical block) order."""
    m = (bt_before < 0) & (bt_after >= 0)
    return bt_after[m]


@settings(max_examples=80, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(transitions())
def test_block_rule_and_bytes(case):
    L, ob, nb, final, waves, alive, seed = case
    n = len(final)
    max_blocks = max(1, int((final.max() + B - 1) // B))
    src_bt, cap0 = W.fragmented_block_table(final, max_blocks, B, seed=seed % 1000)
    K = int(((final + B - 1) // B).sum())
    g = O.geo(L, 1, 8)                                   # 16-byte tokens
    spare = 3
    dp = O.DataPlane(g, ob, nb, cap0, K + spare, n, max_blocks, src_bt)
    live_all = np.nonzero(final)[0].astype(np.int32)
    if len(live_all):
        dp.fill_source(seed, live_all, final[live_all])
    handed = []
    for req, lo, hi in waves:
        before = dp.bt.copy()
        assert dp.wave(req, lo, hi) == 0
        handed.extend(new_ids_of(before, dp.bt).tolist())
    # bump rule: 0..K-1 in wave order, ascending request id within a wave
    assert handed == list(range(K))
    used = dp.bt[dp.bt >= 0]
    assert len(np.unique(used)) == len(used) == K
    # bytes: every synced token equals the payload; nothing else is written
    # (blocks never handed out, and rows past a request's last token, stay zero)
    if len(live_all):
        assert dp.verify(seed, live_all, final[live_all]) == 0
    for pool in dp.new_pools:
        rows = pool.reshape(-1, K + spare, 2, B, 16)      # [layer][block][K|V][token][16 B]
        assert not rows[:, K:].any()
        for r in range(n):
            t = int(final[r])
            if t % B:
                assert not rows[:, dp.bt[r, t // B], :, t % B:].any()
    # idempotence: re-sync the last wave's overlap
    req, lo, hi = waves[-1]
    pools = [p.copy() for p in dp.new_pools]
    bt = dp.bt.copy()
    assert dp.wave(req, np.maximum(0, hi - 5), hi) == 0
    assert np.array_equal(bt, dp.bt) and all(np.array_equal(a, b) for a, b in zip(pools, dp.new_pools))
    # commit: Eq. 10 + compaction + free list
    live = np.nonzero(alive & (final > 0))[0].astype(np.int32)
    kv = final[live].copy()
    if len(live):
        kv[0] += 1                                        # one live request grew past its sync
    v, row_ptr, blocks, free = dp.commit(live, kv)
    assert v == (1 if len(live) else 0)
    nb_live = [int((final[r] + B - 1) // B) for r in live]
    assert row_ptr.tolist() == np.concatenate([[0], np.cumsum(nb_live)]).astype(int).tolist()
    assert blocks.tolist() == [int(x) for r, c in zip(live, nb_live) for x in bt[r, :c]]
    dropped = [r for r in range(n) if r not in set(live.tolist())]
    assert free.tolist() == [int(x) for r in dropped for x in bt[r, :int((final[r] + B - 1) // B)]]


@settings(max_examples=40, deadline=None)
@given(transitions())
def test_stack_manager_fresh_equals_bump(case):
    """A fresh block manager hands out exactly the bump rule's ids."""
    L, ob, nb, final, waves, alive, seed = case
    n = len(final)
    max_blocks = max(1, int((final.max() + B - 1) // B))
    src_bt, cap0 = W.fragmented_block_table(final, max_blocks, B, seed=1)
    K = max(1, int(((final + B - 1) // B).sum()))
    g = O.geo(L, 1, 8)
    a = O.DataPlane(g, ob, nb, cap0, K, n, max_blocks, src_bt, with_pools=False)
    b = O.DataPlane(g, ob, nb, cap0, K, n, max_blocks, src_bt, with_pools=False, bm=O.StackBM(K))
    for req, lo, hi in waves:
        assert a.wave(req, lo, hi) == 0
        assert b.wave(req, lo, hi) == 0
    assert np.array_equal(a.bt, b.bt)
