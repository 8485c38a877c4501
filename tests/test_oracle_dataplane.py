"""Oracle data plane (CPU): the byte-level parity contract the CUDA path is
held to.  Small geometries so every byte is checked in seconds."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import workload as W
from tests.replay import replay

SEED = 1234


def small_plane(scn_layers, old_b, new_b, tokens, max_blocks, heads=2, dim=64, with_pools=True):
    g = O.geo(scn_layers, heads, dim)
    src_bt, old_blocks = W.fragmented_block_table(tokens, max_blocks, 16, seed=7)
    need = int(((tokens + 15) // 16).sum())
    dp = O.DataPlane(g, old_b, new_b, old_blocks, max(need, 1), len(tokens), max_blocks, src_bt,
                     with_pools=with_pools)
    return g, dp


def test_block_rule_known_answer():
    """Two requests, B=16: wave 0 r0=[0,20) r1=[0,16) -> r0 gets blocks 0,1,
    r1 block 2; wave 1 r0=[20,40) adds block 3 (ceil(40/16)=3 > 2), r1=[16,17)
    adds block 4."""
    tokens = np.array([40, 17], np.int64)
    g, dp = small_plane(4, [2], [1, 3], tokens, 4)
    dp.fill_source(SEED, [0, 1], tokens)
    assert dp.wave([0, 1], [0, 0], [20, 16]) == 0
    assert dp.bt[0, :2].tolist() == [0, 1] and dp.bt[1, 0] == 2
    assert dp.wave([0, 1], [20, 16], [40, 17]) == 0
    assert dp.bt[0, :3].tolist() == [0, 1, 3] and dp.bt[1, :2].tolist() == [2, 4]
    v, row_ptr, blocks, free = dp.commit([0, 1], [40, 17])
    assert v == 0 and row_ptr.tolist() == [0, 3, 5] and blocks.tolist() == [0, 1, 3, 2, 4]
    assert free.size == 0
    assert dp.verify(SEED, [0, 1], [40, 17]) == 0


def test_gap_and_order_rejected():
    tokens = np.array([40, 17], np.int64)
    g, dp = small_plane(4, [2], [1, 3], tokens, 4)
    assert dp.wave([0], [5], [10]) == -1          # lo > synced: tokens would be lost
    assert dp.wave([1, 0], [0, 0], [1, 1]) == -1  # not ascending


def test_overflow_rejected():
    tokens = np.array([64], np.int64)
    g, dp = small_plane(4, [2], [1, 3], tokens, 4)
    assert dp.wave([0], [0], [80]) == -1  # 5 blocks > max_blocks


def test_mt_executor_matches_per_token():
    rng = np.random.default_rng(3)
    n = 37
    tokens = rng.integers(0, 90, n).astype(np.int64)
    a_g, a = small_plane(12, [3, 6, 9], [4, 8], tokens, 8)
    b_g, b = small_plane(12, [3, 6, 9], [4, 8], tokens, 8)
    req = np.arange(n, dtype=np.int32)
    a.fill_source(SEED, req, tokens)
    b.fill_source(SEED, req, tokens)
    cut = rng.integers(0, 90, n).astype(np.int64)
    mid = np.minimum(cut, tokens)
    for lo, hi in ((np.zeros(n, np.int64), mid), (mid, tokens)):
        assert a.wave(req, lo, hi) == 0
        assert b.wave(req, lo, hi, threads=4) == 0
    np.testing.assert_array_equal(a.bt, b.bt)
    for pa, pb in zip(a.new_pools, b.new_pools):
        np.testing.assert_array_equal(pa, pb)
    assert a.verify(SEED, req, tokens) == 0


@pytest.mark.parametrize("name", ["engine_mid_decode", "engine_consolidate", "criterion12",
                                  "bursty_repeated", "delta_rounds_cap", "delta_rounds_converge",
                                  "delta_rounds_zero"])
def test_golden_transitions_bytes(name):
    """Every golden transition, replayed through the oracle control plane and
    executed by the oracle data plane: destination bytes equal the pattern of
    every live (request, layer, K/V, token); Eq. 10 matches the reference."""
    scn = W.load_golden(name)
    for t in scn.transitions:
        if t.outcome != "commit":
            continue
        tokens = t.max_tokens(scn.num_requests)
        max_blocks = int(max(1, (tokens.max() + 15) // 16))
        g, dp = small_plane(scn.num_layers, t.old_boundaries, t.new_boundaries, tokens, max_blocks,
                            heads=1, dim=8 if scn.num_requests > 200 else 32)
        live = np.nonzero(tokens)[0].astype(np.int32)
        dp.fill_source(SEED, live, tokens[live])
        ctx = O.ControlCtx(scn.num_requests, scn.max_sync_rounds, scn.kv_bytes_per_token)

        class Shim:
            def begin(self, req, kv):
                r = ctx.begin(req, kv)
                assert dp.wave(req, r[1], r[2]) == 0
                return r

            def on_sync_complete(self, req, kv, inflight):
                r = ctx.on_sync_complete(req, kv, inflight)
                if r[0] != O.ACT_BARRIER_WAIT:
                    assert dp.wave(req, r[2], r[3]) == 0
                return r

        for _ in replay(Shim(), t):
            pass
        ctx.apply()
        v, row_ptr, blocks, free = dp.commit(t.live_req, t.live_kv)
        assert v == t.violations == ctx.violations(t.live_req, t.live_kv)
        assert dp.verify(SEED, t.live_req, t.live_kv) == 0
        # compaction: CSR covers exactly ceil(kv/16) blocks per live request
        np.testing.assert_array_equal(np.diff(row_ptr), (t.live_kv + 15) // 16)
        # every allocated block is either in the live CSR or on the free list, once
        allocated = dp.bt[dp.bt >= 0]
        assert sorted(np.concatenate([blocks, free]).tolist()) == sorted(allocated.tolist())


def test_activation_owner():
    """A batch in transit out of old stage s feeds layer b_old[s]; its new owner
    is the new stage containing that layer (merge 8->4: stages 1,3,5 become
    internal boundaries of new stages 0,1,2; 0,2,4,6 map to new 1,2,3)."""
    ob = [5, 10, 15, 20, 25, 30, 35]
    nb = [10, 20, 30]
    owners = [O.activation_owner(ob, nb, s) for s in range(7)]
    assert owners == [0, 1, 1, 2, 2, 3, 3]
    assert O.activation_owner(ob, nb, 7) == -1  # last stage: nothing in transit


@pytest.mark.parametrize("name", ["criterion12", "bursty_repeated", "delta_rounds_converge"])
def test_fill_layer_is_the_oracle_destination(name):
    """kvo_fill_layer (the full-size parity tests' expected image) equals the
    oracle executor's destination pools layer by layer, zero rows included:
    given the oracle's destination table and synced marks it regenerates
    exactly what the per-token executor wrote."""
    scn = W.load_golden(name)
    L = scn.num_layers
    for t in scn.transitions:
        tokens = t.max_tokens(scn.num_requests)
        max_blocks = int(max(1, (tokens.max() + 15) // 16))
        g, dp = small_plane(L, t.old_boundaries, t.new_boundaries, tokens, max_blocks, heads=1, dim=8)
        live = np.nonzero(tokens)[0].astype(np.int32)
        dp.fill_source(SEED, live, tokens[live])
        ctx = O.ControlCtx(scn.num_requests, scn.max_sync_rounds, scn.kv_bytes_per_token)

        class Shim:
            def begin(self, req, kv):
                r = ctx.begin(req, kv)
                assert dp.wave(req, r[1], r[2]) == 0
                return r

            def on_sync_complete(self, req, kv, inflight):
                r = ctx.on_sync_complete(req, kv, inflight)
                if r[0] != O.ACT_BARRIER_WAIT:
                    assert dp.wave(req, r[2], r[3]) == 0
                return r

        for _ in replay(Shim(), t):
            pass
        req = np.arange(scn.num_requests, dtype=np.int32)
        lb = dp.new_blocks * 2 * 16 * 1 * 8 * 2
        for j, (b, e) in enumerate(W.stage_ranges(L, t.new_boundaries)):
            for ll in range(e - b):
                want = dp.new_pools[j][ll * lb:(ll + 1) * lb]
                got = O.fill_layer(g, SEED, b + ll, dp.new_blocks, req, dp.synced_hi, dp.bt, threads=3)
                np.testing.assert_array_equal(got, want)
