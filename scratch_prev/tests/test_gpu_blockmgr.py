"""Device block manager on the GPU, and a CHAINED pair of refactors that
reuses pools through it: the reference's criterion-12 scenario (4->16 at
400 ms, then 16->4 at 8000 ms, acceptance_main.cpp:631-689) with the second
transition reading the first one's destination pools through the first
one's block table, and writing into the first one's (recycled) source pools.
Tables, free lists, stacks and every pool byte are compared with the oracle
chain; the final KV equals the payload."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import kvx
from paper_2510_11938_b200 import workload as W
from tests.replay import replay

pytestmark = pytest.mark.gpu
SEED = 0xC4A1


def test_blockmgr_basics(gpu_count):
    bm = kvx.BlockManager(0, 10)
    ref = O.StackBM(10)
    try:
        assert bm.pop(3).tolist() == ref.pop(3).tolist() == [0, 1, 2]
        bm.push([1])
        ref.push([1])
        assert bm.pop(2).tolist() == ref.pop(2).tolist() == [1, 3]
        np.testing.assert_array_equal(bm.snapshot(), ref.snapshot())
        with pytest.raises(kvx.NoSpace):
            bm.pop(99)
        with pytest.raises(kvx.KvxError):
            bm.push(list(range(20)))             # more than capacity: a double free
        bm.reset()
        assert bm.free_count() == 10 and bm.pop(1).tolist() == [0]
    finally:
        bm.close()


def _drive(tr, dp, t, N, scn):
    octx = O.ControlCtx(N, scn.max_sync_rounds, scn.kv_bytes_per_token)

    class Shim:
        def begin(self, req, kv):
            tr.begin_refactor((req, kv))
            r = octx.begin(req, kv)
            assert dp.wave(req, r[1], r[2]) == 0
            return r

        def on_sync_complete(self, req, kv, inflight):
            act, tok = tr.on_kv_sync_complete((req, kv), inflight)
            r = octx.on_sync_complete(req, kv, inflight)
            assert (act, tok) == (r[0], r[1])
            if act != kvx.ACT_BARRIER_WAIT:
                assert dp.wave(req, r[2], r[3]) == 0
            return r

    for _ in replay(Shim(), t):
        pass
    res = tr.on_refactor_commit((t.live_req, t.live_kv))
    ov, row_ptr, blocks, free = dp.commit(t.live_req, t.live_kv)
    assert res.violations == ov == t.violations == 0
    np.testing.assert_array_equal(res.blocks, blocks)
    np.testing.assert_array_equal(res.free_list, free)
    np.testing.assert_array_equal(tr.dst_block_table(), dp.bt)
    return res


def test_chained_refactors_reuse_pools(gpu_count):
    scn = W.load_golden("criterion12")
    t1, t2 = scn.transitions
    N, L = scn.num_requests, scn.num_layers
    heads, dim = 2, 64
    g, og = kvx.geometry(L, heads, dim), O.geo(L, heads, dim)
    tok1, tok2 = t1.max_tokens(N), t2.max_tokens(N)
    max_blocks = int((max(tok1.max(), tok2.max()) + 15) // 16)
    src_bt0, cap0 = W.fragmented_block_table(tok1, max_blocks, 16, seed=3, slack=0.5)
    cap1 = int(((np.maximum(tok1, tok2) + 15) // 16).sum()) + 8
    live1 = np.nonzero(tok1)[0].astype(np.int32)

    # ---- serving pipeline before transition 1 (4 stages) + the 16-stage grant
    pools0 = []
    for b, e in W.stage_ranges(L, t1.old_boundaries):
        p = kvx.Pool(0, g, e - b, cap0)
        p.zero()
        p.fill_pattern(SEED, b, live1, tok1[live1], src_bt0)
        pools0.append(p)
    pools1 = []
    for b, e in W.stage_ranges(L, t1.new_boundaries):
        p = kvx.Pool(0, g, e - b, cap1)
        p.zero()
        pools1.append(p)
    bm1, ref1 = kvx.BlockManager(0, cap1), O.StackBM(cap1)
    dp1 = O.DataPlane(og, t1.old_boundaries, t1.new_boundaries, cap0, cap1, N, max_blocks, src_bt0, bm=ref1)
    dp1.fill_source(SEED, live1, tok1[live1])
    tr1 = kvx.Transition(g, t1.old_boundaries, pools0, t1.new_boundaries, pools1, 0, N, max_blocks, cap1,
                         src_bt0, epoch=t1.epoch, max_sync_rounds=scn.max_sync_rounds,
                         kv_bytes_per_token=scn.kv_bytes_per_token, dst_blockmgr=bm1)
    bm0 = None
    try:
        _drive(tr1, dp1, t1, N, scn)
        np.testing.assert_array_equal(bm1.snapshot(), ref1.snapshot())

        # ---- serving on the 16-stage pipeline until transition 2: decode appends
        table = dp1.bt.copy()
        have = dp1.synced_hi.copy()
        grow = [r for r in range(N) if tok2[r] > have[r]]
        for r in grow:
            need = int((tok2[r] + 15) // 16 - (have[r] + 15) // 16)
            if need > 0:
                ids = bm1.pop(need)
                assert ids.tolist() == ref1.pop(need).tolist()
                nb0 = int((have[r] + 15) // 16)
                table[r, nb0:nb0 + need] = ids
        live2 = np.array(sorted(grow), np.int32)
        if len(live2):
            for k, (b, e) in enumerate(W.stage_ranges(L, t1.new_boundaries)):
                pools1[k].fill_pattern(SEED, b, live2, tok2[live2], table)
            fill = O.DataPlane(og, t1.new_boundaries, t1.new_boundaries, cap1, 1, N, max_blocks, table,
                               old_pools=dp1.new_pools, new_pools=[np.zeros(1, np.uint8)] * 16)
            fill.fill_source(SEED, live2, tok2[live2])

        # ---- transition 2: 16 -> 4 back into the recycled 4-stage pools
        bm0, ref0 = kvx.BlockManager(0, cap0), O.StackBM(cap0)
        dp2 = O.DataPlane(og, t2.old_boundaries, t2.new_boundaries, cap1, cap0, N, max_blocks, table,
                          bm=ref0, old_pools=dp1.new_pools, new_pools=dp1.old_pools)
        tr2 = kvx.Transition(g, t2.old_boundaries, pools1, t2.new_boundaries, pools0, 0, N, max_blocks,
                             cap0, table, epoch=t2.epoch, max_sync_rounds=scn.max_sync_rounds,
                             kv_bytes_per_token=scn.kv_bytes_per_token, dst_blockmgr=bm0)
        try:
            _drive(tr2, dp2, t2, N, scn)
            np.testing.assert_array_equal(bm0.snapshot(), ref0.snapshot())
            for k, p in enumerate(pools0):  # recycled pools: stale bytes + new KV, all equal
                np.testing.assert_array_equal(p.read(), dp2.new_pools[k])
            assert tr2.verify_pattern(SEED, t2.live_req, t2.live_kv) == 0
        finally:
            tr2.close()
    finally:
        tr1.close()
        for p in pools0 + pools1:
            p.close()
        bm1.close()
        if bm0 is not None:
            bm0.close()


def test_abort_with_blockmgr_returns_blocks(gpu_count):
    scn = W.load_golden("engine_revoke")
    (t,) = scn.transitions
    N, L = scn.num_requests, scn.num_layers
    g = kvx.geometry(L, 2, 64)
    tok = t.max_tokens(N)
    max_blocks = int((tok.max() + 15) // 16)
    src_bt, cap0 = W.fragmented_block_table(tok, max_blocks, 16, seed=3)
    live = np.nonzero(tok)[0].astype(np.int32)
    old = []
    for b, e in W.stage_ranges(L, t.old_boundaries):
        p = kvx.Pool(0, g, e - b, cap0)
        p.fill_pattern(SEED, b, live, tok[live], src_bt)
        old.append(p)
    cap1 = int(((tok + 15) // 16).sum())
    new = [kvx.Pool(0, g, e - b, cap1) for b, e in W.stage_ranges(L, t.new_boundaries)]
    bm = kvx.BlockManager(0, cap1)
    ref = O.StackBM(cap1)
    dp = O.DataPlane(O.geo(L, 2, 64), t.old_boundaries, t.new_boundaries, cap0, cap1, N, max_blocks, src_bt,
                     bm=ref, with_pools=False)
    tr = kvx.Transition(g, t.old_boundaries, old, t.new_boundaries, new, 0, N, max_blocks, cap1, src_bt,
                        epoch=t.epoch, dst_blockmgr=bm)
    try:
        w0 = t.waves[0]  # the revoked transition got as far as wave 0
        tr.wave(w0.req, w0.lo, w0.hi)
        assert dp.wave(w0.req, w0.lo, w0.hi) == 0
        assert bm.free_count() == ref.top < cap1
        tr.abort()
        dp.abort()
        assert bm.free_count() == ref.top == cap1
        np.testing.assert_array_equal(bm.snapshot(), ref.snapshot())
    finally:
        tr.close()
        for p in old + new:
            p.close()
        bm.close()


def test_shared_blockmgr_across_streams(gpu_count):
    """Two transitions popping from / pushing to ONE block manager on
    different streams take their ids in host issue order.  B pops 6 ids, A
    pops the next 4 behind a long kernel on its stream, then B's commit frees
    3 ids into exactly the stack slots A popped from.  A must still get the
    ids the host mirror promised (6..9), as the sequential oracle does."""
    import torch
    g = kvx.geometry(2, 1, 8)
    N, max_blocks, cap = 4, 4, 16
    src_bt = np.arange(N * max_blocks, dtype=np.int32).reshape(N, max_blocks)
    old = [kvx.Pool(0, g, 2, N * max_blocks) for _ in range(2)]
    for p in old:
        p.zero()
    new = [kvx.Pool(0, g, 2, cap)]
    new[0].zero()
    # warm-up cycle: every kernel of the path launched once, so no lazy
    # module load (which waits for the device to go idle) can order the
    # streams for us below
    bm = kvx.BlockManager(0, cap)
    tw = kvx.Transition(g, [], [old[0]], [], new, 0, N, max_blocks, cap, src_bt, dst_blockmgr=bm)
    tw.wave(np.array([0, 1], np.int32), np.zeros(2, np.int64), np.array([20, 20], np.int64))
    tw.commit(np.array([0], np.int32), np.array([20], np.int64))
    tw.close()
    bm.close()
    bm, ref = kvx.BlockManager(0, cap), O.StackBM(cap)
    sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
    tA = kvx.Transition(g, [], [old[0]], [], new, 0, N, max_blocks, cap, src_bt, stream=sA.cuda_stream,
                        dst_blockmgr=bm)
    tB = kvx.Transition(g, [], [old[1]], [], new, 0, N, max_blocks, cap, src_bt, stream=sB.cuda_stream,
                        dst_blockmgr=bm)
    try:
        req = np.array([0, 1], np.int32)
        tB.wave(req, np.zeros(2, np.int64), np.array([40, 40], np.int64))   # pops ids 0..5
        tB.wait()
        ref.pop(6)
        with torch.cuda.stream(sA):
            torch.cuda._sleep(int(3e8))                                      # ~150 ms on sA
        tA.wave(np.array([0], np.int32), np.zeros(1, np.int64), np.array([50], np.int64))
        want_a = ref.pop(4)                                                  # 6, 7, 8, 9
        res = tB.commit(np.array([0], np.int32), np.array([40], np.int64))   # request 1 finished
        np.testing.assert_array_equal(res.free_list, [3, 4, 5])
        ref.push(res.free_list)
        tA.wait()
        np.testing.assert_array_equal(tA.dst_block_table()[0], want_a)
        np.testing.assert_array_equal(bm.snapshot(), ref.snapshot())
    finally:
        tA.close()
        tB.close()
        for p in old + new:
            p.close()
        bm.close()
