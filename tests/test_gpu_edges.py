"""Edge cases of the kvx C-ABI on the GPU: empty / zero-length waves, block
boundaries, maximum sizes, stale epochs, out-of-order calls, abort."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import kvx
from paper_2510_11938_b200 import workload as W

pytestmark = pytest.mark.gpu
SEED = 99


class Mini:
    """4 layers, 2 old stages -> 3 new stages, 4 requests."""

    def __init__(self, tokens, max_blocks=4, dst_blocks=None, heads=2, dim=64):
        self.g = kvx.geometry(4, heads, dim)
        self.tokens = np.asarray(tokens, np.int64)
        self.N = len(tokens)
        self.max_blocks = max_blocks
        self.src_bt, self.old_blocks = W.fragmented_block_table(self.tokens, max_blocks, 16, seed=3)
        need = int(((self.tokens + 15) // 16).sum())
        self.dst_blocks = dst_blocks or max(need, 1)
        self.ob, self.nb = [2], [1, 3]
        live = np.nonzero(self.tokens)[0]
        self.old = []
        for b, e in W.stage_ranges(4, self.ob):
            p = kvx.Pool(0, self.g, e - b, self.old_blocks)
            p.zero()
            p.fill_pattern(SEED, b, live, self.tokens[live], self.src_bt)
            self.old.append(p)
        self.new = [kvx.Pool(0, self.g, e - b, self.dst_blocks) for b, e in W.stage_ranges(4, self.nb)]
        for p in self.new:
            p.zero()
        self.tr = kvx.Transition(self.g, self.ob, self.old, self.nb, self.new, 0, self.N,
                                 max_blocks, self.dst_blocks, self.src_bt, epoch=5)
        og = O.geo(4, heads, dim)
        self.dp = O.DataPlane(og, self.ob, self.nb, self.old_blocks, self.dst_blocks, self.N,
                              max_blocks, self.src_bt)
        self.dp.fill_source(SEED, live, self.tokens[live])

    def wave(self, req, lo, hi):
        self.tr.wave(req, lo, hi)
        assert self.dp.wave(req, lo, hi) == 0

    def check(self):
        self.tr.wait()
        np.testing.assert_array_equal(self.tr.dst_block_table(), self.dp.bt)
        for k, p in enumerate(self.new):
            np.testing.assert_array_equal(p.read(), self.dp.new_pools[k])

    def close(self):
        self.tr.close()
        for p in self.old + self.new:
            p.close()


def test_empty_and_zero_length_waves(gpu_count):
    m = Mini([0, 5, 16, 0])
    try:
        m.wave([], [], [])
        m.wave([0, 1, 2, 3], [0, 0, 0, 0], [0, 0, 0, 0])
        m.check()
        assert m.tr.bytes_moved() == 0
        m.wave([1, 2], [0, 0], [5, 16])
        m.check()
    finally:
        m.close()


def test_block_boundaries_and_single_tokens(gpu_count):
    m = Mini([64, 33, 17, 1], max_blocks=4)
    try:
        m.wave([0, 1, 2, 3], [0, 0, 0, 0], [15, 16, 16, 1])    # ends exactly on / inside blocks
        m.wave([0, 1, 2], [15, 16, 16], [16, 17, 17])          # single-token tails
        m.wave([0, 1], [16, 17], [64, 33])                     # max_blocks exactly filled
        m.check()
        res = m.tr.commit([0, 1, 2, 3], [64, 33, 17, 1])
        v, row_ptr, blocks, free = m.dp.commit([0, 1, 2, 3], [64, 33, 17, 1])
        assert res.violations == v == 0
        np.testing.assert_array_equal(res.blocks, blocks)
    finally:
        m.close()


def test_overlapping_resync_is_idempotent(gpu_count):
    m = Mini([40, 20, 0, 0])
    try:
        m.wave([0, 1], [0, 0], [30, 20])
        m.wave([0], [10], [40])   # lo < synced: re-copies [10,30), appends [30,40)
        m.check()
    finally:
        m.close()


def test_errors(gpu_count):
    m = Mini([40, 20, 0, 0], max_blocks=3)
    try:
        with pytest.raises(kvx.KvxError) as e:
            m.tr.wave([1, 0], [0, 0], [1, 1])                   # not ascending
        assert e.value.code == kvx.KVX_EINVAL
        with pytest.raises(kvx.KvxError) as e:
            m.tr.wave([0], [8], [16])                            # gap: lo > synced
        assert e.value.code == kvx.KVX_EINVAL
        with pytest.raises(kvx.NoSpace):
            m.tr.wave([0], [0], [49])                            # 4 blocks > max_blocks 3
        with pytest.raises(kvx.StaleEpoch):
            m.tr.wave([0], [0], [1], epoch=4)
        with pytest.raises(kvx.KvxError) as e:
            m.tr.wave([2], [0], [5])                             # request 2 has no source blocks
        assert e.value.code == kvx.KVX_EINVAL
        m.wave([0], [0], [40])
        res = m.tr.commit([0, 1], [40, 20])
        assert res.violations == 1                               # request 1 never synced
        with pytest.raises(kvx.StaleEpoch):
            m.tr.wave([1], [0], [20], epoch=5)                   # commit bumped the epoch
        with pytest.raises(kvx.KvxError) as e:
            m.tr.wave([1], [0], [20], epoch=6)
        assert e.value.code == kvx.KVX_ESTATE
    finally:
        m.close()


def test_destination_full_is_enospc(gpu_count):
    m = Mini([48, 48, 0, 0], dst_blocks=4)
    try:
        m.wave([0], [0], [48])                                   # 3 blocks
        with pytest.raises(kvx.NoSpace):
            m.tr.wave([1], [0], [32])                            # 2 more > 4
        m.check()                                                # nothing half-applied
    finally:
        m.close()


def test_refused_control_wave_leaves_the_mirror_untouched(gpu_count):
    """A delta wave refused for space (KVX_ENOSPC -> the engine holds or
    aborts) must not leave targets behind: request 1 never moved, so the
    commit's Eq. 10 counts it as a violation, on the device and the mirror."""
    m = Mini([48, 32, 0, 0], dst_blocks=4)
    try:
        live0 = (np.array([0], np.int32), np.array([48], np.int64))
        live01 = (np.array([0, 1], np.int32), np.array([48, 32], np.int64))
        m.tr.begin_refactor(live0)                                    # 3 blocks
        before = m.tr.ctl_state()
        with pytest.raises(kvx.NoSpace):
            m.tr.on_kv_sync_complete(live01, 0)                       # delta needs 2 more > 4
        after = m.tr.ctl_state()
        assert (after["rounds"], after["waves"], after["kv_synced_bytes"]) == \
               (before["rounds"], before["waves"], before["kv_synced_bytes"])
        act, tok = m.tr.on_kv_sync_complete(live0, 0)                 # request 1 dropped meanwhile
        assert act == kvx.ACT_FINAL and tok == 0
        res = m.tr.on_refactor_commit(live01)                         # but it is live at commit
        assert res.violations == 1
    finally:
        m.close()


def test_abort_drops_destination_and_invalidates_epoch(gpu_count):
    m = Mini([40, 20, 0, 0])
    try:
        m.tr.wave([0, 1], [0, 0], [40, 20])
        m.tr.abort()
        assert m.tr.epoch == 6
        assert (m.tr.dst_block_table() == -1).all()
        with pytest.raises(kvx.KvxError):
            m.tr.wave([0], [0], [1])
        # source pools untouched: a fresh transition over them succeeds
        tr2 = kvx.Transition(m.g, m.ob, m.old, m.nb, m.new, 0, m.N, m.max_blocks, m.dst_blocks,
                             m.src_bt, epoch=7)
        tr2.wave([0, 1], [0, 0], [40, 20])
        assert m.dp.wave([0, 1], [0, 0], [40, 20]) == 0
        tr2.wait()
        np.testing.assert_array_equal(tr2.dst_block_table(), m.dp.bt)
        for k, p in enumerate(m.new):
            np.testing.assert_array_equal(p.read(), m.dp.new_pools[k])
        tr2.close()
    finally:
        m.close()


def test_commit_frees_finished_requests(gpu_count):
    m = Mini([40, 20, 33, 0])
    try:
        m.wave([0, 1, 2], [0, 0, 0], [40, 20, 33])
        res = m.tr.commit([0, 2], [40, 33])                      # request 1 finished meanwhile
        v, row_ptr, blocks, free = m.dp.commit([0, 2], [40, 33])
        assert res.violations == v == 0
        np.testing.assert_array_equal(res.row_ptr, row_ptr)
        np.testing.assert_array_equal(res.free_list, free)
        assert len(res.free_list) == 2
    finally:
        m.close()


def test_launch_counter_moves(gpu_count):
    before = kvx.launch_count()
    m = Mini([16, 0, 0, 0])
    try:
        m.wave([0], [0], [16])
        m.check()
    finally:
        m.close()
    assert kvx.launch_count() >= before + 2


def test_device_bounds_check_catches_unbacked_source(gpu_count):
    """With the host's per-wave source check bypassed (test hook, read at the
    first wave of the process -- so run in a subprocess), a wave over a
    request with no source blocks reaches the plan kernel, which neutralises
    the segments and reports KVX_ECUDA at wait."""
    import subprocess
    import sys
    code = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"])
from tests.test_gpu_edges import Mini
from paper_2510_11938_b200 import kvx
m = Mini([40, 20, 0, 0])
m.tr.wave([2], [0], [5])            # request 2 has no source blocks: ids are -1
try:
    m.tr.wait()
    print("NOT CAUGHT")
except kvx.KvxError as e:
    print("CAUGHT", e.code, "bounds" in str(e))
m.close()
'''
    import os
    env = dict(os.environ, KVX_TEST_SKIP_HOST_CHECKS="1",
               ROOT=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert "CAUGHT -4 True" in out.stdout, out.stdout + out.stderr


def test_request_longer_than_grid_y(gpu_count):
    """One request of 1.1M tokens = 68,750 blocks (> 65,535, the grid.y
    limit of the payload kernels, which stride over blocks): fill, move,
    commit and verify, bytes compared with the oracle."""
    L, T = 2, 1_100_000
    g, og = kvx.geometry(L, 1, 8), O.geo(L, 1, 8)          # 16 B tokens, 512 B blocks
    mb = (T + 15) // 16
    tokens = np.array([T], np.int64)
    src_bt, cap0 = W.fragmented_block_table(tokens, mb, 16, seed=5, slack=0.0)
    live = np.array([0], np.int32)
    old = [kvx.Pool(0, g, 1, cap0) for _ in range(2)]
    for k, p in enumerate(old):
        p.zero()
        p.fill_pattern(SEED, k, live, tokens, src_bt)
    new = [kvx.Pool(0, g, L, mb)]
    new[0].zero()
    tr = kvx.Transition(g, [1], old, [], new, 0, 1, mb, mb, src_bt)
    dp = O.DataPlane(og, [1], [], cap0, mb, 1, mb, src_bt)
    dp.fill_source(SEED, live, tokens)
    try:
        tr.wave(live, [0], [T])
        assert dp.wave(live, [0], [T]) == 0
        tr.wait()
        np.testing.assert_array_equal(new[0].read(), dp.new_pools[0])
        assert tr.commit(live, tokens).violations == 0
        assert tr.verify_pattern(SEED, live, tokens) == 0
    finally:
        tr.close()
        for p in old + new:
            p.close()


def test_many_requests(gpu_count):
    """200,000 live requests in two waves (the single-CTA plan and commit
    kernels loop over entries and blocks): tables, bytes, compaction and the
    free list equal the oracle's."""
    L, N = 2, 200_000
    rng = np.random.default_rng(42)
    g, og = kvx.geometry(L, 1, 8), O.geo(L, 1, 8)
    final = rng.integers(1, 40, N).astype(np.int64)
    mb = int((final.max() + 15) // 16)
    src_bt, cap0 = W.fragmented_block_table(final, mb, 16, seed=9, slack=0.1)
    cap1 = int(((final + 15) // 16).sum())
    live = np.arange(N, dtype=np.int32)
    old = [kvx.Pool(0, g, 1, cap0) for _ in range(2)]
    for k, p in enumerate(old):
        p.zero()
        p.fill_pattern(SEED, k, live, final, src_bt)
    new = [kvx.Pool(0, g, L, cap1)]
    new[0].zero()
    tr = kvx.Transition(g, [1], old, [], new, 0, N, mb, cap1, src_bt)
    dp = O.DataPlane(og, [1], [], cap0, cap1, N, mb, src_bt)
    dp.fill_source(SEED, live, final)
    try:
        half = final // 2
        tr.wave(live, np.zeros(N, np.int64), half)
        assert dp.wave(live, np.zeros(N, np.int64), half) == 0
        tr.wave(live, half, final)
        assert dp.wave(live, half, final) == 0
        tr.wait()
        np.testing.assert_array_equal(tr.dst_block_table(), dp.bt)
        np.testing.assert_array_equal(new[0].read(), dp.new_pools[0])
        alive = live[rng.random(N) < 0.7]
        res = tr.commit(alive, final[alive])
        v, row_ptr, blocks, free = dp.commit(alive, final[alive])
        assert res.violations == v == 0
        np.testing.assert_array_equal(res.row_ptr, row_ptr)
        np.testing.assert_array_equal(res.blocks, blocks)
        np.testing.assert_array_equal(res.free_list, free)
    finally:
        tr.close()
        for p in old + new:
            p.close()
