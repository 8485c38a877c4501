"""Waves overlap serving: while wave 0 moves [0, T0) of
every request, the serving pipeline keeps appending decode tokens
[T0, T1) into the SAME source pools on another stream.  KV is append-only
(engine.cpp:494-499) and a wave copies only [synced, target), so the
concurrent writer never disturbs it; the delta wave then picks the new
tokens up.  Bytes and tables against the oracle, payload on the device."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import kvx
from paper_2510_11938_b200 import workload as W

pytestmark = pytest.mark.gpu
SEED = 0x0E1A


def test_waves_overlap_decode_appends(gpu_count):
    import torch
    L, H, D, N = 16, 8, 128, 96
    ob, nb = [4, 8, 12], [8]                      # 4 -> 2 merge
    rng = np.random.default_rng(1)
    t0 = rng.integers(20, 300, N).astype(np.int64)
    t1 = t0 + rng.integers(1, 40, N)
    max_blocks = int((t1.max() + 15) // 16)
    src_bt, cap0 = W.fragmented_block_table(t1, max_blocks, 16, seed=2)
    cap1 = int(((t1 + 15) // 16).sum())
    g, og = kvx.geometry(L, H, D), O.geo(L, H, D)
    req = np.arange(N, dtype=np.int32)
    old = []
    for b, e in W.stage_ranges(L, ob):
        p = kvx.Pool(0, g, e - b, cap0)
        p.zero()
        p.fill_pattern(SEED, b, req, t0, src_bt)   # serving state at wave 0
        old.append(p)
    new = []
    for b, e in W.stage_ranges(L, nb):
        p = kvx.Pool(0, g, e - b, cap1)
        p.zero()
        new.append(p)
    tr = kvx.Transition(g, ob, old, nb, new, 0, N, max_blocks, cap1, src_bt, epoch=1)
    side = torch.cuda.Stream()
    try:
        torch.cuda.synchronize()
        tr.wave(req, np.zeros(N, np.int64), t0)             # wave 0 on the transition stream
        for k, (b, e) in enumerate(W.stage_ranges(L, ob)):  # decode appends, concurrently
            old[k].append_pattern(SEED, b, req, t0, t1, src_bt, stream=side.cuda_stream)
        tr.wait()
        side.synchronize()
        tr.wave(req, t0, t1)                                 # delta wave: the appended tokens
        res = tr.commit(req, t1)
        assert res.violations == 0
        assert tr.verify_pattern(SEED, req, t1) == 0
        dp = O.DataPlane(og, ob, nb, cap0, cap1, N, max_blocks, src_bt)
        dp.fill_source(SEED, req, t1)
        assert dp.wave(req, np.zeros(N, np.int64), t0) == 0 and dp.wave(req, t0, t1) == 0
        np.testing.assert_array_equal(tr.dst_block_table(), dp.bt)
        for k, p in enumerate(new):
            np.testing.assert_array_equal(p.read(), dp.new_pools[k])
        for k, p in enumerate(old):                          # the writer's output is the payload too
            np.testing.assert_array_equal(p.read(), dp.old_pools[k])
    finally:
        tr.close()
        for p in old + new:
            p.close()
