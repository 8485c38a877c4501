"""Randomised parity: random stage plans (merge, split, uneven re-cut),
geometries, request lengths, wave splits (delta waves with re-synced
overlaps), finished-request sets at commit, bump rule or block manager, LSU
or bulk mover -- GPU bytes, tables, compaction and free lists against the
oracle, bit for bit.  Seeds are fixed so failures reproduce."""
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import kvx
from paper_2510_11938_b200 import workload as W

pytestmark = pytest.mark.gpu


def random_plan(rng, L):
    k = int(rng.integers(1, min(L, 9) + 1))
    cuts = sorted(rng.choice(np.arange(1, L), size=k - 1, replace=False).tolist()) if k > 1 else []
    return cuts


def one_case(seed):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(2, 24))
    elem = int(rng.choice([1, 2, 4]))            # fp8 / fp16 / fp32 KV
    heads = int(rng.choice([1, 2, 4, 8]))
    dim = int(rng.choice([16, 64, 128])) if elem == 1 else int(rng.choice([8, 16, 64, 128]))
    B = int(rng.choice([8, 16, 32]))             # paged-KV block size
    ob, nb = random_plan(rng, L), random_plan(rng, L)
    N = int(rng.integers(1, 80))
    final = rng.integers(0, 200, N).astype(np.int64)
    final[rng.random(N) < 0.15] = 0
    max_blocks = int(max(1, (final.max() + B - 1) // B))
    use_bm = bool(rng.random() < 0.5)
    return rng, L, heads, dim, elem, B, ob, nb, N, final, max_blocks, use_bm


@pytest.mark.parametrize("seed", range(int(os.environ.get("KVX_RANDOM_SEEDS", "40"))))  # soak: more seeds
def test_random_transition_bit_exact(gpu_count, seed, max_ctas=0):
    rng, L, heads, dim, elem, B, ob, nb, N, final, max_blocks, use_bm = one_case(seed)
    g, og = kvx.geometry(L, heads, dim, elem, B), O.geo(L, heads, dim, elem, B)
    src_bt, cap0 = W.fragmented_block_table(final, max_blocks, B, seed=seed, slack=float(rng.random()))
    need = int(((final + B - 1) // B).sum())
    cap1 = max(1, need + int(rng.integers(0, 8)))
    live = np.nonzero(final)[0].astype(np.int32)
    old = []
    for b, e in W.stage_ranges(L, ob):
        p = kvx.Pool(0, g, e - b, cap0)
        p.zero()
        if len(live):
            p.fill_pattern(seed, b, live, final[live], src_bt)
        old.append(p)
    new = []
    for b, e in W.stage_ranges(L, nb):
        p = kvx.Pool(0, g, e - b, cap1)
        p.zero()
        new.append(p)
    bm = kvx.BlockManager(0, cap1) if use_bm else None
    ref_bm = O.StackBM(cap1) if use_bm else None
    if use_bm and rng.random() < 0.5:  # a used manager: some ids popped and pushed back shuffled
        k = int(rng.integers(0, cap1 + 1))
        ids = bm.pop(k)
        assert ids.tolist() == ref_bm.pop(k).tolist()
        ids = rng.permutation(ids)
        bm.push(ids)
        ref_bm.push(ids)
    dp = O.DataPlane(og, ob, nb, cap0, cap1, N, max_blocks, src_bt, bm=ref_bm)
    if len(live):
        dp.fill_source(seed, live, final[live])
    tr = kvx.Transition(g, ob, old, nb, new, 0, N, max_blocks, cap1, src_bt, epoch=1, dst_blockmgr=bm,
                        max_ctas=max_ctas)
    try:
        synced = np.zeros(N, np.int64)
        waves = int(rng.integers(1, 5))
        for w in range(waves):
            target = final if w == waves - 1 else np.minimum(final, synced + rng.integers(0, 90, N))
            req = np.nonzero((target > 0) | (rng.random(N) < 0.3))[0].astype(np.int32)
            lo = synced[req].copy()
            back = rng.integers(0, 20, len(req))          # occasional re-synced overlap
            lo = np.where(rng.random(len(req)) < 0.2, np.maximum(0, lo - back), lo)
            hi = np.maximum(target[req], synced[req])
            tr.wave(req, lo, hi)
            assert dp.wave(req, lo, hi) == 0
            synced[req] = np.maximum(synced[req], hi)
        tr.wait()
        np.testing.assert_array_equal(tr.dst_block_table(), dp.bt)
        for k, p in enumerate(new):
            np.testing.assert_array_equal(p.read(), dp.new_pools[k])
        # commit: some requests finished meanwhile
        alive = live[rng.random(len(live)) < 0.8] if len(live) else live
        res = tr.commit(alive, final[alive])
        v, row_ptr, blocks, free = dp.commit(alive, final[alive])
        assert res.violations == v == 0
        np.testing.assert_array_equal(res.row_ptr, row_ptr)
        np.testing.assert_array_equal(res.blocks, blocks)
        np.testing.assert_array_equal(res.free_list, free)
        if use_bm:
            np.testing.assert_array_equal(bm.snapshot(), ref_bm.snapshot())
    finally:
        tr.close()
        for p in old + new:
            p.close()
        if bm is not None:
            bm.close()


@pytest.mark.parametrize("impl", ["lsu", "bulk"])
def test_movers_agree_on_random_case(gpu_count, impl, monkeypatch):
    """Both movers (KVX_MOVE_IMPL, read at kvx_begin) produce the same bytes."""
    monkeypatch.setenv("KVX_MOVE_IMPL", impl)
    test_random_transition_bit_exact(gpu_count, 101)


@pytest.mark.parametrize("max_ctas", [1, 3, 7])
def test_capped_mover_grid_bit_exact(gpu_count, max_ctas):
    """desc.max_ctas (sharing HBM with serving) only narrows the grid."""
    for seed in (5, 17, 23):
        test_random_transition_bit_exact(gpu_count, seed, max_ctas=max_ctas)
