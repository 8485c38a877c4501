"""KV layouts either side of the transition: old and new pools in the block
layout ([blocks][2][B][H][D] per layer, FlashInfer's NHD paged cache), the K/V
plane layout ([2][blocks][B][H][D] per layer, FlashAttention's) or the
head-major layout ([blocks][2][H][B][D], FlashInfer HND -- what vLLM's
FlashInfer backend requires on B200; token-major <-> head-major moves go
through the transposing mover), single
allocations or one caller-owned tensor per layer (kvx_pool_wrap_layers).  A
refactor then also converts the cache between backends.  The oracle works in
the block layout; a layout is a permutation of the same bytes, so every pool
is compared with the oracle's pool permuted into its layout, bit for bit."""
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import kvx
from paper_2510_11938_b200 import workload as W
from tests.test_gpu_random import one_case

pytestmark = pytest.mark.gpu


def in_layout(block_bytes_arr: np.ndarray, layers: int, blocks: int, layout: int, B: int = 16,
              heads: int = 1) -> np.ndarray:
    """Oracle pool bytes (block layout [L][blocks][2][B][H][D]) -> the same
    bytes in `layout`, shaped [layer, -1]."""
    a = block_bytes_arr.reshape(layers, blocks, 2, B, heads, -1)
    if layout == kvx.LAYOUT_KV_PLANES:
        a = a.transpose(0, 2, 1, 3, 4, 5)
    elif layout == kvx.LAYOUT_HEADS:
        a = a.transpose(0, 1, 2, 4, 3, 5)
    return np.ascontiguousarray(a).reshape(layers, -1)


class LayerTensors:
    """One torch uint8 tensor per layer, wrapped as one kvx pool."""

    def __init__(self, torch, g, layers, blocks, layout):
        self.t = [torch.zeros(blocks * g.block_bytes, dtype=torch.uint8, device="cuda:0") for _ in range(layers)]
        self.pool = kvx.Pool.wrap_layers(0, [x.data_ptr() for x in self.t], blocks * g.block_bytes, g, blocks,
                                         layout)

    def read(self):
        return np.stack([x.cpu().numpy() for x in self.t])


def make_pool(torch, rng, g, layers, blocks, allow_wrap, layout=None):
    layout = int(rng.integers(0, 3)) if layout is None else layout
    if allow_wrap and rng.random() < 0.5:
        lt = LayerTensors(torch, g, layers, blocks, layout)
        return lt.pool, lt.read, layout, lt
    p = kvx.Pool(0, g, layers, blocks, layout)
    p.zero()
    return p, (lambda p=p: p.read().reshape(layers, -1)), layout, None


@pytest.mark.parametrize("seed", range(int(os.environ.get("KVX_LAYOUT_SEEDS", "24"))))  # soak: more seeds
def test_random_layouts_bit_exact(gpu_count, seed, uniform=None):
    """uniform = (old layout, new layout) for every stage; None = random per stage."""
    import torch
    rng, L, heads, dim, elem, B, ob, nb, N, final, max_blocks, use_bm = one_case(1000 + seed)
    g, og = kvx.geometry(L, heads, dim, elem, B), O.geo(L, heads, dim, elem, B)
    src_bt, cap0 = W.fragmented_block_table(final, max_blocks, B, seed=seed, slack=float(rng.random()))
    cap1 = max(1, int(((final + B - 1) // B).sum()) + int(rng.integers(0, 8)))
    live = np.nonzero(final)[0].astype(np.int32)
    keep, old, old_read, old_lay = [], [], [], []
    for b, e in W.stage_ranges(L, ob):
        p, rd, lay, k = make_pool(torch, rng, g, e - b, cap0, allow_wrap=True,
                                  layout=None if uniform is None else uniform[0])
        if len(live):
            p.fill_pattern(seed, b, live, final[live], src_bt)
        old.append(p), old_read.append(rd), old_lay.append(lay), keep.append(k)
    new, new_read, new_lay = [], [], []
    for b, e in W.stage_ranges(L, nb):
        p, rd, lay, k = make_pool(torch, rng, g, e - b, cap1, allow_wrap=True,
                                  layout=None if uniform is None else uniform[1])
        new.append(p), new_read.append(rd), new_lay.append(lay), keep.append(k)
    torch.cuda.synchronize()
    dp = O.DataPlane(og, ob, nb, cap0, cap1, N, max_blocks, src_bt)
    if len(live):
        dp.fill_source(seed, live, final[live])
    for k, (b, e) in enumerate(W.stage_ranges(L, ob)):      # payload written in each pool's layout
        np.testing.assert_array_equal(old_read[k](), in_layout(dp.old_pools[k], e - b, cap0, old_lay[k], B, heads))
    tr = kvx.Transition(g, ob, old, nb, new, 0, N, max_blocks, cap1, src_bt, epoch=1)
    try:
        synced = np.zeros(N, np.int64)
        waves = int(rng.integers(1, 4))
        for w in range(waves):
            target = final if w == waves - 1 else np.minimum(final, synced + rng.integers(0, 90, N))
            req = np.nonzero(target > synced)[0].astype(np.int32)
            lo = synced[req].copy()
            back = rng.integers(0, 20, len(req))                 # re-synced overlaps (partial blocks)
            lo = np.where(rng.random(len(req)) < 0.2, np.maximum(0, lo - back), lo)
            hi = target[req]
            tr.wave(req, lo, hi)
            assert dp.wave(req, lo, hi) == 0
            synced[req] = np.maximum(synced[req], hi)
        tr.wait()
        np.testing.assert_array_equal(tr.dst_block_table(), dp.bt)
        for k, (b, e) in enumerate(W.stage_ranges(L, nb)):
            np.testing.assert_array_equal(new_read[k](), in_layout(dp.new_pools[k], e - b, cap1, new_lay[k], B, heads),
                                          err_msg=f"new stage {k} (layout {new_lay[k]})")
        res = tr.commit(live, final[live])
        assert res.violations == 0
        assert tr.verify_pattern(seed, live, final[live]) == 0
    finally:
        tr.close()
        for p in old + new:
            p.close()


@pytest.mark.parametrize("impl", ["lsu", "lsu256"])
def test_lsu_movers_convert_layouts(gpu_count, impl, monkeypatch):
    """The LSU movers (KVX_MOVE_IMPL) honour the layouts too."""
    monkeypatch.setenv("KVX_MOVE_IMPL", impl)
    for seed in (3, 7):
        test_random_layouts_bit_exact(gpu_count, seed)


@pytest.mark.parametrize("pair", [(2, 2), (0, 2), (2, 0), (1, 2), (2, 1)],
                         ids=["heads", "blocks-to-heads", "heads-to-blocks", "planes-to-heads", "heads-to-planes"])
@pytest.mark.parametrize("impl", ["bulk", "lsu"])
def test_head_major_layouts(gpu_count, pair, impl, monkeypatch):
    """Head-major pools on every stage of one side or both: head-major to
    head-major through run copies (2*H runs per partial block), the rest
    through the transposing row mover."""
    monkeypatch.setenv("KVX_MOVE_IMPL", impl)
    for seed in (11, 12, 13):
        test_random_layouts_bit_exact(gpu_count, seed, uniform=pair)


@pytest.mark.parametrize("pair", [(0, 2), (2, 0), (1, 2), (2, 1)],
                         ids=["blocks-to-heads", "heads-to-blocks", "planes-to-heads", "heads-to-planes"])
@pytest.mark.parametrize("tmap", ["on", "off"])
def test_transposes_tmap_and_row_mover(gpu_count, pair, tmap, monkeypatch):
    """Every transposing pairing with the TMA tensor-map transposer for whole
    blocks (the default) and without it (KVX_TMAP=0: the row mover moves all)."""
    monkeypatch.setenv("KVX_TMAP", "1" if tmap == "on" else "0")
    for seed in range(20, 28):
        test_random_layouts_bit_exact(gpu_count, seed, uniform=pair)
