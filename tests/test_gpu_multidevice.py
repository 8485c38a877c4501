"""One process, several GPUs: a pool of this process on another device is a
peer pool (NVLink, peer access enabled by kvx_begin), and one transition
handle per device moves the layers whose old pool is on it (push) or whose
new pool is on it (pull) -- the single-process analogue of one rank per GPU,
as a single-process engine (the reference's is one) would drive it.  Every
destination byte, block table and commit against the oracle.  With one
visible GPU both 'devices' are device 0 (one handle)."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import kvx
from paper_2510_11938_b200 import shard as S
from paper_2510_11938_b200 import workload as W
from tests.gpu_harness import SEED

pytestmark = pytest.mark.gpu


def run_multidevice(name, heads, dim, placement, pull, gpu_count):
    scn = W.load_golden(name)
    t = scn.transitions[0]
    L, N = scn.num_layers, scn.num_requests
    g = kvx.geometry(L, heads, dim)
    ndev = min(2, gpu_count)
    tokens = t.max_tokens(N)
    max_blocks = int(max(1, (tokens.max() + 15) // 16))
    src_bt, old_blocks = W.fragmented_block_table(tokens, max_blocks, 16, seed=7)
    dst_blocks = max(1, int(((tokens + 15) // 16).sum()))
    live = np.nonzero(tokens)[0].astype(np.int32)
    old_dev, new_dev = S.placement(L, t.old_boundaries, t.new_boundaries, 2, placement)
    old_dev = [d % ndev for d in old_dev]
    new_dev = [d % ndev for d in new_dev]
    old_pools, new_pools = [], []
    for k, (b, e) in enumerate(W.stage_ranges(L, t.old_boundaries)):
        p = kvx.Pool(old_dev[k], g, e - b, old_blocks)
        p.zero()
        p.fill_pattern(SEED, b, live, tokens[live], src_bt)
        old_pools.append(p)
    for j, (b, e) in enumerate(W.stage_ranges(L, t.new_boundaries)):
        p = kvx.Pool(new_dev[j], g, e - b, dst_blocks)
        p.zero()
        new_pools.append(p)
    handles = [kvx.Transition(g, t.old_boundaries, old_pools, t.new_boundaries, new_pools, d, N, max_blocks,
                              dst_blocks, src_bt, epoch=t.epoch, pull=pull) for d in range(ndev)]
    dp = O.DataPlane(O.geo(L, heads, dim), t.old_boundaries, t.new_boundaries, old_blocks, dst_blocks, N,
                     max_blocks, src_bt)
    dp.fill_source(SEED, live, tokens[live])
    try:
        moved = 0
        for w in t.waves:
            for h in handles:
                h.wave(w.req, w.lo, w.hi)
            for h in handles:  # every device's moves land before the next wave (a barrier)
                h.wait()
            assert dp.wave(w.req, w.lo, w.hi) == 0
        for h in handles:
            np.testing.assert_array_equal(h.dst_block_table(), dp.bt)
            moved += h.bytes_moved()
        for k, p in enumerate(new_pools):
            got = p.read()
            want = dp.new_pools[k]
            assert np.array_equal(got, want), f"new stage {k}: {(got != want).sum()} bytes differ"
        if t.outcome == "commit":
            ov, row_ptr, blocks, free = dp.commit(t.live_req, t.live_kv)
            for h in handles:
                res = h.commit(t.live_req, t.live_kv)
                assert res.violations == ov == t.violations
                np.testing.assert_array_equal(res.blocks, blocks)
        return moved
    finally:
        for h in handles:
            h.close()
        for p in old_pools + new_pools:
            p.close()


@pytest.mark.parametrize("pull", [False, True], ids=["push", "pull"])
@pytest.mark.parametrize("placement", ["disjoint", "affinity", "oneway"])
@pytest.mark.parametrize("name,heads,dim", [("criterion12", 2, 64), ("engine_consolidate", 2, 64),
                                            ("llama13b_8to4", 2, 64)])
def test_one_process_two_devices_bit_exact(gpu_count, name, heads, dim, placement, pull):
    run_multidevice(name, heads, dim, placement, pull, gpu_count)


def test_one_process_c1_real_geometry(gpu_count):
    """BASELINE C1 (7B, 4->2) at its real shape, disjoint placement: every layer crosses devices."""
    run_multidevice("llama7b_4to2", 32, 128, "disjoint", False, gpu_count)
