"""ABI 4 serving-side calls on the GPU: stream-ordered block-manager pop/push
with device id arrays, and a grant whose source block table is the serving
engine's device copy (no host table, no host scan) -- bit-exact against the
oracle, same as the host-table grant."""
import numpy as np
import pytest

from paper_2510_11938_b200 import kvx
from paper_2510_11938_b200 import workload as W
from tests.gpu_harness import GpuCase

pytestmark = pytest.mark.gpu


def test_bm_async_pop_push_match_host_semantics(gpu_count):
    import torch
    cap = 64
    a, b = kvx.BlockManager(0, cap), kvx.BlockManager(0, cap)
    s = torch.cuda.Stream()
    try:
        ids = torch.full((10,), -7, dtype=torch.int32, device="cuda")
        a.pop_async(10, ids.data_ptr(), s.cuda_stream)
        want = b.pop(10)                          # host pop: LIFO order
        s.synchronize()
        np.testing.assert_array_equal(ids.cpu().numpy(), want)
        assert a.free_count() == b.free_count() == cap - 10
        # push back in a different order, on the stream; snapshots agree
        back = torch.flip(ids, [0]).contiguous()
        a.push_async(10, back.data_ptr(), s.cuda_stream)
        b.push(want[::-1].copy())
        np.testing.assert_array_equal(a.snapshot(), b.snapshot())
        assert a.free_count() == cap
        # an id outside [0, capacity) is dropped on the device and reported next call
        a.pop(1)
        bad = torch.tensor([cap + 5], dtype=torch.int32, device="cuda")
        a.push_async(1, bad.data_ptr(), s.cuda_stream)
        s.synchronize()
        with pytest.raises(kvx.KvxError):
            a.pop(1)
        with pytest.raises(kvx.NoSpace):
            b.pop_async(cap + 1, ids.data_ptr(), s.cuda_stream)
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("name", ["llama7b_4to2", "engine_consolidate", "delta_rounds_cap"])
def test_device_source_table_bit_exact(gpu_count, name):
    scn = W.load_golden(name)
    t = scn.transitions[0]
    heads, dim = (32, 128) if name == "llama7b_4to2" else (2, 64)
    case = GpuCase(scn, t, heads, dim, dev_table=True)
    try:
        case.run_ctl()
        res = case.tr.on_refactor_commit((t.live_req, t.live_kv))
        v, row_ptr, blocks, free = case.dp.commit(t.live_req, t.live_kv)
        assert res.violations == v == t.violations
        np.testing.assert_array_equal(res.blocks, blocks)
        case.compare_tables()
        case.compare_bytes()
    finally:
        case.close()


def test_device_table_bad_id_fails_on_the_device(gpu_count):
    """No host scan with a device table: an id beyond the old pools is caught by
    the plan kernel's bounds check and reported by kvx_wait (KVX_ECUDA)."""
    import torch
    scn = W.load_golden("engine_consolidate")
    t = scn.transitions[0]
    case = GpuCase(scn, t, 2, 64, oracle=False, dev_table=True)
    try:
        r = int(case.live[0])
        case.dev_bt[r, 0] = case.old_blocks + 3
        torch.cuda.synchronize()
        case.tr.close()
        case.tr = kvx.Transition(case.g, t.old_boundaries, case.old_pools, t.new_boundaries, case.new_pools, 0,
                                 case.N, case.max_blocks, case.dst_blocks, None, epoch=t.epoch,
                                 src_block_table_dev=case.dev_bt.data_ptr())
        case.tr.wave(np.array([r], np.int32), np.zeros(1, np.int64), np.array([case.tokens[r]], np.int64))
        with pytest.raises(kvx.KvxError) as e:
            case.tr.wait()
        assert e.value.code == kvx.KVX_ECUDA
    finally:
        case.close()
