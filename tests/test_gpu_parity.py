"""GPU parity: the kvx CUDA path vs the CPU oracle on the reference's own
transitions (tests/golden).  Bit-exact: block tables, every KV byte of every
destination pool, commit compaction and the Eq. 10 violation count."""
import numpy as np
import pytest

from paper_2510_11938_b200 import kvx
from paper_2510_11938_b200 import workload as W
from tests.gpu_harness import SEED, GpuCase

pytestmark = pytest.mark.gpu

SMALL = [("engine_mid_decode", 2, 64), ("engine_consolidate", 2, 64), ("criterion12", 2, 64),
         ("engine_zero_inflight", 2, 64), ("bursty_repeated", 1, 8), ("delta_rounds_cap", 2, 64),
         ("delta_rounds_converge", 2, 64), ("delta_rounds_zero", 2, 64), ("adaptive_cv4", 1, 8), ("adaptive_cv7", 1, 8)]


def _commit_and_compare(case):
    t = case.t
    res = case.tr.on_refactor_commit((t.live_req, t.live_kv))
    ov, row_ptr, blocks, free = case.dp.commit(t.live_req, t.live_kv)
    assert res.violations == ov == t.violations
    np.testing.assert_array_equal(res.row_ptr, row_ptr)
    np.testing.assert_array_equal(res.blocks, blocks)
    np.testing.assert_array_equal(res.free_list, free)
    return res


@pytest.mark.parametrize("name,heads,dim", SMALL)
def test_small_goldens_bit_exact(gpu_count, name, heads, dim):
    scn = W.load_golden(name)
    for t in scn.transitions:
        case = GpuCase(scn, t, heads, dim)
        try:
            case.compare_source()          # device fill == kvo_fill pattern
            case.run_ctl()
            case.compare_tables()
            case.compare_bytes()
            if t.outcome == "commit":
                _commit_and_compare(case)
                assert case.tr.verify_pattern(SEED, t.live_req, t.live_kv) == 0
                assert case.dp.verify(SEED, t.live_req, t.live_kv) == 0
        finally:
            case.close()


def test_c1_llama7b_4to2_full_bytes(gpu_count):
    """BASELINE config 1 at its real shape (32 layers, 32 KV heads, d=128,
    ~4k tokens = 2 GiB): every destination byte compared with the oracle."""
    scn = W.load_golden("llama7b_4to2")
    (t,) = scn.transitions
    case = GpuCase(scn, t, 32, 128)
    try:
        case.compare_source()
        case.run_ctl()
        case.compare_tables()
        case.compare_bytes()
        _commit_and_compare(case)
    finally:
        case.close()


@pytest.mark.parametrize("name", ["llama13b_8to4", "llama7b_2to8", "llama70b_8to2to8"])
def test_full_size_properties(gpu_count, name):
    """BASELINE configs 2-4 at full size (C3: 17 GB, C2: 69 GB of live KV):
    the oracle replays the block rule (allocation-only), then EVERY byte of
    every destination pool is compared with the oracle's image of it, one
    layer at a time (kvo_fill_layer over the oracle's destination table:
    payload on synced rows, zeros on partial-block tails, spare and unused
    blocks).  A single stray byte anywhere in a pool fails the test
    (test_full_size_compare_catches_a_stray_byte)."""
    scn = W.load_golden(name)
    L, H, D = W.shape_for(scn)
    for t in scn.transitions:
        case = GpuCase(scn, t, H, D, oracle_pools=False)
        try:
            case.run_ctl()
            case.compare_tables()
            case.compare_bytes_by_layer()
            res = _commit_and_compare(case)
            assert res.violations == 0
            moved = sum(int((w.hi - w.lo).clip(min=0).sum()) for w in t.waves)
            assert case.tr.bytes_moved() == moved * 2 * case.g.token_bytes * L
        finally:
            case.close()


@pytest.mark.parametrize("where", ["tail", "spare", "live"])
def test_full_size_compare_catches_a_stray_byte(gpu_count, where):
    """The layer-by-layer oracle compare fails on one flipped byte in a row no
    wave writes (a partial block's tail rows, a spare block past the last
    allocated one) as well as in a live row."""
    scn = W.load_golden("criterion12")
    t = [x for x in scn.transitions if x.outcome == "commit"][-1]
    case = GpuCase(scn, t, 2, 64, oracle_pools=False, dst_blocks=None)
    try:
        case.run_ctl()
        case.tr.wait()
        case.compare_bytes_by_layer()             # clean
        g, B = case.g, 16
        r = int(np.argmax(case.dp.synced_hi % B))  # a request whose last block is partial
        s = int(case.dp.synced_hi[r])
        assert s % B, "the scenario has a partial block"
        blk = int(case.dp.bt[r, s // B])
        if where == "tail":
            off = blk * g.block_bytes + (s % B) * g.token_bytes        # K row just past the last token
        elif where == "spare":
            used = int((case.dp.bt >= 0).sum())
            assert used <= case.dst_blocks
            off = (case.dst_blocks - 1) * g.block_bytes + 7 if used < case.dst_blocks else \
                blk * g.block_bytes + g.block_bytes - 1                 # V row tail of the partial block
        else:
            off = int(case.dp.bt[r, 0]) * g.block_bytes + 3
        p = case.new_pools[0]
        old = p.read(off, 1)
        p.write(np.array([old[0] ^ 0x5A], np.uint8), off)
        with pytest.raises(AssertionError):
            case.compare_bytes_by_layer()
    finally:
        case.close()


def test_c4_same_k_replacement_full_size(gpu_count):
    """BASELINE config 4: every 10-layer stage of the 80-layer 70B-GQA model
    re-placed (same boundaries on both sides) -- no reference path
    (engine.cpp:562), so the oracle restatement is the only pin: block table
    identical to the oracle's, every live word equal to the payload."""
    import copy
    scn = W.load_golden("llama70b_8to2to8")
    t = copy.copy([x for x in scn.transitions if x.outcome == "commit"][-1])
    t.old_boundaries = list(t.new_boundaries)
    assert len(t.old_boundaries) == 7
    case = GpuCase(scn, t, 8, 128, oracle_pools=False)
    try:
        case.run_ctl()
        case.compare_tables()
        case.compare_bytes_by_layer()
        res = _commit_and_compare(case)
        assert res.violations == 0
    finally:
        case.close()


def test_c5_adaptive_chain_full_shape(gpu_count):
    """BASELINE config 5: the reference controller's own refactor chain on a
    gamma trace (CV=7, tests/golden/adaptive_cv7.jsonl: 4->16, then 16<->8
    re-cuts chosen by Alg. 1) at the Llama-2-7B shape.  Every third
    transition whose source + destination footprint fits one GPU (the largest
    touches ~300k token slots, ~150 GB per side) is moved at full size:
    tables and compaction equal the oracle's, every live word equals the
    payload, moved bytes equal the waves' token sum.  All 39 are compared
    byte for byte at a small geometry in test_small_goldens_bit_exact."""
    scn = W.load_golden("adaptive_cv7")
    L, H, D = W.SHAPES["llama2-7b"]
    token_bytes = 2 * H * D * 2
    ran = 0
    for t in scn.transitions[::3]:
        if int(t.max_tokens(scn.num_requests).sum()) * token_bytes * L * 2 > 60e9:
            continue
        case = GpuCase(scn, t, H, D, oracle_pools=False)
        try:
            case.run_ctl()
            case.compare_tables()
            res = _commit_and_compare(case)
            assert res.violations == 0
            assert case.tr.verify_pattern(SEED, t.live_req, t.live_kv) == 0
            moved = sum(int((w.hi - w.lo).clip(min=0).sum()) for w in t.waves)
            assert case.tr.bytes_moved() == moved * 2 * case.g.token_bytes * L
            ran += 1
        finally:
            case.close()
    assert ran >= 8


