"""GPU stage-boundary activation handoff vs the oracle plan: every in-flight
micro-batch the reference leaves at a barrier lands, byte-identical, in the
arena of the new stage that owns its resume layer."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import workload as W
from paper_2510_11938_b200 import kvx
from tests.gpu_harness import SEED, GpuCase
from tests.test_handoff_oracle import CASES

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,ti,t,b", CASES, ids=[f"{c[0]}-{c[1]}" for c in CASES])
def test_handoff_bit_exact(gpu_count, name, ti, t, b):
    import torch
    scn = W.load_golden(name)
    case = GpuCase(scn, t, 1, 8, oracle=False)
    try:
        row = 1024 if name.startswith(("engine", "criterion")) else 5120 * 2
        torch.manual_seed(ti)
        srcs = [torch.randint(0, 256, (max(m.tokens, 1) * row,), dtype=torch.uint8, device="cuda")
                for m in b.microbatches]
        after = [m.after for m in b.microbatches]
        tokens = [m.tokens for m in b.microbatches]
        total = sum(m.tokens * row + 256 for m in b.microbatches) + 256
        arenas = [torch.zeros(total, dtype=torch.uint8, device="cuda")
                  for _ in range(len(t.new_boundaries) + 1)]
        torch.cuda.synchronize()
        slots = case.tr.handoff(row, [(m.batch, m.after, m.tokens, s.data_ptr())
                                      for m, s in zip(b.microbatches, srcs)],
                                [a.data_ptr() for a in arenas], [total] * len(arenas))
        case.tr.wait()
        rc, ns, rl, off, by = O.handoff_plan(t.old_boundaries, t.new_boundaries, row, after, tokens,
                                             [total] * len(arenas))
        assert rc == 0
        for i, (bid, k, layer, o, nbytes) in enumerate(slots):
            assert (bid, k, layer, o, nbytes) == (b.microbatches[i].batch, ns[i], rl[i], off[i], by[i])
            if nbytes:
                got = arenas[k][o:o + nbytes].cpu().numpy()
                want = srcs[i][:nbytes].cpu().numpy()
                assert np.array_equal(got, want), f"batch {bid} differs"
    finally:
        case.close()


@pytest.mark.parametrize("name", ["llama13b_8to4", "engine_consolidate", "delta_rounds_cap"])
def test_handoff_mode_commits_at_the_barrier(gpu_count, name):
    """kvx_ctl_set_handoff: the barrier decision issues the final wave at once
    (no drain); the data plane over the barrier's live set is the oracle's
    (control replayed with inflight = 0) and the payload checks out."""
    scn = W.load_golden(name)
    t = scn.transitions[0]
    L, H, D = W.shape_for(scn)
    case = GpuCase(scn, t, H if name.startswith("llama") else 2, D if name.startswith("llama") else 64,
                   oracle_pools=False)
    try:
        octx = O.ControlCtx(case.N, scn.max_sync_rounds, scn.kv_bytes_per_token)
        tr = case.tr
        tr.set_handoff(True)
        w0 = t.waves[0]
        tr.begin_refactor((w0.req, w0.hi))
        r = octx.begin(w0.req, w0.hi)
        assert case.dp.wave(w0.req, r[1], r[2]) == 0
        for e in t.events[1:]:
            if isinstance(e, W.Barrier):
                bar = e
                break
            act, _ = tr.on_kv_sync_complete((e.req, e.hi), 1)
            r = octx.on_sync_complete(e.req, e.hi, 1)
            assert act == r[0] == kvx.ACT_DELTA
            assert case.dp.wave(e.req, r[2], r[3]) == 0
        assert bar.inflight_batches > 0
        act, tok = tr.on_kv_sync_complete((bar.req, bar.kv), bar.inflight_batches)
        r = octx.on_sync_complete(bar.req, bar.kv, 0)      # handed off == nothing left in flight
        assert act == r[0] == kvx.ACT_FINAL and tok == r[1]
        assert case.dp.wave(bar.req, r[2], r[3]) == 0
        res = tr.on_refactor_commit((bar.req, bar.kv))
        v, row_ptr, blocks, free = case.dp.commit(bar.req, bar.kv)
        assert res.violations == v == 0
        np.testing.assert_array_equal(res.blocks, blocks)
        np.testing.assert_array_equal(tr.dst_block_table(), case.dp.bt)
        assert tr.verify_pattern(SEED, bar.req, bar.kv) == 0
    finally:
        case.close()


def test_handoff_finished_and_out_of_range(gpu_count):
    """The product follows the oracle at the edges: a batch past the last old
    stage gets no slot, an after_stage beyond the old pipeline is KVX_EINVAL."""
    import torch
    scn = W.load_golden("engine_consolidate")
    t = scn.transitions[0]
    case = GpuCase(scn, t, 1, 8, oracle=False)
    try:
        k_old = len(t.old_boundaries) + 1
        src = torch.zeros(4 * 256, dtype=torch.uint8, device="cuda")
        arenas = [torch.zeros(1 << 16, dtype=torch.uint8, device="cuda")
                  for _ in range(len(t.new_boundaries) + 1)]
        slots = case.tr.handoff(256, [(7, k_old - 1, 4, src.data_ptr()), (8, -1, 4, src.data_ptr())],
                                [a.data_ptr() for a in arenas], [1 << 16] * len(arenas))
        assert slots[0][1:] == (-1, -1, 0, 0) and slots[1][1:] == (0, 0, 0, 0)
        with pytest.raises(kvx.KvxError):
            case.tr.handoff(256, [(9, k_old, 4, src.data_ptr())], [a.data_ptr() for a in arenas],
                            [1 << 16] * len(arenas))
    finally:
        case.close()
