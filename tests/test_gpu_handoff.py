"""GPU stage-boundary activation handoff vs the oracle plan: every in-flight
micro-batch the reference leaves at a barrier lands, byte-identical, in the
arena of the new stage that owns its resume layer."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import workload as W
from tests.gpu_harness import GpuCase
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
