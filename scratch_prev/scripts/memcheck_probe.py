"""Small end-to-end exercise for compute-sanitizer memcheck: the smoke
transition, an edge-case transition with block manager + abort, a handoff and
a weight migration -- every kernel family of libkvx.so, tiny sizes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import __graft_entry__ as g  # noqa: E402

g.smoke()

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_11938_b200 import kvx  # noqa: E402
from tests.test_gpu_random import test_random_transition_bit_exact  # noqa: E402
from tests.test_gpu_edges import test_errors, test_abort_drops_destination_and_invalidates_epoch  # noqa: E402

for seed in (3, 7, 11):
    test_random_transition_bit_exact(1, seed)
test_errors(1)
test_abort_drops_destination_and_invalidates_epoch(1)
# handoff + weights through the copy-list kernel
L, lb = 8, 1 << 16
old = [torch.randint(0, 255, (4 * lb,), dtype=torch.uint8, device="cuda") for _ in range(2)]
new = [torch.zeros(2 * lb, dtype=torch.uint8, device="cuda") for _ in range(4)]
kvx.weights_migrate(0, L, lb, [4], [t.data_ptr() for t in old], [2, 4, 6], [t.data_ptr() for t in new])
torch.cuda.synchronize()
assert torch.equal(new[1][:lb], old[0][2 * lb:3 * lb])
print("memcheck probe done")
