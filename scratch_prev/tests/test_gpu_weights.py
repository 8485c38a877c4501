"""GPU stage weight migration vs the oracle routing (kvo_weights_plan):
device-to-device layer gather plus host-tier loads from a pinned cache."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import kvx
from paper_2510_11938_b200 import workload as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("L,ob,nb,layer_bytes,host_layers", [
    (40, [5, 10, 15, 20, 25, 30, 35], [10, 20, 30], 3 << 20, []),          # 13B 8->4
    (32, [16], [4, 8, 12, 16, 20, 24, 28], (1 << 20) + 48, [0, 7, 31]),    # 7B 2->8, ragged size
    (80, [10, 20, 30, 40, 50, 60, 70], [40], 1 << 18, list(range(0, 80, 9))),
])
def test_weights_bit_exact(gpu_count, L, ob, nb, layer_bytes, host_layers):
    import torch
    g = torch.Generator(device="cpu").manual_seed(L)
    old = [torch.randint(0, 256, ((e - b) * layer_bytes,), dtype=torch.uint8, generator=g).cuda()
           for b, e in W.stage_ranges(L, ob)]
    new = [torch.zeros((e - b) * layer_bytes, dtype=torch.uint8, device="cuda") for b, e in W.stage_ranges(L, nb)]
    host = torch.randint(0, 256, (L * layer_bytes,), dtype=torch.uint8, generator=g).pin_memory()
    from_host = np.zeros(L, np.uint8)
    from_host[host_layers] = 1
    torch.cuda.synchronize()
    db, hb = kvx.weights_migrate(0, L, layer_bytes, ob, [t.data_ptr() for t in old], nb,
                                 [t.data_ptr() for t in new], host_cache=host.data_ptr(),
                                 from_host=from_host)
    torch.cuda.synchronize()
    assert db == (L - len(host_layers)) * layer_bytes and hb == len(host_layers) * layer_bytes
    ss, so, ds, do = O.weights_plan(L, layer_bytes, ob, nb)
    newh = [t.cpu().numpy() for t in new]
    oldh = [t.cpu().numpy() for t in old]
    hosth = host.numpy()
    for l in range(L):
        got = newh[ds[l]][int(do[l]):int(do[l]) + layer_bytes]
        want = hosth[l * layer_bytes:(l + 1) * layer_bytes] if from_host[l] else \
            oldh[ss[l]][int(so[l]):int(so[l]) + layer_bytes]
        assert np.array_equal(got, want), f"layer {l}"
