"""Multi-process transitions: world_size-2 host logic on CPU (gloo), and the
NVLink P2P push path on 2 GPUs (-m gpu; skipped on a 1-GPU box)."""
import multiprocessing as mp
import random

import pytest

from tests import mgpu_worker


def _run(target, world, *args, timeout=600):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, status, payload = q.get(timeout=timeout)
        res[rank] = (status, payload)
    for p in procs:
        p.join(timeout=60)
    for rank, (status, payload) in res.items():
        assert status == "ok", f"rank {rank}:\n{payload}"
    return {r: p for r, (_, p) in res.items()}


def test_two_ranks_shard_every_layer_once_cpu():
    res = _run(mgpu_worker.cpu_worker, 2)
    for mode in ("affinity", "disjoint"):
        every, handles, old_dev, new_dev = res[0][mode]
        assert res[1][mode][0] == every  # both ranks agree on the sharding
        flat = sorted(l for layers in every for l in layers)
        assert flat == list(range(40))   # each layer moved by exactly one rank
        owners = {j for hs in handles for j in hs}
        assert owners == set(range(4))   # every new stage exported by its owner
    _, _, old_dev, new_dev = res[0]["affinity"]
    assert old_dev == [0, 0, 0, 0, 1, 1, 1, 1] and new_dev == [0, 0, 1, 1]
    _, _, old_dev, new_dev = res[0]["disjoint"]
    assert new_dev == [1, 1, 0, 0]


@pytest.mark.gpu
@pytest.mark.parametrize("pull", [False, True], ids=["push", "pull"])
@pytest.mark.parametrize("mode", ["affinity", "disjoint"])
@pytest.mark.parametrize("name,heads,dim", [("criterion12", 2, 64), ("engine_consolidate", 2, 64)])
def test_two_gpu_transition_bit_exact(gpu_count, mode, name, heads, dim, pull):
    if gpu_count < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    res = _run(mgpu_worker.gpu_worker, 2, name, heads, dim, mode, pull)
    assert sum(r["checked"] for r in res.values()) >= 2


@pytest.mark.gpu
def test_two_gpu_activation_handoff(gpu_count):
    if gpu_count < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    res = _run(mgpu_worker.handoff_worker, 2)
    assert sum(r["checked"] for r in res.values()) >= 10
    assert sum(r["crossed"] for r in res.values()) >= 10
