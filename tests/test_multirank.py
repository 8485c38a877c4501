"""Multi-process transitions: world_size-2 host logic on CPU (gloo), and the
NVLink P2P push / pull paths with 2 ranks (-m gpu).

On a box with fewer GPUs than ranks the ranks fold onto the visible GPUs
(mgpu_worker.device_of: rank % gpu_count).  CUDA IPC between processes on
one device is legal, so a 1-GPU run still exercises IPC export/import, the
imported-pool movers (push into a peer's pool, pull out of one), the
peer/local CTA split and the system fences, bit for bit against the oracle;
`gpurun --gpus 2` runs the same tests with the bytes crossing NVLink."""
import multiprocessing as mp
import os
import random

import pytest

from tests import mgpu_worker


def _free_port() -> int:
    """A TCP port nothing listens on now (the gloo store binds it next); a
    random pick could collide and leave the other ranks waiting for a store
    that never comes up."""
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _run(target, world, *args, timeout=600):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            try:
                rank, status, payload = q.get(timeout=timeout)
            except Exception:  # queue.Empty: report who never answered, and how they ended
                codes = {i: p.exitcode for i, p in enumerate(procs)}
                raise AssertionError(f"ranks {sorted(set(range(world)) - set(res))} gave no result within "
                                     f"{timeout} s; exit codes {codes}; results so far {res}")
            res[rank] = (status, payload)
            # a failed rank will not reach the others' barriers: fail now, not at the timeout
            assert status == "ok", f"rank {rank}:\n{payload}"
    finally:
        for p in procs:
            p.join(timeout=60 if len(res) == world else 1)
            if p.is_alive():
                p.terminate()
                p.join(timeout=10)
    return {r: p for r, (_, p) in res.items()}


@pytest.mark.parametrize("world", [2, 4, 8])
def test_ranks_shard_every_layer_once_cpu(world):
    res = _run(mgpu_worker.cpu_worker, world)
    for mode in ("affinity", "disjoint", "spread"):
        every, handles, old_dev, new_dev = res[0][mode]
        for r in range(1, world):
            assert res[r][mode][0] == every  # every rank agrees on the sharding
        flat = sorted(l for layers in every for l in layers)
        assert flat == list(range(40))   # each layer moved by exactly one rank
        owners = {j for hs in handles for j in hs}
        assert owners == set(range(4))   # every new stage exported by its owner
        assert all(0 <= d < world for d in old_dev + new_dev)
    _, _, old_dev, new_dev = res[0]["affinity"]
    if world == 2:
        assert old_dev == [0, 0, 0, 0, 1, 1, 1, 1] and new_dev == [0, 0, 1, 1]
        assert res[0]["disjoint"][3] == [1, 1, 0, 0]
    if world == 8:
        assert old_dev == list(range(8)) and new_dev == [0, 2, 4, 6]   # half of each stage crosses NVLink


@pytest.mark.parametrize("world", [2, 4])
def test_rank_pool_mapping_for_every_mover_policy_cpu(world):
    """The real shard.setup_rank_pools across gloo ranks: every layer a rank
    moves has both pools there (local or IPC-mapped from its owner)."""
    res = _run(mgpu_worker.mapping_worker, world)
    assert sum(r["checked"] for r in res.values()) == 4 * 3 * 40   # each layer moved once per case


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("placement", ["affinity", "disjoint", "spread", "oneway"])
@pytest.mark.parametrize("policy", ["auto", "push", "pull"])
def test_move_plan_moves_every_layer_once_cpu(world, placement, policy):
    """kvx_begin's per-layer mover selection (both pools local: move here;
    else layer_pull[l] ? the destination's rank : the source's rank), run
    over every rank: each layer of C3 is moved by exactly one rank, and
    'auto' pulls exactly the one-way cross-GPU layers."""
    from paper_2510_11938_b200 import shard as S
    ob, nb, L = [5, 10, 15, 20, 25, 30, 35], [10, 20, 30], 40
    old_dev, new_dev = S.placement(L, ob, nb, world, placement)
    lp = S.move_plan(L, ob, nb, old_dev, new_dev, policy)
    for l in range(L):
        s, d = old_dev[S.stage_of(ob, l)], new_dev[S.stage_of(nb, l)]
        movers = [r for r in range(world)
                  if (s == r and d == r) or (s != d and ((lp[l] and d == r) or (not lp[l] and s == r)))]
        assert len(movers) == 1, (l, s, d, movers)
    cross = [l for l in range(L) if old_dev[S.stage_of(ob, l)] != new_dev[S.stage_of(nb, l)]]
    if policy == "auto" and world == 8 and placement == "affinity":
        assert [l for l in range(L) if lp[l]] == cross and len(cross) == 20   # one-way pairs: pulled
    if policy == "auto" and placement == "disjoint" and world in (2, 4):
        assert sum(lp) == 0                                                   # two-way: pushed


@pytest.mark.gpu
@pytest.mark.parametrize("pull", [False, True, "auto"], ids=["push", "pull", "auto"])
@pytest.mark.parametrize("mode", ["affinity", "disjoint", "oneway"])
@pytest.mark.parametrize("name,heads,dim", [("criterion12", 2, 64), ("engine_consolidate", 2, 64)])
def test_two_gpu_transition_bit_exact(gpu_count, mode, name, heads, dim, pull):
    res = _run(mgpu_worker.gpu_worker, 2, name, heads, dim, mode, pull, 0, (0, 0))
    assert sum(r["checked"] for r in res.values()) >= 2


@pytest.mark.gpu
@pytest.mark.parametrize("name,mode,pull", [
    ("llama13b_8to4", "affinity", "auto"), ("llama13b_8to4", "disjoint", False), ("llama13b_8to4", "disjoint", True),
    ("llama13b_8to4", "spread", "auto"), ("llama13b_8to4", "oneway", "auto"), ("criterion12", "disjoint", "auto"),
    ("criterion12", "spread", False)])
def test_four_rank_transition_bit_exact(gpu_count, mode, name, pull):
    """World size 4 (the N=4 scaling run's shape): each rank owns a quarter of
    the stages; every destination pool is compared with the oracle by the rank
    that owns it, so all new stages are checked exactly once.  Ranks fold onto
    the visible GPUs (four physical GPUs on a 4-GPU box)."""
    res = _run(mgpu_worker.gpu_worker, 4, name, 2, 64, mode, pull, 0, (0, 0))
    from paper_2510_11938_b200 import workload as W
    t = [x for x in W.load_golden(name).transitions if x.outcome == "commit"][-1]
    assert sum(r["checked"] for r in res.values()) == len(t.new_boundaries) + 1


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["affinity", "spread"])
def test_two_gpu_controller_chain_bit_exact(gpu_count, mode):
    """BASELINE C5 across 2 GPUs: every 4th transition of the refactor chain
    the reference's own controller chose on the CV=7 gamma trace (4->16,
    16<->8 re-cuts; tests/golden/adaptive_cv7.jsonl), each pushed over
    NVLink and compared with the oracle byte for byte."""
    res = _run(mgpu_worker.gpu_worker, 2, "adaptive_cv7", 1, 8, mode, False, 4, (0, 0))
    assert all(r["transitions"] == 10 for r in res.values())
    assert sum(r["checked"] for r in res.values()) >= 10


@pytest.mark.gpu
@pytest.mark.parametrize("pull", [False, True], ids=["push", "pull"])
@pytest.mark.parametrize("layouts", [(1, 0), (0, 1), (1, 1), (2, 2), (0, 2), (2, 1)],
                         ids=["planes-to-blocks", "blocks-to-planes", "planes", "heads", "blocks-to-heads",
                              "heads-to-planes"])
def test_two_gpu_layout_conversion_bit_exact(gpu_count, layouts, pull):
    """Cross-GPU transitions between K/V-plane and block pools: peers map each
    other's pools with their layout (kvx_pool_import_layout); the moved
    bytes land permuted into the destination layout, bit for bit."""
    res = _run(mgpu_worker.gpu_worker, 2, "criterion12", 2, 64, "disjoint", pull, 0, layouts)
    assert sum(r["checked"] for r in res.values()) >= 2


@pytest.mark.gpu
def test_two_gpu_activation_handoff(gpu_count):
    res = _run(mgpu_worker.handoff_worker, 2)
    assert sum(r["checked"] for r in res.values()) >= 10
    assert sum(r["crossed"] for r in res.values()) >= 10


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(int(os.environ.get("KVX_MGPU_SEEDS", "6"))))  # soak: more seeds
def test_two_gpu_random_bit_exact(gpu_count, seed):
    _run(mgpu_worker.random_worker, 2, seed)
