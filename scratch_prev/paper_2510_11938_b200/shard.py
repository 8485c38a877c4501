"""Placement of logical pipeline stages on the physical GPUs of one node and
the per-rank pool set-up of a multi-GPU transition.

The reference grants every new stage a GPU that hosts no stage of the model
(engine.cpp:584-591), which needs K_old + K_new GPUs; on one 8-GPU box the
logical GPUs are mapped onto the physical ones.  Every (request, layer) slab
has exactly one source stage and one destination stage, so the transition
shards by layer: the rank that owns a layer's OLD stage moves it and pushes
it into the destination pool -- its own HBM, or a peer's through NVLink P2P
(CUDA IPC mapping).  No collective is needed: the destination block rule is
deterministic, so every rank derives the same destination block table.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional, Sequence, Tuple

from . import workload as W


def stage_of(boundaries: Sequence[int], layer: int) -> int:
    """PartitionPlan::stage_of_op (modelgraph.cpp:55-62)."""
    s = 0
    for b in boundaries:
        if layer < b:
            break
        s += 1
    return s


def placement(L: int, ob: Sequence[int], nb: Sequence[int], n_gpus: int,
              mode: str = "affinity") -> Tuple[List[int], List[int]]:
    """Old stage k -> GPU floor(k * N / K_old).  New stage j -> the GPU that
    already holds most of its layers (warm-start affinity, cluster.cpp:525-536
    and AffinityHistory::covers, cluster.cpp:158-199), ties to the lowest id.
    mode='disjoint' shifts each new stage by N/2 GPUs so all of its KV crosses
    NVLink, the physical analogue of the reference's disjoint grant.
    mode='spread' puts new stage j on GPU floor(j * N / K_new): a split fans
    its new stages out over every GPU (what a split is for).
    mode='oneway' puts every new stage on GPU 0: GPU 0 keeps its own layers
    and receives the rest one way -- at N=2 the traffic pattern of a C3
    receiver at N=8 (half local, half from one partner)."""
    k_old = len(ob) + 1
    old_dev = [k * n_gpus // k_old for k in range(k_old)]
    if mode == "spread":
        k_new = len(nb) + 1
        return old_dev, [j * n_gpus // k_new for j in range(k_new)]
    if mode == "oneway":
        return old_dev, [0] * (len(nb) + 1)
    new_dev = []
    for b, e in W.stage_ranges(L, nb):
        share: Dict[int, int] = {}
        for l in range(b, e):
            d = old_dev[stage_of(ob, l)]
            share[d] = share.get(d, 0) + 1
        best = sorted(share.items(), key=lambda kv: (-kv[1], kv[0]))[0][0]
        if mode == "disjoint" and n_gpus > 1:
            best = (best + n_gpus // 2) % n_gpus
        new_dev.append(best)
    return old_dev, new_dev


def move_plan(L: int, ob: Sequence[int], nb: Sequence[int], old_dev: Sequence[int],
              new_dev: Sequence[int], policy: str = "auto") -> List[int]:
    """kvx_transition_desc.layer_pull: per layer, 1 = the destination GPU pulls
    it, 0 = the source GPU pushes it (same-GPU layers move locally either way).
    policy 'push' / 'pull' for every layer; 'auto' pulls a cross-GPU layer
    s -> d when the traffic is one way at both ends (d sends nothing over
    NVLink, s receives nothing) and pushes it otherwise.  Through NVSwitch
    every GPU's links carry all of its egress and ingress; a pull's read
    requests travel d -> s.  Measured on B200 NVLink 5
    (profiles/r01_nvlink_split.jsonl): one way, TMA pull 790 GB/s vs push 718;
    both ways, push 712 vs pull 677 per direction."""
    if policy in ("push", "pull"):
        return [1 if policy == "pull" else 0] * L
    sends, recvs = set(), set()
    for l in range(L):
        s, d = old_dev[stage_of(ob, l)], new_dev[stage_of(nb, l)]
        if s != d:
            sends.add(s)
            recvs.add(d)
    plan = []
    for l in range(L):
        s, d = old_dev[stage_of(ob, l)], new_dev[stage_of(nb, l)]
        plan.append(1 if s != d and d not in sends and s not in recvs else 0)
    return plan


def layers_of_rank(L: int, ob: Sequence[int], old_dev: Sequence[int], rank: int) -> List[int]:
    """Layers whose KV this rank moves (its old stages' layers)."""
    return [l for l in range(L) if old_dev[stage_of(ob, l)] == rank]


def link_bytes(L: int, ob, nb, old_dev, new_dev, layer_bytes: int, n_gpus: int):
    """Per-GPU (HBM read+write, NVLink out, NVLink in) bytes of one transition
    that moves `layer_bytes` of K+V per layer."""
    hbm = [0] * n_gpus
    out = [0] * n_gpus
    inn = [0] * n_gpus
    for l in range(L):
        s, d = old_dev[stage_of(ob, l)], new_dev[stage_of(nb, l)]
        hbm[s] += layer_bytes
        hbm[d] += layer_bytes
        if s != d:
            out[s] += layer_bytes
            inn[d] += layer_bytes
    return hbm, out, inn


def setup_rank_pools(kvx, g, ob, nb, old_dev, new_dev, rank: int, device: int, old_blocks: int,
                     dst_blocks: int, all_gather: Optional[Callable] = None,
                     fill: Optional[tuple] = None, zero_new: bool = True, pull: bool = False,
                     old_layout: int = 0, new_layout: int = 0, layer_pull: Optional[Sequence[int]] = None):
    """Creates this rank's pools and maps every peer's new-stage pool.

    fill = (seed, live_req, tokens, src_bt) writes the synthetic payload into
    the local old pools.  all_gather(obj) -> list of every rank's obj (e.g.
    torch.distributed.all_gather_object); None for a single process.
    pull=False maps peers' NEW pools (this rank pushes its old layers into
    them); pull=True maps peers' OLD pools (this rank pulls the layers of its
    new stages out of them).
    old_layout / new_layout: KVX_LAYOUT_* of the old / new pools (peers map
    them with the same layout).
    layer_pull (move_plan): peers' pools are mapped on the side each layer's
    mover needs -- peers' NEW pools for the layers this rank pushes, peers'
    OLD pools for the layers it pulls.
    Returns (old_pools, new_pools) indexed by stage (None where remote/absent).
    """
    L = g.num_layers
    # which side of the peers' pools this rank maps
    map_old = pull or layer_pull is not None
    map_new = not pull or layer_pull is not None
    old_pools: List = [None] * (len(ob) + 1)
    mine = {"old": {}, "new": {}}
    for k, (b, e) in enumerate(W.stage_ranges(L, ob)):
        if old_dev[k] == rank:
            p = kvx.Pool(device, g, e - b, old_blocks, old_layout)
            if fill is not None:
                seed, live, tokens, src_bt = fill
                p.zero()
                p.fill_pattern(seed, b, live, tokens, src_bt)
            old_pools[k] = p
            if map_old and all_gather is not None:
                mine["old"][k] = p.export_ipc()
    new_pools: List = [None] * (len(nb) + 1)
    for j, (b, e) in enumerate(W.stage_ranges(L, nb)):
        if new_dev[j] == rank:
            p = kvx.Pool(device, g, e - b, dst_blocks, new_layout)
            if zero_new:
                p.zero()
            new_pools[j] = p
            if map_new and all_gather is not None:
                mine["new"][j] = p.export_ipc()
    if all_gather is not None:
        sides = {"old": (old_pools, W.stage_ranges(L, ob), old_blocks, old_layout),
                 "new": (new_pools, W.stage_ranges(L, nb), dst_blocks, new_layout)}
        for r, handles in enumerate(all_gather(mine)):
            if r == rank:
                continue
            for side, (target, ranges, blocks, layout) in sides.items():
                for j, h in handles[side].items():
                    b, e = ranges[int(j)]
                    target[int(j)] = kvx.Pool.import_ipc(device, h, g, e - b, blocks, layout)
    return old_pools, new_pools
