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
    its new stages out over every GPU (what a split is for)."""
    k_old = len(ob) + 1
    old_dev = [k * n_gpus // k_old for k in range(k_old)]
    if mode == "spread":
        k_new = len(nb) + 1
        return old_dev, [j * n_gpus // k_new for j in range(k_new)]
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
                     old_layout: int = 0, new_layout: int = 0):
    """Creates this rank's pools and maps every peer's new-stage pool.

    fill = (seed, live_req, tokens, src_bt) writes the synthetic payload into
    the local old pools.  all_gather(obj) -> list of every rank's obj (e.g.
    torch.distributed.all_gather_object); None for a single process.
    pull=False maps peers' NEW pools (this rank pushes its old layers into
    them); pull=True maps peers' OLD pools (this rank pulls the layers of its
    new stages out of them).
    old_layout / new_layout: KVX_LAYOUT_* of the old / new pools (peers map
    them with the same layout).
    Returns (old_pools, new_pools) indexed by stage (None where remote/absent).
    """
    L = g.num_layers
    old_pools: List = [None] * (len(ob) + 1)
    mine = {}
    for k, (b, e) in enumerate(W.stage_ranges(L, ob)):
        if old_dev[k] == rank:
            p = kvx.Pool(device, g, e - b, old_blocks, old_layout)
            if fill is not None:
                seed, live, tokens, src_bt = fill
                p.zero()
                p.fill_pattern(seed, b, live, tokens, src_bt)
            old_pools[k] = p
            if pull and all_gather is not None:
                mine[k] = p.export_ipc()
    new_pools: List = [None] * (len(nb) + 1)
    for j, (b, e) in enumerate(W.stage_ranges(L, nb)):
        if new_dev[j] == rank:
            p = kvx.Pool(device, g, e - b, dst_blocks, new_layout)
            if zero_new:
                p.zero()
            new_pools[j] = p
            if not pull and all_gather is not None:
                mine[j] = p.export_ipc()
    if all_gather is not None:
        target, ranges, blocks, layout = (old_pools, W.stage_ranges(L, ob), old_blocks, old_layout) if pull else \
            (new_pools, W.stage_ranges(L, nb), dst_blocks, new_layout)
        for r, handles in enumerate(all_gather(mine)):
            if r == rank:
                continue
            for j, h in handles.items():
                b, e = ranges[int(j)]
                target[int(j)] = kvx.Pool.import_ipc(device, h, g, e - b, blocks, layout)
    return old_pools, new_pools
