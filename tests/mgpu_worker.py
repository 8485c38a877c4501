"""Worker of the multi-process transition tests: one process per rank, gloo
for the host plumbing (IPC-handle exchange, barriers).  With cuda=True each
rank owns one GPU and pushes its layers' KV into peer pools over NVLink; the
CPU variant (cuda=False) checks the host-side sharding logic only."""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

SEED = 0x77


def device_of(rank: int) -> int:
    """The GPU rank `rank` runs on: its own on a box with >= world GPUs, else
    ranks fold onto the visible ones (rank % gpu_count).  CUDA IPC between two
    processes on one device is legal, so a folded run still goes through
    IPC export/import, the imported-pool (peer) paths of the movers, the
    peer/local CTA split and the system fences -- only the bytes stay in one
    HBM instead of crossing NVLink."""
    from paper_2510_11938_b200 import kvx
    n = kvx.device_count()
    if n < 1:
        raise RuntimeError("no CUDA device visible to libkvx.so")
    return rank % n


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def cpu_worker(rank, world, port, out):
    try:
        dist = _init(rank, world, port)
        from paper_2510_11938_b200 import shard as S
        from paper_2510_11938_b200 import workload as W
        scn = W.load_golden("llama13b_8to4")
        t = scn.transitions[0]
        L = scn.num_layers
        res = {}
        for mode in ("affinity", "disjoint", "spread"):
            old_dev, new_dev = S.placement(L, t.old_boundaries, t.new_boundaries, world, mode)
            mine = S.layers_of_rank(L, t.old_boundaries, old_dev, rank)
            every = [None] * world
            dist.all_gather_object(every, mine)
            # exchange of fake IPC handles: the same protocol setup_rank_pools uses
            handles = {j: bytes([rank, j]) * 32 for j, d in enumerate(new_dev) if d == rank}
            hs = [None] * world
            dist.all_gather_object(hs, handles)
            res[mode] = (every, hs, old_dev, new_dev)
        dist.barrier()
        dist.destroy_process_group()
        out.put((rank, "ok", res))
    except Exception:
        out.put((rank, "err", traceback.format_exc()))


def gpu_worker(rank, world, port, name, heads, dim, mode, pull, stride, layouts, out):
    """stride=0: the scenario's last committed transition; stride=k: every
    k-th transition of the scenario (e.g. the controller-chosen chain).
    layouts = (old, new) KVX_LAYOUT_* of the pools."""
    try:
        dist = _init(rank, world, port)
        from paper_2510_11938_b200 import workload as W

        scn = W.load_golden(name)
        ts = [[x for x in scn.transitions if x.outcome == "commit"][-1]] if not stride \
            else scn.transitions[::stride]
        checked, moved = 0, 0
        for t in ts:
            c, m, old_dev, new_dev = _gpu_transition(dist, rank, world, scn, t, heads, dim, mode, pull, layouts)
            checked += c
            moved += m
        dist.destroy_process_group()
        out.put((rank, "ok", {"checked": checked, "moved": moved, "old_dev": old_dev,
                              "new_dev": new_dev, "transitions": len(ts)}))
    except Exception:
        out.put((rank, "err", traceback.format_exc()))


def _gpu_transition(dist, rank, world, scn, t, heads, dim, mode, pull, layouts=(0, 0)):
    import numpy as np
    from oracle import pyoracle as O
    from paper_2510_11938_b200 import kvx
    from paper_2510_11938_b200 import shard as S
    from paper_2510_11938_b200 import workload as W
    from tests.replay import replay

    L = scn.num_layers
    g = kvx.geometry(L, heads, dim)
    N = scn.num_requests
    tokens = t.max_tokens(N)
    max_blocks = int(max(1, (tokens.max() + 15) // 16))
    src_bt, old_blocks = W.fragmented_block_table(tokens, max_blocks, 16, seed=7)
    dst_blocks = max(1, int(((tokens + 15) // 16).sum()))
    live = np.nonzero(tokens)[0].astype(np.int32)
    old_dev, new_dev = S.placement(L, t.old_boundaries, t.new_boundaries, world, mode)
    # pull: False (push), True (pull) or "auto" (per-layer movers, shard.move_plan)
    layer_pull = S.move_plan(L, t.old_boundaries, t.new_boundaries, old_dev, new_dev) if pull == "auto" else None
    pull = pull is True

    def gather(obj):
        o = [None] * world
        dist.all_gather_object(o, obj)
        return o

    dev = device_of(rank)
    old_pools, new_pools = S.setup_rank_pools(
        kvx, g, t.old_boundaries, t.new_boundaries, old_dev, new_dev, rank, dev, old_blocks,
        dst_blocks, all_gather=gather, fill=(SEED, live, tokens[live], src_bt), pull=pull,
        old_layout=layouts[0], new_layout=layouts[1], layer_pull=layer_pull)
    dist.barrier()
    tr = kvx.Transition(g, t.old_boundaries, old_pools, t.new_boundaries, new_pools, dev, N,
                        max_blocks, dst_blocks, src_bt, epoch=t.epoch,
                        max_sync_rounds=scn.max_sync_rounds,
                        kv_bytes_per_token=scn.kv_bytes_per_token, pull=pull, layer_pull=layer_pull)
    octx = O.ControlCtx(N, scn.max_sync_rounds, scn.kv_bytes_per_token)
    dp = O.DataPlane(O.geo(L, heads, dim), t.old_boundaries, t.new_boundaries, old_blocks,
                     dst_blocks, N, max_blocks, src_bt)
    dp.fill_source(SEED, live, tokens[live])

    class Shim:
        def begin(self, req, kv):
            tr.begin_refactor((req, kv))
            r = octx.begin(req, kv)
            assert dp.wave(req, r[1], r[2]) == 0
            return r

        def on_sync_complete(self, req, kv, inflight):
            act, tok = tr.on_kv_sync_complete((req, kv), inflight)
            r = octx.on_sync_complete(req, kv, inflight)
            assert (act, tok) == (r[0], r[1])
            if act != kvx.ACT_BARRIER_WAIT:
                assert dp.wave(req, r[2], r[3]) == 0
            return r

    for _ in replay(Shim(), t):
        pass
    if t.outcome == "commit":
        res = tr.on_refactor_commit((t.live_req, t.live_kv))
        ov, row_ptr, blocks, free = dp.commit(t.live_req, t.live_kv)
        assert res.violations == ov == t.violations
        assert np.array_equal(res.blocks, blocks) and np.array_equal(res.free_list, free)
    assert np.array_equal(tr.dst_block_table(), dp.bt)
    dist.barrier()  # every rank's pushes have landed (kernels end with a system fence)
    checked = 0
    for j, (b, e) in enumerate(W.stage_ranges(L, t.new_boundaries)):
        if new_dev[j] == rank:
            got = new_pools[j].read().reshape(e - b, -1)
            want = dp.new_pools[j].reshape(e - b, dst_blocks, 2, 16, heads, -1)  # the oracle: block layout
            if layouts[1] == kvx.LAYOUT_KV_PLANES:
                want = want.transpose(0, 2, 1, 3, 4, 5)
            elif layouts[1] == kvx.LAYOUT_HEADS:
                want = want.transpose(0, 1, 2, 4, 3, 5)
            assert np.array_equal(got, np.ascontiguousarray(want).reshape(e - b, -1)), \
                f"new stage {j} differs on rank {rank}"
            checked += 1
    moved = tr.bytes_moved()
    tr.close()
    dist.barrier()
    for p in old_pools + new_pools:      # unmap peers' pools first ...
        if p is not None and p.imported:
            p.close()
    dist.barrier()
    for p in old_pools + new_pools:      # ... then free our own
        if p is not None and not p.imported:
            p.close()
    dist.barrier()
    return checked, moved, old_dev, new_dev


def handoff_worker(rank, world, port, out):
    """Cross-GPU activation handoff: criterion12's second transition (16 -> 4)
    with the old stages split over 2 GPUs and the new stages shifted ('disjoint'
    placement), so every in-flight micro-batch crosses NVLink into an arena
    mapped from the peer through CUDA IPC."""
    try:
        dist = _init(rank, world, port)
        import numpy as np
        import torch
        from oracle import pyoracle as O
        from paper_2510_11938_b200 import kvx
        from paper_2510_11938_b200 import shard as S
        from paper_2510_11938_b200 import workload as W

        dev = device_of(rank)
        torch.cuda.set_device(dev)
        scn = W.load_golden("engine_consolidate")   # 16 -> 4, 19 in-flight micro-batches at the barrier
        t = scn.transitions[0]
        bar = next(e for e in t.events if isinstance(e, W.Barrier))
        L, N = scn.num_layers, scn.num_requests
        g = kvx.geometry(L, 1, 8)
        old_dev, new_dev = S.placement(L, t.old_boundaries, t.new_boundaries, world, "disjoint")
        tokens = t.max_tokens(N)
        max_blocks = int(max(1, (tokens.max() + 15) // 16))
        src_bt, cap0 = W.fragmented_block_table(tokens, max_blocks, 16, seed=7)
        dst = max(1, int(((tokens + 15) // 16).sum()))

        def gather(obj):
            o = [None] * world
            dist.all_gather_object(o, obj)
            return o

        old_pools, new_pools = S.setup_rank_pools(kvx, g, t.old_boundaries, t.new_boundaries, old_dev,
                                                  new_dev, rank, dev, cap0, dst, all_gather=gather)
        row = 512
        cap = sum(m.tokens * row + 256 for m in bar.microbatches) + 256
        # activation arenas of the new stages: raw pools, exported to the peer
        ablocks = cap // g.block_bytes + 1
        arenas, mine = [None] * len(new_dev), {}
        for j, d in enumerate(new_dev):
            if d == rank:
                arenas[j] = kvx.Pool(dev, g, 1, ablocks)
                arenas[j].zero()
                mine[j] = arenas[j].export_ipc()
        for r, hs in enumerate(gather(mine)):
            for j, h in hs.items():
                if r != rank:
                    arenas[int(j)] = kvx.Pool.import_ipc(dev, h, g, 1, ablocks)

        def payload(m):
            gen = torch.Generator(device="cpu").manual_seed(int(m.batch))
            return torch.randint(0, 256, (max(m.tokens, 1) * row,), dtype=torch.uint8, generator=gen)

        srcs = []
        for m in bar.microbatches:
            local = m.after >= 0 and m.after + 1 < len(old_dev) and old_dev[m.after] == rank
            srcs.append(payload(m).cuda() if local else torch.empty(16, dtype=torch.uint8, device="cuda"))
        torch.cuda.synchronize()
        tr = kvx.Transition(g, t.old_boundaries, old_pools, t.new_boundaries, new_pools, dev, N,
                            max_blocks, dst, src_bt, epoch=t.epoch)
        slots = tr.handoff(row, [(m.batch, m.after, m.tokens, s.data_ptr())
                                 for m, s in zip(bar.microbatches, srcs)],
                           [a.ptr for a in arenas], [cap] * len(arenas))
        tr.wait()
        rc, ns, rl, off, by = O.handoff_plan(t.old_boundaries, t.new_boundaries, row,
                                             [m.after for m in bar.microbatches],
                                             [m.tokens for m in bar.microbatches], [cap] * len(arenas))
        assert rc == 0
        for i, sl in enumerate(slots):
            assert tuple(sl) == (bar.microbatches[i].batch, ns[i], rl[i], off[i], by[i])
        dist.barrier()   # every rank's pushes have landed
        checked = crossed = 0
        for i, m in enumerate(bar.microbatches):
            k, nbytes = int(ns[i]), int(by[i])
            if nbytes == 0 or new_dev[k] != rank:
                continue
            got = arenas[k].read(int(off[i]), nbytes)
            assert np.array_equal(got, payload(m)[:nbytes].numpy()), f"batch {m.batch}"
            checked += 1
            crossed += old_dev[m.after] != rank
        tr.close()
        dist.barrier()
        for p in arenas + old_pools + new_pools:
            if p is not None and p.imported:
                p.close()
        dist.barrier()
        for p in arenas + old_pools + new_pools:
            if p is not None and not p.imported:
                p.close()
        dist.barrier()
        dist.destroy_process_group()
        out.put((rank, "ok", {"checked": checked, "crossed": crossed}))
    except Exception:
        out.put((rank, "err", traceback.format_exc()))


def random_worker(rank, world, port, seed, out):
    """Random plans, geometries, lengths, waves and a random stage->GPU map
    over the ranks (push or pull, bump rule or block manager): every rank's
    local destination pools must equal the oracle's, byte for byte."""
    try:
        dist = _init(rank, world, port)
        import numpy as np
        from oracle import pyoracle as O
        from paper_2510_11938_b200 import kvx
        from paper_2510_11938_b200 import shard as S
        from paper_2510_11938_b200 import workload as W

        rng = np.random.default_rng(seed)
        L = int(rng.integers(2, 20))
        heads, dim = int(rng.choice([1, 2, 4])), int(rng.choice([8, 64, 128]))

        def plan():
            k = int(rng.integers(1, min(L, 8) + 1))
            return sorted(rng.choice(np.arange(1, L), size=k - 1, replace=False).tolist()) if k > 1 else []
        ob, nb = plan(), plan()
        old_dev = rng.integers(0, world, len(ob) + 1).tolist()
        new_dev = rng.integers(0, world, len(nb) + 1).tolist()
        pull = bool(rng.random() < 0.5)
        use_bm = bool(rng.random() < 0.5)
        N = int(rng.integers(1, 40))
        final = rng.integers(0, 150, N).astype(np.int64)
        max_blocks = int(max(1, (final.max() + 15) // 16))
        src_bt, cap0 = W.fragmented_block_table(final, max_blocks, 16, seed=seed)
        cap1 = max(1, int(((final + 15) // 16).sum()))
        live = np.nonzero(final)[0].astype(np.int32)
        g, og = kvx.geometry(L, heads, dim), O.geo(L, heads, dim)

        def gather(obj):
            o = [None] * world
            dist.all_gather_object(o, obj)
            return o

        dev = device_of(rank)
        old_pools, new_pools = S.setup_rank_pools(
            kvx, g, ob, nb, old_dev, new_dev, rank, dev, cap0, cap1, all_gather=gather,
            fill=(seed, live, final[live], src_bt) if len(live) else None, pull=pull)
        for k, p in enumerate(old_pools):   # zero-filled sources where nothing is live
            if p is not None and not p.imported and not len(live):
                p.zero()
        bm = kvx.BlockManager(dev, cap1) if use_bm else None
        ref_bm = O.StackBM(cap1) if use_bm else None
        dist.barrier()
        tr = kvx.Transition(g, ob, old_pools, nb, new_pools, dev, N, max_blocks, cap1, src_bt, epoch=1,
                            dst_blockmgr=bm, pull=pull)
        dp = O.DataPlane(og, ob, nb, cap0, cap1, N, max_blocks, src_bt, bm=ref_bm)
        if len(live):
            dp.fill_source(seed, live, final[live])
        synced = np.zeros(N, np.int64)
        for w in range(int(rng.integers(1, 4))):
            target = final if w == 2 else np.minimum(final, synced + rng.integers(0, 80, N))
            req = np.arange(N, dtype=np.int32)
            hi = np.maximum(target, synced)
            tr.wave(req, synced, hi)
            assert dp.wave(req, synced, hi) == 0
            synced = hi
        req = np.arange(N, dtype=np.int32)
        tr.wave(req, synced, final)          # make sure everything landed
        assert dp.wave(req, synced, final) == 0
        tr.wait()
        dist.barrier()                       # peers' pushes have landed
        checked = 0
        for j, d in enumerate(new_dev):
            if d == rank:
                assert np.array_equal(new_pools[j].read(), dp.new_pools[j]), f"stage {j} rank {rank}"
                checked += 1
        assert np.array_equal(tr.dst_block_table(), dp.bt)
        res = tr.commit(live, final[live])
        assert res.violations == 0
        tr.close()
        dist.barrier()
        for p in old_pools + new_pools:
            if p is not None and p.imported:
                p.close()
        dist.barrier()
        for p in old_pools + new_pools:
            if p is not None and not p.imported:
                p.close()
        if bm is not None:
            bm.close()
        dist.barrier()
        dist.destroy_process_group()
        out.put((rank, "ok", {"checked": checked, "pull": pull, "bm": use_bm}))
    except Exception:
        out.put((rank, "err", traceback.format_exc()))


def mapping_worker(rank, world, port, out):
    """shard.setup_rank_pools with a fake kvx over gloo: for every placement
    and mover policy, every layer this rank moves (kvx_begin's selection) has
    both of its pools here, local or mapped from the owning peer."""
    try:
        dist = _init(rank, world, port)
        from paper_2510_11938_b200 import shard as S
        from paper_2510_11938_b200 import workload as W

        class FakePool:
            def __init__(self, device, g, layers, blocks, layout=0, owner=None, stage=None):
                self.device, self.layers, self.blocks, self.layout = device, layers, blocks, layout
                self.imported, self.owner = owner is not None, owner if owner is not None else rank

            def zero(self):
                pass

            def fill_pattern(self, *a):
                pass

            def export_ipc(self):
                return bytes([rank]) * 64

            @classmethod
            def import_ipc(cls, device, h, g, layers, blocks, layout=0):
                return cls(device, g, layers, blocks, layout, owner=h[0])

        class FakeKvx:
            Pool = FakePool

        class G:
            num_layers = 40

        scn = W.load_golden("llama13b_8to4")
        t = scn.transitions[0]
        ob, nb, L = t.old_boundaries, t.new_boundaries, 40
        checked = 0
        for mode in ("affinity", "disjoint", "spread", "oneway"):
            old_dev, new_dev = S.placement(L, ob, nb, world, mode)
            for policy in ("push", "pull", "auto"):
                lp = S.move_plan(L, ob, nb, old_dev, new_dev, policy)

                def gather(obj):
                    o = [None] * world
                    dist.all_gather_object(o, obj)
                    return o

                old, new = S.setup_rank_pools(FakeKvx, G, ob, nb, old_dev, new_dev, rank, rank, 8, 8,
                                              all_gather=gather, layer_pull=lp, new_layout=2)
                for l in range(L):
                    so, sn = S.stage_of(ob, l), S.stage_of(nb, l)
                    s, d = old_dev[so], new_dev[sn]
                    moves_here = (s == rank and d == rank) or (s != d and ((lp[l] and d == rank) or
                                                                           (not lp[l] and s == rank)))
                    if moves_here:
                        assert old[so] is not None and new[sn] is not None, (mode, policy, l)
                        assert old[so].owner == s and new[sn].owner == d
                        assert new[sn].layout == 2          # peers map pools with their layout
                        checked += 1
        dist.barrier()
        dist.destroy_process_group()
        out.put((rank, "ok", {"checked": checked}))
    except Exception:
        out.put((rank, "err", traceback.format_exc()))
