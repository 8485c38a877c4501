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


def gpu_worker(rank, world, port, name, heads, dim, mode, pull, out):
    try:
        dist = _init(rank, world, port)
        import numpy as np
        from oracle import pyoracle as O
        from paper_2510_11938_b200 import kvx
        from paper_2510_11938_b200 import shard as S
        from paper_2510_11938_b200 import workload as W
        from tests.replay import replay

        scn = W.load_golden(name)
        t = [x for x in scn.transitions if x.outcome == "commit"][-1]
        L = scn.num_layers
        g = kvx.geometry(L, heads, dim)
        N = scn.num_requests
        tokens = t.max_tokens(N)
        max_blocks = int(max(1, (tokens.max() + 15) // 16))
        src_bt, old_blocks = W.fragmented_block_table(tokens, max_blocks, 16, seed=7)
        dst_blocks = max(1, int(((tokens + 15) // 16).sum()))
        live = np.nonzero(tokens)[0].astype(np.int32)
        old_dev, new_dev = S.placement(L, t.old_boundaries, t.new_boundaries, world, mode)

        def gather(obj):
            o = [None] * world
            dist.all_gather_object(o, obj)
            return o

        old_pools, new_pools = S.setup_rank_pools(
            kvx, g, t.old_boundaries, t.new_boundaries, old_dev, new_dev, rank, rank, old_blocks,
            dst_blocks, all_gather=gather, fill=(SEED, live, tokens[live], src_bt), pull=pull)
        dist.barrier()
        tr = kvx.Transition(g, t.old_boundaries, old_pools, t.new_boundaries, new_pools, rank, N,
                            max_blocks, dst_blocks, src_bt, epoch=t.epoch,
                            max_sync_rounds=scn.max_sync_rounds,
                            kv_bytes_per_token=scn.kv_bytes_per_token, pull=pull)
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
        res = tr.on_refactor_commit((t.live_req, t.live_kv))
        ov, row_ptr, blocks, free = dp.commit(t.live_req, t.live_kv)
        assert res.violations == ov == t.violations
        assert np.array_equal(res.blocks, blocks) and np.array_equal(res.free_list, free)
        assert np.array_equal(tr.dst_block_table(), dp.bt)
        dist.barrier()  # every rank's pushes have landed (kernels end with a system fence)
        checked = 0
        for j, p in enumerate(new_pools):
            if new_dev[j] == rank:
                got = p.read()
                assert np.array_equal(got, dp.new_pools[j]), f"new stage {j} differs on rank {rank}"
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
        dist.destroy_process_group()
        out.put((rank, "ok", {"checked": checked, "moved": moved, "old_dev": old_dev,
                              "new_dev": new_dev}))
    except Exception:
        out.put((rank, "err", traceback.format_exc()))


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

        torch.cuda.set_device(rank)
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
                                                  new_dev, rank, rank, cap0, dst, all_gather=gather)
        row = 512
        cap = sum(m.tokens * row + 256 for m in bar.microbatches) + 256
        # activation arenas of the new stages: raw pools, exported to the peer
        ablocks = cap // g.block_bytes + 1
        arenas, mine = [None] * len(new_dev), {}
        for j, d in enumerate(new_dev):
            if d == rank:
                arenas[j] = kvx.Pool(rank, g, 1, ablocks)
                arenas[j].zero()
                mine[j] = arenas[j].export_ipc()
        for r, hs in enumerate(gather(mine)):
            for j, h in hs.items():
                if r != rank:
                    arenas[int(j)] = kvx.Pool.import_ipc(rank, h, g, 1, ablocks)

        def payload(m):
            gen = torch.Generator(device="cpu").manual_seed(int(m.batch))
            return torch.randint(0, 256, (max(m.tokens, 1) * row,), dtype=torch.uint8, generator=gen)

        srcs = []
        for m in bar.microbatches:
            local = m.after >= 0 and m.after + 1 < len(old_dev) and old_dev[m.after] == rank
            srcs.append(payload(m).cuda() if local else torch.empty(16, dtype=torch.uint8, device="cuda"))
        torch.cuda.synchronize()
        tr = kvx.Transition(g, t.old_boundaries, old_pools, t.new_boundaries, new_pools, rank, N,
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
