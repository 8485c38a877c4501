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
        for mode in ("affinity", "disjoint"):
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
