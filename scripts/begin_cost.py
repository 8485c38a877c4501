"""Host cost of the API calls of one C3 transition (kvx_begin, the waves, the
commit, kvx_destroy), wall clock per call, median over reps -- the host side
of e2e, which bounds it at N>1 where the device step is short."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2510_11938_b200 import shard as S  # noqa: E402


def main():
    import torch
    from paper_2510_11938_b200 import kvx
    torch.cuda.set_device(0)
    plan = bench.Plan("c3")
    t = plan.t
    g = kvx.geometry(plan.L, plan.H, plan.D)
    old_dev, new_dev = S.placement(plan.L, t.old_boundaries, t.new_boundaries, 1)
    old, new = S.setup_rank_pools(kvx, g, t.old_boundaries, t.new_boundaries, old_dev, new_dev, 0, 0,
                                  plan.old_blocks, plan.dst_blocks)
    st = torch.cuda.Stream()
    rows = {"begin": [], "waves": [], "commit": [], "destroy": []}
    for rep in range(60):
        torch.cuda.synchronize()
        a = time.perf_counter()
        tr = kvx.Transition(g, t.old_boundaries, old, t.new_boundaries, new, 0, plan.N, plan.max_blocks,
                            plan.dst_blocks, plan.src_bt, epoch=t.epoch, max_sync_rounds=plan.scn.max_sync_rounds,
                            kv_bytes_per_token=plan.kv_bytes_per_token, stream=st.cuda_stream)
        b = time.perf_counter()
        w0 = t.events[0]
        tr.begin_refactor((w0.req, w0.hi))
        bench.run_events(tr, t.events[1:])
        c = time.perf_counter()
        tr.on_refactor_commit((t.live_req, t.live_kv), wait=False)
        d = time.perf_counter()
        tr.collect_commit()
        e = time.perf_counter()
        tr.close()
        f = time.perf_counter()
        if rep >= 10:
            rows["begin"].append((b - a) * 1e3)
            rows["waves"].append((c - b) * 1e3)
            rows["commit"].append((d - c) * 1e3)
            rows["destroy"].append((f - e) * 1e3)
    print(json.dumps({k: round(statistics.median(v), 4) for k, v in rows.items()} | {"unit": "ms host, median"}))
    for p in old + new:
        p.close()


if __name__ == "__main__":
    main()
