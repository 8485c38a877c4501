"""Device-time breakdown of one C3 transition step on one GPU: stream-ordered
events between the API calls (wave 0 incl. plan, final wave, commit, and the
gap to the next step)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_11938_b200 import kvx  # noqa: E402
from paper_2510_11938_b200 import shard as S  # noqa: E402
from paper_2510_11938_b200 import workload as W  # noqa: E402

plan = bench.Plan("c3")
t = plan.t
g = kvx.geometry(plan.L, plan.H, plan.D)
old_dev, new_dev = S.placement(plan.L, t.old_boundaries, t.new_boundaries, 1)
old, new = S.setup_rank_pools(kvx, g, t.old_boundaries, t.new_boundaries, old_dev, new_dev, 0, 0,
                              plan.old_blocks, plan.dst_blocks,
                              fill=(1, plan.live, plan.tokens[plan.live], plan.src_bt))
st = torch.cuda.Stream()
K = 30
trs = [kvx.Transition(g, t.old_boundaries, old, t.new_boundaries, new, 0, plan.N, plan.max_blocks,
                      plan.dst_blocks, plan.src_bt, epoch=t.epoch, stream=st.cuda_stream) for _ in range(K + 3)]
bar = next(e for e in t.events if isinstance(e, W.Barrier))
fin = t.waves[-1]
w0 = t.waves[0]
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
rows = []
for i, tr in enumerate(trs):
    ev = [E() for _ in range(5)]
    ev[0].record(st)
    tr.begin_refactor((w0.req, w0.hi))
    ev[1].record(st)
    tr.on_kv_sync_complete((bar.req, bar.kv), bar.inflight_batches)
    tr.on_kv_sync_complete((fin.req, fin.hi), 0)
    ev[2].record(st)
    tr.on_refactor_commit((t.live_req, t.live_kv), wait=False)
    ev[3].record(st)
    rows.append(ev)
torch.cuda.synchronize()
seg = {"wave0 (plan+move)": [], "final wave": [], "commit": [], "gap to next step": []}
for i in range(3, K + 2):
    ev = rows[i]
    seg["wave0 (plan+move)"].append(ev[0].elapsed_time(ev[1]))
    seg["final wave"].append(ev[1].elapsed_time(ev[2]))
    seg["commit"].append(ev[2].elapsed_time(ev[3]))
    seg["gap to next step"].append(ev[3].elapsed_time(rows[i + 1][0]))
mv = [tr.move_timings() for tr in trs[3:K + 2]]
out = {k: round(statistics.median(v) * 1000, 1) for k, v in seg.items()}
out["wave0 mover kernel"] = round(statistics.median(m[0][0] for m in mv) * 1000, 1)
out["final mover kernel"] = round(statistics.median(m[1][0] for m in mv) * 1000, 1)
print({"us": out})
for tr in trs:
    tr.collect_commit()
    tr.close()
