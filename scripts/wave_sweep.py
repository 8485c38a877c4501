"""Mover ring / grid sweep per wave kind, in one process (pools built once).

For each (KVX_BULK_CFG_TOK | KVX_BULK_CFG_SLAB variant, grid) the C3 (or
--config) transition runs --steps times and the median CUDA-event time of
each wave's mover is printed as one JSON line.  Every configuration's
destination is checked against the payload before it is timed.
Usage (gpurun): python scripts/wave_sweep.py --kind tok --variants 0,8,9 --grids 148,296
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2510_11938_b200 import shard as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--kind", default="tok", choices=["tok", "slab"])
    ap.add_argument("--variants", default="0")
    ap.add_argument("--grids", default="148")
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    import torch
    from paper_2510_11938_b200 import kvx
    torch.cuda.set_device(0)
    plan = bench.Plan(args.config)
    t = plan.t
    g = kvx.geometry(plan.L, plan.H, plan.D)
    old_dev, new_dev = S.placement(plan.L, t.old_boundaries, t.new_boundaries, 1)
    old_pools, new_pools = S.setup_rank_pools(
        kvx, g, t.old_boundaries, t.new_boundaries, old_dev, new_dev, 0, 0, plan.old_blocks, plan.dst_blocks,
        fill=(bench.SEED, plan.live, plan.tokens[plan.live], plan.src_bt))
    stream = torch.cuda.Stream()
    peak = bench.peaks()[0]
    for v in args.variants.split(","):
        for grid in [int(x) for x in args.grids.split(",")]:
            os.environ["KVX_BULK_CFG_" + args.kind.upper()] = v
            if args.kind == "tok":
                os.environ["KVX_BULK_GRID_TOK"] = str(grid)
            else:
                os.environ["KVX_BULK_GRID"] = str(grid)
            times = []
            for s in range(args.steps + 2):
                tr = kvx.Transition(g, t.old_boundaries, old_pools, t.new_boundaries, new_pools, 0, plan.N,
                                    plan.max_blocks, plan.dst_blocks, plan.src_bt, epoch=t.epoch,
                                    max_sync_rounds=plan.scn.max_sync_rounds,
                                    kv_bytes_per_token=plan.kv_bytes_per_token, stream=stream.cuda_stream)
                bench.run_step(tr, t)
                torch.cuda.synchronize()
                if s == 0:
                    bad = tr.verify_pattern(bench.SEED, t.live_req, t.live_kv)
                    assert bad == 0, (v, grid, bad)
                if s >= 2:
                    times.append(tr.move_timings())
                tr.close()
            n = len(times[0])
            ms = [statistics.median(m[i][0] for m in times) for i in range(n)]
            by = [times[0][i][1] for i in range(n)]
            print(json.dumps({"config": args.config, "kind": args.kind, "variant": v, "grid": grid,
                              "move_ms_by_wave": [round(x, 4) for x in ms],
                              "frac_by_wave": [round(b / (m * 1e-3) / 1e9 / peak, 4) for b, m in zip(by, ms)]}),
                  flush=True)
            for k in ("KVX_BULK_CFG_TOK", "KVX_BULK_CFG_SLAB", "KVX_BULK_GRID_TOK", "KVX_BULK_GRID"):
                os.environ.pop(k, None)
    if args.kind == "tok":
        # control: one contiguous copy of the final wave's bytes (read side), so the
        # token wave's scatter cost is separated from what a launch of this size costs
        fin = [w for w in t.waves if w.final] or t.waves[-1:]
        nbytes = int((fin[0].hi - fin[0].lo).clip(min=0).sum()) * 2 * plan.token_bytes * plan.L
        a = torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda")
        b = torch.empty_like(a)
        best = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.copy_(a)
            e1.record()
            torch.cuda.synchronize()
            best.append(e0.elapsed_time(e1))
        ms = statistics.median(best)
        print(json.dumps({"config": args.config, "control": "contiguous torch copy of the final wave's bytes",
                          "bytes_read": nbytes, "ms": round(ms, 4),
                          "frac": round(2 * nbytes / (ms * 1e-3) / 1e9 / peak, 4)}), flush=True)
    for p in old_pools + new_pools:
        p.close()


if __name__ == "__main__":
    main()
