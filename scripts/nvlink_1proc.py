"""C3 (13B 8->4, real geometry) across two GPUs from ONE process (one kvx
handle per device, pools of the other device as NVLink peers): the shape
ncu can profile (a multi-rank run under ncu hangs in CUDA IPC).
  python scripts/nvlink_1proc.py --placement disjoint|oneway --move push|pull [--reps R]
prints one JSON line per rep: wave-0 mover ms per device, GB/s per direction.
Under ncu (scripts/nvlink_ncu.sh) the kvx_bulk_kernel launches carry the
nvltx / nvlrx byte counters."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2510_11938_b200 import shard as S  # noqa: E402
from paper_2510_11938_b200 import workload as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--placement", default="disjoint")
    ap.add_argument("--move", default="push", choices=["push", "pull"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--verify", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_2510_11938_b200 import kvx
    if kvx.device_count() < 2:
        raise SystemExit("needs 2 GPUs")
    plan = bench.Plan("c3")
    t = plan.t
    L = plan.L
    g = kvx.geometry(L, plan.H, plan.D)
    old_dev, new_dev = S.placement(L, t.old_boundaries, t.new_boundaries, 2, args.placement)
    old_pools, new_pools = [], []
    for k, (b, e) in enumerate(W.stage_ranges(L, t.old_boundaries)):
        p = kvx.Pool(old_dev[k], g, e - b, plan.old_blocks)
        p.fill_pattern(bench.SEED, b, plan.live, plan.tokens[plan.live], plan.src_bt)
        old_pools.append(p)
    for j, (b, e) in enumerate(W.stage_ranges(L, t.new_boundaries)):
        new_pools.append(kvx.Pool(new_dev[j], g, e - b, plan.dst_blocks))
    hbm, out, inn = S.link_bytes(L, t.old_boundaries, t.new_boundaries, old_dev, new_dev,
                                 plan.wave0_tokens * 2 * plan.token_bytes, 2)
    for rep in range(args.reps):
        hs = [kvx.Transition(g, t.old_boundaries, old_pools, t.new_boundaries, new_pools, d, plan.N,
                             plan.max_blocks, plan.dst_blocks, plan.src_bt, epoch=t.epoch,
                             pull=args.move == "pull") for d in (0, 1)]
        for d in (0, 1):
            torch.cuda.synchronize(d)
        w0 = t.waves[0]
        for h in hs:
            h.wave(w0.req, w0.lo, w0.hi)
        for h in hs:
            h.wait()
        ms = [h.move_timings()[0][0] if h.move_timings() else 0.0 for h in hs]
        bad = 0
        if args.verify and rep == args.reps - 1:
            for w in t.waves[1:]:
                for h in hs:
                    h.wave(w.req, w.lo, w.hi)
                for h in hs:
                    h.wait()
            bad = sum(h.verify_pattern(bench.SEED, t.live_req, t.live_kv) for h in hs)
        print(json.dumps({"placement": args.placement, "move": args.move, "rep": rep,
                          "wave0_mover_ms": [round(x, 4) for x in ms],
                          "nvlink_out_bytes": out, "nvlink_in_bytes": inn,
                          "GBps_per_direction": [round(o / (m * 1e-3) / 1e9, 1) if m else None
                                                 for o, m in zip(out, ms)],
                          "frac_of_770": [round(o / (m * 1e-3) / 1e9 / 770.0, 4) if m else None
                                          for o, m in zip(out, ms)],
                          "mismatched_words": int(bad)}), flush=True)
        for h in hs:
            h.close()
    for p in old_pools + new_pools:
        p.close()


if __name__ == "__main__":
    main()
