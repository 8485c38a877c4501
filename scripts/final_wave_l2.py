"""What the L2 holds when the barrier falls, and what that does to the stall.

The bench issues the final post-barrier wave right behind wave 0's 17 GB
mover, so the final wave starts with L2 full of wave 0's dirty lines.  In
the reference's timeline (engine.cpp:491-507, 637-687) decode iterations run
between wave 0 and the barrier, and the final wave moves what the last one
appended.  Modes (each rep: a fresh transition, wave 0, then):
  b2b     barrier + final wave right behind wave 0 (the bench's step)
  clean   a 1 GiB read between wave 0 and the barrier (L2 holds clean lines)
  decode  the 1 GiB read, then the last decode step re-appends the final
          wave's source rows (same payload) -- they sit dirty in L2, as after
          a real decode iteration
Prints one JSON line per mode: final-wave mover us (its own %globaltimer) and
barrier -> commit-result stall us (CUDA events), medians.
Usage (gpurun): python scripts/final_wave_l2.py --reps 15
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
from paper_2510_11938_b200 import workload as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--modes", default="b2b,clean,decode")
    args = ap.parse_args()
    import numpy as np
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
    sp = stream.cuda_stream
    flush = torch.empty(1 << 28, dtype=torch.float32, device="cuda")  # 1 GiB
    flush.fill_(1.0)
    fin = [w for w in t.waves if w.final][-1]
    ranges = W.stage_ranges(plan.L, t.old_boundaries)

    def make():
        return kvx.Transition(g, t.old_boundaries, old_pools, t.new_boundaries, new_pools, 0, plan.N,
                              plan.max_blocks, plan.dst_blocks, plan.src_bt, epoch=t.epoch,
                              max_sync_rounds=plan.scn.max_sync_rounds,
                              kv_bytes_per_token=plan.kv_bytes_per_token, stream=sp)

    out = []
    for mode in args.modes.split(","):
        fw, st = [], []
        for r in range(args.reps + 2):
            tr = make()
            w0 = t.events[0]
            tr.begin_refactor((w0.req, w0.hi))
            rem = bench.run_events(tr, t.events[1:], None, stop_at_barrier=True)
            if mode in ("clean", "decode"):
                with torch.cuda.stream(stream):
                    flush.sum()
            if mode == "decode":
                for k, (b, e) in enumerate(ranges):
                    old_pools[k].append_pattern(bench.SEED, b, fin.req, fin.lo, fin.hi, plan.src_bt, stream=sp)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            bench.run_events(tr, rem, lambda: e0.record(stream))
            tr.on_refactor_commit((t.live_req, t.live_kv), wait=True)
            e1.record(stream)
            torch.cuda.synchronize()
            if r == 0:
                bad = tr.verify_pattern(bench.SEED, t.live_req, t.live_kv)
                assert bad == 0, (mode, bad)
            if r >= 2:
                mv = tr.move_timings()
                fw.append(mv[-1][0] * 1e3)
                st.append(e0.elapsed_time(e1) * 1e3)
            tr.close()
        fb = int(np.sum(fin.hi - fin.lo)) * plan.token_bytes * plan.L * 2
        line = {"mode": mode, "final_wave_us": round(statistics.median(fw), 2), "final_wave_min_us": round(min(fw), 2),
                "stall_us": round(statistics.median(st), 2), "stall_min_us": round(min(st), 2),
                "final_wave_rw_bytes": fb,
                "final_wave_frac": round(fb / (statistics.median(fw) * 1e-6) / 1e9 / bench.peaks()[0], 4)}
        print(json.dumps(line), flush=True)
        out.append(line)


if __name__ == "__main__":
    main()
