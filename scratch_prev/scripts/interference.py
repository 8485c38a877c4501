"""Sharing HBM with serving: wave 0 of the C3 refactor runs while a serving
proxy (back-to-back HBM-bound copies, the profile of decode attention reading
the KV cache) runs on another stream.  For each mover CTA cap
(kvx_transition_desc.max_ctas) prints the wave's time and KV GB/s and the
proxy's GB/s inside the wave window, against the proxy alone.

  python scripts/interference.py   (one B200; writes JSON lines to stdout)
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2510_11938_b200 import kvx  # noqa: E402
from paper_2510_11938_b200 import shard as S  # noqa: E402


def main():
    torch.cuda.set_device(0)
    plan = bench.Plan("c3")
    t = plan.t
    g = kvx.geometry(plan.L, plan.H, plan.D)
    old_dev, new_dev = S.placement(plan.L, t.old_boundaries, t.new_boundaries, 1)
    old_pools, new_pools = S.setup_rank_pools(kvx, g, t.old_boundaries, t.new_boundaries, old_dev, new_dev, 0, 0,
                                              plan.old_blocks, plan.dst_blocks,
                                              fill=(bench.SEED, plan.live, plan.tokens[plan.live], plan.src_bt))
    w0 = t.waves[0]
    kv_bytes = int((w0.hi - w0.lo).clip(min=0).sum()) * plan.kv_bytes_per_token
    # serving proxy: 2 GiB copies (read + write), back to back
    n = 1 << 30
    a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    a.fill_(1.0)
    s_srv, s_kv = torch.cuda.Stream(), torch.cuda.Stream()
    copy_bytes = 2 * a.numel() * a.element_size()

    def proxy(k):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(k + 1)]
        with torch.cuda.stream(s_srv):
            evs[0].record(s_srv)
            for i in range(k):
                b.copy_(a)
                evs[i + 1].record(s_srv)
        return evs

    # proxy alone
    torch.cuda.synchronize()
    evs = proxy(20)
    torch.cuda.synchronize()
    alone = copy_bytes * 19 / (evs[1].elapsed_time(evs[-1]) * 1e-3) / 1e9
    for cap in [0, 96, 64, 48, 32, 24, 16, 8]:
        res = []
        for rep in range(3):
            tr = kvx.Transition(g, t.old_boundaries, old_pools, t.new_boundaries, new_pools, 0, plan.N,
                                plan.max_blocks, plan.dst_blocks, plan.src_bt, epoch=t.epoch,
                                stream=s_kv.cuda_stream, max_ctas=cap)
            torch.cuda.synchronize()
            base = torch.cuda.Event(enable_timing=True)
            base.record(s_srv)
            evs = proxy(40)                       # ~40 x 0.65 ms of serving traffic queued
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_kv.wait_event(evs[2])               # the wave starts once serving is running
            e0.record(s_kv)
            tr.wave(w0.req, w0.lo, w0.hi)
            e1.record(s_kv)
            torch.cuda.synchronize()
            t0, t1 = base.elapsed_time(e0), base.elapsed_time(e1)
            stamps = [base.elapsed_time(e) for e in evs]
            inside = [i for i in range(1, len(stamps)) if stamps[i - 1] >= t0 and stamps[i] <= t1]
            srv = (copy_bytes * len(inside) / ((stamps[inside[-1]] - stamps[inside[0] - 1]) * 1e-3) / 1e9
                   if inside else None)
            res.append((t1 - t0, srv, stamps[-1] <= t1))
            tr.close()
        ms = float(np.median([r[0] for r in res]))
        srv = [r[1] for r in res if r[1] is not None]
        print(json.dumps({"max_ctas": cap, "wave0_ms": round(ms, 3), "kv_GBps": round(kv_bytes / (ms * 1e-3) / 1e9, 1),
                          "serving_GBps_during": round(float(np.median(srv)), 1) if srv else None,
                          "serving_alone_GBps": round(alone, 1),
                          "serving_outlasted_wave": not any(r[2] for r in res)}), flush=True)


if __name__ == "__main__":
    main()
