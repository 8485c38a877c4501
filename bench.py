#!/usr/bin/env python
"""Benchmark of the B200-native inflight-refactor KV transition.

One "step" = one complete inflight refactor of the BASELINE config-3 workload
(Llama-2-13B shape, 8->4 stage merge, ~17 GB live paged KV), driven by the
reference engine's OWN wave plan for it (tests/golden/llama13b_8to4.jsonl,
extracted from the unmodified reference): wave 0 over every live token, the
barrier / drain decision, the final post-barrier wave, commit (Eq. 10 check +
block-table compaction).  All through the kvx C-ABI (include/kvx.h).

  value     KV-refactor GB/s = reference-accounted KV bytes of the step
            (kv_synced_bytes, engine.cpp:644-684) / device time per step,
            KV resident in HBM (CUDA events on the transition stream).
  e2e       same metric through the public API with the control inputs in
            host memory: kvx_begin (grant + source block table H2D), the wave
            descriptors H2D, the commit result (violations + compacted block
            table + free list) D2H for every step -- collected once the next
            step is issued (async commit) -- host wall clock.
  stall     barrier -> commit (engine.cpp:676-686), three ways: device time
            of the final wave + commit; host-observed (barrier handler call ->
            commit result on the host); and under the reference's conditions
            (weights migrated beside wave 0, commit at max(final wave, weights
            ready), handoff measured / drain = the reference's simulated drain
            + measured final wave and commit).
  roofline  dominant kernel = the TMA bulk mover (kvx_bulk_kernel) of wave 0:
            algorithmic read+write bytes / its CUDA-event duration vs
            MEASURED_PEAKS hbm_gbs (N>1: vs the HBM / NVLink bound of the
            busiest GPU); traffic = DRAM bytes of the same launch from an ncu
            pass run by this bench (child `--traffic-probe`), N=1.

`--impl reference` times the reference's CPU path for the same metric and
config: the oracle restatement (oracle/kvx_oracle.c, all host threads) over
the full wave plan, since the reference itself moves no bytes.

Launch: python bench.py [--gpus N --steps K --warmup W]; N>1 via
torch.distributed.run (one rank per GPU, NVLink P2P through CUDA IPC pools).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2510_11938_b200 import shard as S  # noqa: E402
from paper_2510_11938_b200 import workload as W  # noqa: E402

CONFIGS = {
    # name: (golden, shape, description)
    "c3": ("llama13b_8to4", "llama2-13b",
           "Llama-2-13B shape (40 layers, 40 KV heads, d=128, fp16), 8->4 stage merge, "
           "256 live requests, ~17 GB paged KV (16-token blocks)"),
    "c1": ("llama7b_4to2", "llama2-7b",
           "Llama-2-7B shape (32 layers, 32 KV heads), 4->2 merge, 16 requests, ~4k tokens"),
    "c2": ("llama7b_2to8", "llama2-7b",
           "Llama-2-7B shape, 2->8 split, 1024 live requests"),
    "c4": ("llama70b_8to2to8", "llama2-70b",
           "Llama-2-70B GQA shape (80 layers, 8 KV heads), 8->2 and 2->8"),
    "c4r": ("llama70b_8to2to8", "llama2-70b",
            "Llama-2-70B GQA shape (80 layers, 8 KV heads), same-K re-placement of all 8 stages "
            "(10 layers each), ~64k live tokens = 21 GB; wave plan of the reference's 2->8 transition"),
}
SEED = 0xB200
METRIC = "KV-refactor GB/s (% of HBM/NVLink roofline); refactor stall ms at 1/2/4/8 B200"


def source_hash() -> str:
    """sha256 (16 hex) of the product sources: csrc/* and include/kvx.h.  An
    ncu capture is only quoted for the build it was taken of."""
    import hashlib
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2510_11938_b200", "csrc")
    for f in sorted(os.listdir(csrc)) + ["../../include/kvx.h"]:
        with open(os.path.join(csrc, f), "rb") as fh:
            h.update(f.encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


def _ncu_dram(path: str):
    """dram__bytes_read.sum + dram__bytes_write.sum (bytes) and
    gpu__time_duration.sum (ms) of the single launch in an ncu --csv log."""
    import csv
    total, dur = 0.0, None
    with open(path) as f:
        rows = [r for r in csv.reader(f) if len(r) > 14]
    if not rows:
        return None, None
    head = rows[0]
    try:
        im, iu, iv = head.index("Metric Name"), head.index("Metric Unit"), head.index("Metric Value")
    except ValueError:
        im, iu, iv = 12, 13, 14
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    for r in rows[1:]:
        v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        if r[im] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            total += v
        elif r[im] == "gpu__time_duration.sum":
            dur = v
    return (total or None), dur


def ncu_traffic(cfg: str, timeout_s: float = 240.0, world: int = 1, placement: str = "affinity"):
    """DRAM traffic of the dominant launch (the wave-0 TMA bulk mover), taken
    IN THIS RUN: ncu (one pass, two dram counters, --clock-control none) over
    a child `bench.py --traffic-probe` that builds the same pools and issues
    the same wave 0 once.  Returns (bytes or None, provenance dict)."""
    import shutil
    import subprocess
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    src = {"source_hash": source_hash(), "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
           "-k regex:kvx_bulk_kernel -c 1 over `bench.py --traffic-probe` (this run, this build)"}
    if not ncu:
        return None, dict(src, error="ncu not found")
    log = os.path.join("/tmp", f"kvx_traffic_{os.getpid()}.csv")
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:kvx_bulk_kernel", "-c", "1", "--csv", "--log-file", log,
           sys.executable, os.path.abspath(__file__), "--traffic-probe", "--config", cfg,
           "--probe-world", str(world), "--placement", placement]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s)
        if out.returncode != 0:
            return None, dict(src, error=f"ncu rc={out.returncode}: {(out.stderr or out.stdout)[-300:]}")
        traffic, dur = _ncu_dram(log)
        return traffic, dict(src, ncu_launch_ms=dur)
    except Exception as e:  # report, never fail the bench on it
        return None, dict(src, error=str(e)[:300])
    finally:
        if os.path.exists(log):
            os.remove(log)


def traffic_probe(args):
    """Child of ncu_traffic (runs under ncu): the bench's pools for the config
    and its wave 0, once; the first kvx_bulk_kernel launch is wave 0's mover.
    --probe-world N: rank 0's share of the N-GPU placement (its own pools
    only; used when rank 0 moves no layer over NVLink)."""
    import torch
    from paper_2510_11938_b200 import kvx
    torch.cuda.set_device(0)
    plan = Plan(args.config)
    t = plan.t
    g = kvx.geometry(plan.L, plan.H, plan.D)
    old_dev, new_dev = S.placement(plan.L, t.old_boundaries, t.new_boundaries, args.probe_world, args.placement)
    old_pools, new_pools = S.setup_rank_pools(kvx, g, t.old_boundaries, t.new_boundaries, old_dev, new_dev, 0, 0,
                                              plan.old_blocks, plan.dst_blocks, all_gather=None, fill=None)
    for j, (b, e) in enumerate(W.stage_ranges(plan.L, t.new_boundaries)):
        if new_pools[j] is None:  # another rank's new stage: kvx_begin wants every pool; none of
            new_pools[j] = kvx.Pool(0, g, e - b, plan.dst_blocks)  # rank 0's layers go there
    tr = kvx.Transition(g, t.old_boundaries, old_pools, t.new_boundaries, new_pools, 0, plan.N, plan.max_blocks,
                        plan.dst_blocks, plan.src_bt, epoch=t.epoch, max_sync_rounds=plan.scn.max_sync_rounds,
                        kv_bytes_per_token=plan.kv_bytes_per_token)
    if args.probe_all_waves:  # every wave + commit (ncu -s k picks the k-th mover launch)
        run_step(tr, t)
    else:
        w0 = t.waves[0]
        tr.wave(w0.req, w0.lo, w0.hi)
        tr.wait()
    tr.close()
    for p in old_pools + new_pools:
        if p is not None:
            p.close()
    return 0


def host_cpu():
    """(logical CPUs usable by this process, CPU model) of the host."""
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return n, model


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled in-process through NVML (one call
    per 20 ms from a thread) while the timed region runs."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int, period_s: float = 0.02):
        self.index, self.period = index, period_s
        self.rows = []
        self.err = None
        self._stop = threading.Event()
        self._thr = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # NVML absent
            self.err = f"nvml: {e}"
            return
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.rows.append((time.time(), sm, rs))
            except Exception as e:
                self.err = str(e)
                return
            self._stop.wait(self.period)

    def stop(self):
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=2)

    def summary(self, t0: float, t1: float):
        sel = [r for r in self.rows if t0 - 0.025 <= r[0] <= t1 + 0.025] or self.rows[-3:]
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": self.err or "no samples"}
        reasons = set()
        for _, _, rs in sel:
            for bit, name in self.REASONS.items():
                if rs & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r[1] for r in sel), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sel), "source": "nvml"}


# ------------------------------------------------------------------ workload
class Plan:
    """The golden transition and everything derived from it."""

    def __init__(self, cfg: str):
        golden, shape, self.desc = CONFIGS[cfg]
        self.golden = golden
        self.scn = W.load_golden(golden)
        self.t = [t for t in self.scn.transitions if t.outcome == "commit"][-1] if cfg in ("c4", "c4r") \
            else self.scn.transitions[0]
        if cfg == "c4r":
            # BASELINE C4: same-K re-placement.  The reference drops same-plan
            # directives (engine.cpp:562) -- parity unpinned; its last wave
            # plan is reused with the old 8-stage cut on both sides.
            import copy
            self.t = copy.copy(self.t)
            self.t.old_boundaries = list(self.t.new_boundaries)
        self.L, self.H, self.D = W.SHAPES[shape]
        self.N = self.scn.num_requests
        self.tokens = self.t.max_tokens(self.N)
        self.max_blocks = int(max(1, (self.tokens.max() + 15) // 16))
        self.src_bt, self.old_blocks = W.fragmented_block_table(self.tokens, self.max_blocks, 16, seed=7)
        self.dst_blocks = int(((self.tokens + 15) // 16).sum())
        self.live = np.nonzero(self.tokens)[0].astype(np.int32)
        self.token_bytes = self.H * self.D * 2
        self.kv_bytes_per_token = self.scn.kv_bytes_per_token
        self.step_tokens = sum(int((w.hi - w.lo).clip(min=0).sum()) for w in self.t.waves)
        self.step_bytes = self.step_tokens * self.kv_bytes_per_token  # reference-accounted
        w0 = self.t.waves[0]
        self.wave0_tokens = int((w0.hi - w0.lo).clip(min=0).sum())


def run_events(tr, ev, at_barrier=None, stop_at_barrier=False):
    """Issue a transition's events after wave 0 through the reference-shaped
    handlers, in engine order (engine.cpp:651-688): delta waves, barrier
    waits, the final wave.  at_barrier() is called right before the handler
    call that issues the final post-barrier wave.  stop_at_barrier: return
    the remaining events at the first barrier / final wave instead."""
    from paper_2510_11938_b200 import kvx
    ev = list(ev)
    while ev:
        e = ev[0]
        if stop_at_barrier and (isinstance(e, W.Barrier) or e.final):
            return ev
        ev.pop(0)
        if isinstance(e, W.Barrier):
            if e.inflight_batches > 0:
                act, _ = tr.on_kv_sync_complete((e.req, e.kv), e.inflight_batches)
                assert act == kvx.ACT_BARRIER_WAIT, act
                continue
            if at_barrier is not None:
                at_barrier()
            act, _ = tr.on_kv_sync_complete((e.req, e.kv), 0)
            assert act == kvx.ACT_FINAL, act
            ev.pop(0)  # the final wave this handler just issued
        elif e.final:
            if at_barrier is not None:
                at_barrier()
            act, _ = tr.on_kv_sync_complete((e.req, e.hi), 0)
            assert act == kvx.ACT_FINAL, act
        else:
            act, _ = tr.on_kv_sync_complete((e.req, e.hi), 1)
            assert act == kvx.ACT_DELTA, act
    return []


def run_step(tr, t, stall_ev=None, wait=True, mark=None):
    """One transition through the reference-shaped handlers, in the order the
    reference engine issued them (engine.cpp:637-713).  stall_ev = (start,
    end, stream): start is recorded right before the call that issues the
    final post-barrier wave, end after commit -- the B200 refactor stall.
    mark(kind) is called at the same two points ("barrier", "commit")."""
    w0 = t.events[0]
    tr.begin_refactor((w0.req, w0.hi))

    def at_barrier():
        if stall_ev is not None:
            stall_ev[0].record(stall_ev[2])
        if mark is not None:
            mark("barrier")

    run_events(tr, t.events[1:], at_barrier)
    res = tr.on_refactor_commit((t.live_req, t.live_kv), wait=wait)
    if stall_ev is not None:
        stall_ev[1].record(stall_ev[2])  # device time at which the commit result is on the host
    if mark is not None:
        mark("commit")
    return res


def host_observed_stall(make, t, reps: int = 8):
    """The stall as the engine's handlers see it on the host: from the call of
    the barrier handler that issues the final wave (engine.cpp:676-687) --
    after the host learnt that the earlier waves completed (kvx_wait, the
    KvSyncComplete arrival) -- to the commit result (violations + compacted
    block table) back on the host (engine.cpp:690-713).  Wall clock, median."""
    out = []
    for rep in range(reps + 1):
        tr = make()
        marks = {}

        def mark(kind):
            if kind == "barrier":
                tr.wait()
            marks[kind] = time.perf_counter()
        run_step(tr, t, mark=mark)
        tr.close()
        if rep:
            out.append((marks["commit"] - marks["barrier"]) * 1e3)
    return statistics.median(out), min(out), max(out)


def serving_stall(make, t, old_pools, old_ranges, src_bt, stream, dev, reps: int = 8, read_bytes: int = 1 << 30):
    """The device stall with a decode iteration between the last pre-barrier
    wave and the barrier, as in the reference's timeline: the final wave moves
    the tokens decode appended after the last snapshot (engine.cpp:491-507,
    676-687), so at least one decode step runs between wave 0 and the
    barrier.  The timed loop's step issues the final wave right behind wave
    0's 17 GB mover instead, and the final wave then pays the write-back of
    wave 0's dirty L2 lines (`scripts/final_wave_l2.py`: 74 vs 63 us).
    Stand-in for the decode step, per rep: the append of exactly the rows the
    final wave moves (kvx_pool_append_pattern: same payload, dirty in L2),
    then `read_bytes` of reads (the step's attention reads of the KV cache,
    which leave L2 holding clean lines).  Returns the median barrier ->
    commit-result device time and the final-wave mover time (ms)."""
    import torch
    fin = next((w for w in reversed(t.waves) if w.final), None)
    if fin is None:
        return None
    flush = torch.ones(read_bytes // 4, dtype=torch.float32, device=dev)
    sp = stream.cuda_stream
    st, fw = [], []
    for rep in range(reps + 1):
        tr = make()
        w0 = t.events[0]
        tr.begin_refactor((w0.req, w0.hi))
        ev = run_events(tr, t.events[1:], stop_at_barrier=True)
        for k, (b, _e) in enumerate(old_ranges):
            if old_pools[k] is not None and not old_pools[k].imported:  # this rank's own old stages
                old_pools[k].append_pattern(SEED, b, fin.req, fin.lo, fin.hi, src_bt, stream=sp)
        with torch.cuda.stream(stream):
            flush.sum()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        run_events(tr, ev, lambda: a0.record(stream))
        tr.on_refactor_commit((t.live_req, t.live_kv), wait=False)
        a1.record(stream)
        torch.cuda.synchronize(dev)
        res = tr.collect_commit()
        assert res.violations == t.violations, res.violations
        if rep:
            st.append(a0.elapsed_time(a1))
            mv = tr.move_timings()
            fw.append(mv[-1][0] if mv else 0.0)  # 0: no mover of this rank's own (max over ranks)
        tr.close()
    del flush
    return statistics.median(st), statistics.median(fw), min(st)


def reference_condition_stall(make, t, plan, shape, stream, dev, reps: int = 4):
    """The stall under the reference's own conditions (engine.cpp:614-687):
    the new stages' weights are migrated WHILE wave 0 runs (same HBM; the
    reference starts the loads at the grant, :621-631), and commit waits for
    max(final wave, weights ready) (:686).  Measured on the device for two
    barrier policies:
      handoff  the in-flight micro-batches move to their new owners at the
               barrier (kvx_handoff), the final wave goes out at once, commit
               waits on the weights: barrier -> commit, all measured;
      drain    the reference's policy: the old pipeline finishes its in-flight
               micro-batches first.  The drain is compute this data plane does
               not run, so its length is the reference's simulated one (barrier
               -> final wave in the golden timeline); the rest is measured:
               max(drain, weights left at the barrier) + final wave + commit.
    Returns a dict (None when the plan has no barrier or weights do not fit)."""
    import torch
    from paper_2510_11938_b200 import kvx
    bars = [e for e in t.events if isinstance(e, W.Barrier)]
    fin = next((w for w in t.waves if w.final), None)
    L = plan.L
    params = {"llama2-13b": 26.0e9, "llama2-7b": 13.5e9, "llama2-70b": 138.0e9}[shape]
    lb = int(params / L) // 4096 * 4096
    if lb * L * 2 > 120e9 or fin is None:
        return None
    wold = [torch.empty((e - b) * lb, dtype=torch.uint8, device=dev) for b, e in W.stage_ranges(L, t.old_boundaries)]
    wnew = [torch.empty((e - b) * lb, dtype=torch.uint8, device=dev) for b, e in W.stage_ranges(L, t.new_boundaries)]
    wstream = torch.cuda.Stream(device=dev)
    row = {"llama2-13b": 5120, "llama2-7b": 4096, "llama2-70b": 8192}[shape] * 2
    bar = bars[0] if bars else None
    mbs = bar.microbatches if bar is not None else []
    srcs = [torch.full((max(m.tokens, 1) * row,), m.batch % 251, dtype=torch.uint8, device=dev) for m in mbs]
    cap = sum(m.tokens * row + 256 for m in mbs) + 256
    arenas = [torch.zeros(cap, dtype=torch.uint8, device=dev) for _ in range(len(t.new_boundaries) + 1)]
    res = {}
    for mode in ("handoff", "drain"):
        rows = []
        for rep in range(reps + 1):
            tr = make()
            if mode == "handoff":
                tr.set_handoff(True)
            torch.cuda.synchronize(dev)
            E = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            E[0].record(stream)                       # the grant: loads and wave 0 start together
            wstream.wait_event(E[0])
            kvx.weights_migrate(dev, L, lb, t.old_boundaries, [x.data_ptr() for x in wold], t.new_boundaries,
                                [x.data_ptr() for x in wnew], stream=wstream.cuda_stream)
            E[1].record(wstream)                      # weights ready (load_ready_ms)
            w0 = t.events[0]
            tr.begin_refactor((w0.req, w0.hi))
            ev = run_events(tr, t.events[1:], stop_at_barrier=True)   # delta waves before the barrier
            E[2].record(stream)                       # the barrier: earlier waves done
            e = ev[0]
            if mode == "handoff" and isinstance(e, W.Barrier):
                live = (e.req, e.kv)
                act, _ = tr.on_kv_sync_complete(live, e.inflight_batches)
                assert act == kvx.ACT_FINAL, act
                if mbs:
                    tr.handoff(row, [(m.batch, m.after, m.tokens, s_.data_ptr()) for m, s_ in zip(mbs, srcs)],
                               [x.data_ptr() for x in arenas], [cap] * len(arenas))
                want_v = 0
            else:  # drain: barrier wait(s), then the final wave over the drained live set
                run_events(tr, ev)
                live, want_v = (t.live_req, t.live_kv), t.violations
            E[3].record(stream)                       # final wave (+ handoff) issued
            stream.wait_event(E[1])                   # commit at max(final, load_ready) (:686)
            r = tr.on_refactor_commit(live)
            E[4].record(stream)
            torch.cuda.synchronize(dev)
            assert r.violations == want_v, (mode, r.violations, want_v)
            tr.close()
            if rep:
                rows.append((E[0].elapsed_time(E[2]), E[0].elapsed_time(E[1]), E[2].elapsed_time(E[4])))
        med = [statistics.median(x[i] for x in rows) for i in range(3)]
        res[mode] = {"barrier_after_grant_ms": round(med[0], 4), "weights_ready_after_grant_ms": round(med[1], 4),
                     "barrier_to_commit_ms": round(med[2], 4)}
    drain_sim = (fin.t_ms - bar.barrier_ms) if (bar is not None and getattr(fin, "t_ms", None) is not None) else None
    d = res["drain"]
    w_left = max(0.0, d["weights_ready_after_grant_ms"] - d["barrier_after_grant_ms"])
    out = {"weights_bytes": lb * L, "weights_concurrent_with_wave0": True,
           "handoff": dict(res["handoff"], stall_ms=res["handoff"]["barrier_to_commit_ms"]),
           "drain": dict(d, drain_ms_reference_simulated=drain_sim,
                         stall_ms=None if drain_sim is None else round(max(drain_sim, w_left) + d["barrier_to_commit_ms"], 4)),
           "reference_simulated_stall_ms": t.simulated_stall_ms(),
           "note": "reference condition (engine.cpp:614-687): weights migrated concurrently with wave 0 on the "
                   "same HBM, commit at max(final wave, weights ready); handoff = measured barrier -> commit "
                   "on the device; drain = the reference's simulated drain + measured final wave and commit"}
    del wold, wnew, arenas, srcs
    return out


def nvlink_probe(kvx, torch, dist, plan, g, rank, world, dev, gather, reps: int = 5):
    """Wave 0 of the same transition under the reference's DISJOINT grant
    (engine.cpp:584-591: the new stages on GPUs that do not hold the model's
    old stages; placement 'disjoint'), so every KV byte crosses NVLink, with
    the default per-layer movers.  Max over ranks of the mover time against
    the NVLink roofline (770 GB/s per direction, measured peer copy).  The
    bench's own placement (affinity) keeps layers local where it can; this
    puts the link itself in every N>1 line.  Returns a dict."""
    t, L = plan.t, plan.L
    old_dev, new_dev = S.placement(L, t.old_boundaries, t.new_boundaries, world, "disjoint")
    layer_pull = S.move_plan(L, t.old_boundaries, t.new_boundaries, old_dev, new_dev, "auto")
    old_pools, new_pools = S.setup_rank_pools(
        kvx, g, t.old_boundaries, t.new_boundaries, old_dev, new_dev, rank, dev, plan.old_blocks, plan.dst_blocks,
        all_gather=gather, fill=(SEED, plan.live, plan.tokens[plan.live], plan.src_bt), layer_pull=layer_pull)
    dist.barrier()
    stream = torch.cuda.Stream(device=dev)
    w0 = t.waves[0]
    ms = []
    for rep in range(reps + 1):
        tr = kvx.Transition(g, t.old_boundaries, old_pools, t.new_boundaries, new_pools, dev, plan.N,
                            plan.max_blocks, plan.dst_blocks, plan.src_bt, epoch=t.epoch,
                            stream=stream.cuda_stream, layer_pull=layer_pull)
        dist.barrier()
        torch.cuda.synchronize(dev)
        tr.wave(w0.req, w0.lo, w0.hi)
        tr.wait()
        m = tr.move_timings()
        if rep:
            ms.append(m[0][0] if m else 0.0)
        tr.close()
    dist.barrier()
    med = torch.tensor([statistics.median(ms)], dtype=torch.float64, device=dev)
    dist.all_reduce(med, op=dist.ReduceOp.MAX)
    w0_ms = float(med.item())
    hbm, out, inn = S.link_bytes(L, t.old_boundaries, t.new_boundaries, old_dev, new_dev,
                                 plan.wave0_tokens * 2 * plan.token_bytes, world)
    t_roof = max(max(o for o in out) / 770e9, max(i for i in inn) / 770e9, max(h for h in hbm) / (peaks()[0] * 1e9))
    for p in old_pools + new_pools:
        if p is not None and p.imported:
            p.close()
    dist.barrier()
    for p in old_pools + new_pools:
        if p is not None and not p.imported:
            p.close()
    dist.barrier()
    return {"placement": {"mode": "disjoint", "old_stage_gpu": old_dev, "new_stage_gpu": new_dev},
            "movers": "auto", "pulled_layers": int(sum(layer_pull)), "wave0_mover_ms": round(w0_ms, 4),
            "nvlink_out_bytes_per_gpu": [int(x) for x in out], "nvlink_in_bytes_per_gpu": [int(x) for x in inn],
            "t_roof_ms": round(t_roof * 1e3, 4), "frac": round(t_roof * 1e3 / w0_ms, 4),
            "GBps_per_direction_busiest": round(max(out + inn) / (w0_ms * 1e-3) / 1e9, 1),
            "note": "every KV byte crosses NVLink (the reference's disjoint grant); max over ranks; roofline "
                    "770 GB/s per direction (measured peer copy), HBM for the local share"}


# ------------------------------------------------------------ NCCL baseline
def nccl_baseline(kvx, torch, dist, plan, g, old_pools, old_dev, new_dev, rank, world, dev, stream,
                  reps=5):
    """Wave 0 the library-call way: gather every local-source layer into a
    local copy of the destination layout (the same kvx mover, local HBM
    only), then ship each remote layer region with NCCL send/recv (grouped,
    batch_isend_irecv) straight into the owner's pool.  Returns device ms
    (gather, nccl, total), max over ranks, or None if nothing crosses GPUs."""
    t, L = plan.t, plan.L
    ob, nb = t.old_boundaries, t.new_boundaries
    cross = [l for l in range(L) if old_dev[S.stage_of(ob, l)] != new_dev[S.stage_of(nb, l)]]
    if not cross:
        return None
    bb = g.block_bytes
    ranges = W.stage_ranges(L, nb)
    bufs, pools = [], []
    for j, (b, e) in enumerate(ranges):
        n = (e - b) * plan.dst_blocks * bb
        buf = torch.empty(n, dtype=torch.uint8, device=dev)
        bufs.append(buf)
        pools.append(kvx.Pool.wrap(dev, buf.data_ptr(), n, g, e - b, plan.dst_blocks))
    w0 = t.waves[0]
    alloc0 = int(((w0.hi + 15) // 16).sum())  # fresh pools: wave 0 fills blocks [0, alloc0) per layer
    ops_spec = []
    for l in cross:
        src, dst = old_dev[S.stage_of(ob, l)], new_dev[S.stage_of(nb, l)]
        j = S.stage_of(nb, l)
        off = (l - ranges[j][0]) * plan.dst_blocks * bb
        if rank == src:
            ops_spec.append(("send", j, off, dst))
        elif rank == dst:
            ops_spec.append(("recv", j, off, src))
    sp = stream.cuda_stream
    res = []
    for rep in range(reps + 1):
        tr = kvx.Transition(g, ob, old_pools, nb, pools, dev, plan.N, plan.max_blocks, plan.dst_blocks,
                            plan.src_bt, epoch=t.epoch, stream=sp)
        dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        with torch.cuda.stream(stream):
            e0.record(stream)
            tr.wave(w0.req, w0.lo, w0.hi)
            e1.record(stream)
            ops = [dist.P2POp(dist.isend if k == "send" else dist.irecv,
                              bufs[j][off:off + alloc0 * bb], peer) for k, j, off, peer in ops_spec]
            for r in dist.batch_isend_irecv(ops) if ops else []:
                r.wait()
            e2.record(stream)
        torch.cuda.synchronize(dev)
        tr.close()
        if rep:
            res.append((e0.elapsed_time(e1), e1.elapsed_time(e2), e0.elapsed_time(e2)))
    med = [statistics.median(x[i] for x in res) for i in range(3)]
    tm = torch.tensor(med, dtype=torch.float64, device=dev)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    for p in pools:
        p.close()
    del bufs
    return [float(x) for x in tm.tolist()]


# -------------------------------------------------------------- CPU baseline
def mem_available() -> int:
    """MemAvailable of this host in bytes (0 when unknown)."""
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def cpu_run(plan: Plan, steps, warmup: int, threads: int, target_bytes=None, seconds: float = 8.0):
    """The oracle executor (oracle/kvx_oracle.c, pthreads) over the SAME
    transition: every live request of the plan (target_bytes=None) -- the
    full wave plan, every byte the GPU arm moves -- or, when the host lacks
    the memory for source + destination pools (or target_bytes is given), the
    first requests whose KV totals ~target_bytes.  steps=None: as many steps
    as fill ~`seconds` of CPU work (at least 2), sized from the warm-up step.
    Returns (GB/s, sample description, bytes per step, full plan?)."""
    from oracle import pyoracle as O
    per_req = plan.tokens * plan.kv_bytes_per_token
    order = plan.live
    g = O.geo(plan.L, plan.H, plan.D)
    bb = 2 * 16 * plan.token_bytes
    full = target_bytes is None
    why = "sample"
    if full:
        need = (plan.old_blocks + plan.dst_blocks) * plan.L * bb
        avail = mem_available()
        if avail and need > 0.8 * avail:
            full, target_bytes = False, 0.3 * avail * plan.step_bytes / need
            why = "host memory bound"
    if full:
        sel = np.sort(order)
    else:
        csum = np.cumsum(per_req[order])
        nsel = int(np.searchsorted(csum, target_bytes) + 1)
        sel = np.sort(order[:max(1, nsel)])
    tokens = np.zeros_like(plan.tokens)
    tokens[sel] = plan.tokens[sel]
    if full:
        src_bt, old_blocks = plan.src_bt, plan.old_blocks
    else:
        src_bt, old_blocks = W.fragmented_block_table(tokens, plan.max_blocks, 16, seed=7)
    dst_blocks = int(((tokens + 15) // 16).sum())
    t = plan.t
    waves = []
    for w in t.waves:
        m = np.isin(w.req, sel)
        waves.append((w.req[m], w.lo[m], w.hi[m]))
    step_bytes = sum(int((hi - lo).clip(min=0).sum()) for _, lo, hi in waves) * plan.kv_bytes_per_token
    dp = O.DataPlane(g, t.old_boundaries, t.new_boundaries, old_blocks, dst_blocks, plan.N,
                     plan.max_blocks, src_bt)
    for p in dp.old_pools:  # touch every page (a real KV cache is resident)
        p.fill(0x5A)
    for p in dp.new_pools:
        p[:] = 0
    live_m = np.isin(t.live_req, sel)

    def one_step():
        dp.bt[:] = -1
        dp.synced_hi[:] = 0
        dp.d.next_block = 0
        t0 = time.perf_counter()
        for req, lo, hi in waves:
            assert dp.wave(req, lo, hi, threads=threads) == 0
        dp.commit(t.live_req[live_m], t.live_kv[live_m])
        return time.perf_counter() - t0

    warm = [one_step() for _ in range(max(1, warmup))]
    if steps is None:
        steps = int(min(500, max(2, round(seconds / max(1e-6, min(warm))))))
    times = [one_step() for _ in range(steps)]
    gbs = step_bytes * len(times) / sum(times) / 1e9
    what = (f"the full wave plan of {plan.golden} (all {len(sel)} live requests)" if full else
            f"{len(sel)} of {len(plan.live)} live requests of {plan.golden} ({why})")
    desc = (f"{what}: {step_bytes / 1e9:.2f} GB of KV per step, real geometry, same wave plan and block "
            f"tables, oracle run-granular memcpy on {threads} threads, {len(times)} steps")
    del dp
    return gbs, desc, step_bytes, full


def reference_control_plane(golden: str):
    """The reference's OWN transition handlers (oracle/_ref/extract_waves, the
    unmodified reference library) timed on this host for the same scenario:
    refactor_begin / kv_sync_complete / refactor_commit wall us (median).  The
    reference moves no bytes, so this is its whole CPU path for the
    transition; None when the prebuilt binary is absent."""
    import subprocess
    exe = os.path.join(ROOT, "oracle", "_ref", "extract_waves")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe, "--time", golden, "5"], capture_output=True, text=True, timeout=120)
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as e:  # report, never fail the bench on it
        return {"error": str(e)}


def bench_config(plan: Plan, args, n_gpus: int):
    """The `config` object of the JSON line, shared by both arms (the
    reference arm reports the same workload keys)."""
    t, L = plan.t, plan.L
    old_dev, new_dev = S.placement(L, t.old_boundaries, t.new_boundaries, n_gpus, args.placement)
    move = "pull" if args.pull else args.move
    layer_pull = S.move_plan(L, t.old_boundaries, t.new_boundaries, old_dev, new_dev, move)
    return {"workload": plan.desc, "golden_wave_plan": plan.golden,
            "bytes_per_step": plan.step_bytes, "tokens_per_step": plan.step_tokens,
            "placement": {"mode": args.placement, "old_stage_gpu": old_dev, "new_stage_gpu": new_dev},
            "kv_layouts": args.layouts,
            "movers": {"policy": move, "pulled_layers": int(sum(layer_pull)),
                       "cross_gpu_layers": sum(1 for l in range(L) if old_dev[S.stage_of(t.old_boundaries, l)]
                                               != new_dev[S.stage_of(t.new_boundaries, l)])},
            "l2": "inputs (17 GB) larger than L2 (126 MB); no flush needed"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    plan = Plan(args.config)
    threads, model = host_cpu()
    steps = args.steps
    gbs, desc, step_bytes, full = cpu_run(plan, steps, max(1, args.warmup), threads,
                                          target_bytes=args.sample_gb * 1e9 if args.sample_gb else None)
    ms = step_bytes / (gbs * 1e9) * 1e3
    n_gpus = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s",
        "n_gpus": n_gpus, "steps": steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp16 (u16 words)",
        "data": "synthetic", "config": bench_config(plan, args, n_gpus),
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "cpu_model": model,
                         "kind": "port", "sample": desc, "full_plan": full,
                         "reference_control_plane": reference_control_plane(plan.golden)},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference (pipesim) is a simulator that moves no bytes; its CPU path for this "
                "metric is the oracle restatement executing the identical byte plan on all host threads",
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------- repeated refactors (C5)
def run_chain(args):
    """BASELINE config 5: the reference's bursty, mixed-length trace
    (tests/golden/bursty_repeated.jsonl: gamma arrivals CV=4) drives two
    consecutive inflight refactors, 8->4 then 4->8, at the Llama-2-13B shape.
    The second reads the first one's destination pools through its block
    table; destination blocks come from device block managers; the serving
    pipeline's decode appends between the two are emulated (untimed).  One
    step = both transitions; value = their reference-accounted KV bytes / the
    transitions' device time."""
    import torch
    from paper_2510_11938_b200 import kvx
    dev = 0
    torch.cuda.set_device(dev)
    scn = W.load_golden("bursty_repeated")
    t1, t2 = [t for t in scn.transitions if t.outcome == "commit"][:2]
    N = scn.num_requests
    L, H, D = W.SHAPES["llama2-13b"]
    g = kvx.geometry(L, H, D)
    tok1, tok2 = t1.max_tokens(N), t2.max_tokens(N)
    max_blocks = int((max(tok1.max(), tok2.max()) + 15) // 16)
    need2 = int(((tok2 + 15) // 16).sum())
    src_bt1, capA = W.fragmented_block_table(tok1, max_blocks, 16, seed=7)
    capA = max(capA, need2 + 16)
    capB = int(((np.maximum(tok1, tok2) + 15) // 16).sum()) + 16
    live1 = np.nonzero(tok1)[0].astype(np.int32)
    poolsA = [kvx.Pool(dev, g, e - b, capA) for b, e in W.stage_ranges(L, t1.old_boundaries)]
    poolsB = [kvx.Pool(dev, g, e - b, capB) for b, e in W.stage_ranges(L, t1.new_boundaries)]
    bmA, bmB = kvx.BlockManager(dev, capA), kvx.BlockManager(dev, capB)
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream
    bytes1 = sum(int((w.hi - w.lo).clip(min=0).sum()) for w in t1.waves) * scn.kv_bytes_per_token
    bytes2 = sum(int((w.hi - w.lo).clip(min=0).sum()) for w in t2.waves) * scn.kv_bytes_per_token
    times, stalls, bad = [], [], 0
    for s in range(args.warmup + args.steps):
        for k, (b, e) in enumerate(W.stage_ranges(L, t1.old_boundaries)):
            poolsA[k].fill_pattern(SEED, b, live1, tok1[live1], src_bt1)
        bmA.reset()
        bmB.reset()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        st1 = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), stream)
        st2 = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), stream)
        tr1 = kvx.Transition(g, t1.old_boundaries, poolsA, t1.new_boundaries, poolsB, dev, N, max_blocks, capB,
                             src_bt1, epoch=t1.epoch, max_sync_rounds=scn.max_sync_rounds,
                             kv_bytes_per_token=scn.kv_bytes_per_token, stream=sp, dst_blockmgr=bmB)
        torch.cuda.synchronize(dev)
        ev[0].record(stream)
        run_step(tr1, t1, st1)
        ev[1].record(stream)
        torch.cuda.synchronize(dev)
        table = tr1.dst_block_table()
        tr1.close()
        # serving between the refactors: decode appends into the 4-stage pools
        grown = W.serving_append(bmB.pop, table, t1.live_kv_map(N), tok2)
        if len(grown):
            for k, (b, e) in enumerate(W.stage_ranges(L, t1.new_boundaries)):
                poolsB[k].fill_pattern(SEED, b, grown, tok2[grown], table)
        tr2 = kvx.Transition(g, t2.old_boundaries, poolsB, t2.new_boundaries, poolsA, dev, N, max_blocks, capA,
                             table, epoch=t2.epoch, max_sync_rounds=scn.max_sync_rounds,
                             kv_bytes_per_token=scn.kv_bytes_per_token, stream=sp, dst_blockmgr=bmA)
        torch.cuda.synchronize(dev)
        ev[2].record(stream)
        run_step(tr2, t2, st2)
        ev[3].record(stream)
        torch.cuda.synchronize(dev)
        if s == args.warmup + args.steps - 1:
            bad = tr2.verify_pattern(SEED, t2.live_req, t2.live_kv)
        tr2.close()
        if s >= args.warmup:
            times.append((ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])))
            stalls.append((st1[0].elapsed_time(st1[1]), st2[0].elapsed_time(st2[1])))
    if bad:
        raise SystemExit(f"bench c5: final KV differs from the payload ({bad} words)")
    ms1 = statistics.median(x[0] for x in times)
    ms2 = statistics.median(x[1] for x in times)
    value = (bytes1 + bytes2) / ((ms1 + ms2) * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms1 + ms2, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp16 (u16 words)", "data": "synthetic",
        "config": {"workload": "BASELINE C5: bursty gamma trace (CV=4), mixed lengths, repeated inflight "
                               "refactors 8->4->8 at the Llama-2-13B shape, chained through device block "
                               "managers", "golden_wave_plan": "bursty_repeated",
                   "transitions": [{"stages": f"{t1.old_stages}->{t1.new_stages}", "bytes": bytes1,
                                    "ms": round(ms1, 4), "stall_ms": round(statistics.median(x[0] for x in stalls), 4)},
                                   {"stages": f"{t2.old_stages}->{t2.new_stages}", "bytes": bytes2,
                                    "ms": round(ms2, 4), "stall_ms": round(statistics.median(x[1] for x in stalls), 4)}]},
        "verified_words_mismatched": int(bad),
    }
    print(json.dumps(line), flush=True)
    for p in poolsA + poolsB:
        p.close()
    bmA.close()
    bmB.close()
    return 0


# ------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="kvx", choices=["kvx", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS) + ["c5"])
    ap.add_argument("--placement", default="affinity", choices=["affinity", "disjoint", "spread", "oneway"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--no-weights", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--move", default="auto", choices=["auto", "push", "pull"],
                    help="who moves a cross-GPU layer: auto = pull on one-way traffic, push on two-way "
                         "(shard.move_plan); push = the source GPU; pull = the destination GPU")
    ap.add_argument("--pull", action="store_true", help="alias of --move pull")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--sample-gb", type=float, default=None,
                    help="KV GB per step of the CPU runs (--impl reference, cpu_baseline); default: the "
                         "full wave plan (falls back to a sample only when host memory is short)")
    ap.add_argument("--no-ncu", action="store_true", help="skip the in-run ncu traffic pass")
    ap.add_argument("--no-nvlink-probe", action="store_true", help="N>1: skip the disjoint-grant NVLink wave")
    ap.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--probe-all-waves", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--probe-world", type=int, default=1, help=argparse.SUPPRESS)
    ap.add_argument("--layouts", default="blocks,blocks",
                    help="old,new pool layouts: blocks (FlashInfer NHD [blocks][2][B][H][D]), planes "
                         "(FlashAttention [2][blocks][B][H][D]) or heads (FlashInfer HND [blocks][2][H][B][D], "
                         "vLLM's FlashInfer layout on B200); unequal = the refactor converts")
    args = ap.parse_args()
    if args.traffic_probe:
        return traffic_probe(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c5":
        return run_chain(args)
    if args.warmup < 3:
        args.warmup = 3

    import torch
    import torch.distributed as dist
    from paper_2510_11938_b200 import kvx

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n_gpus = world
    # KVX_BENCH_FOLD=n (functional testing only): fold the ranks onto n
    # physical GPUs, e.g. the N=8 placement on a 4-GPU box.  NCCL refuses two
    # ranks on one GPU, so the host plumbing goes over gloo, the NCCL baseline
    # is skipped and the line is marked as not a measurement.
    fold = int(os.environ.get("KVX_BENCH_FOLD", "0"))
    dev = (local % fold if fold else local) if world > 1 else 0
    if fold:
        args.no_nccl = True
    if world > 1:
        torch.cuda.set_device(dev)
        if fold:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)

    plan = Plan(args.config)
    t = plan.t
    L = plan.L
    layouts = [{"blocks": kvx.LAYOUT_BLOCKS, "planes": kvx.LAYOUT_KV_PLANES, "heads": kvx.LAYOUT_HEADS}[x]
               for x in args.layouts.split(",")]
    g = kvx.geometry(L, plan.H, plan.D)
    old_dev, new_dev = S.placement(L, t.old_boundaries, t.new_boundaries, n_gpus, args.placement)
    if args.pull:
        args.move = "pull"
    layer_pull = S.move_plan(L, t.old_boundaries, t.new_boundaries, old_dev, new_dev, args.move)

    # ---- pools on this GPU; new-stage pools of peers mapped through CUDA IPC
    def gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    old_pools, new_pools = S.setup_rank_pools(
        kvx, g, t.old_boundaries, t.new_boundaries, old_dev, new_dev, rank, dev, plan.old_blocks,
        plan.dst_blocks, all_gather=gather if world > 1 else None,
        fill=(SEED, plan.live, plan.tokens[plan.live], plan.src_bt), layer_pull=layer_pull,
        old_layout=layouts[0], new_layout=layouts[1])
    if world > 1:
        dist.barrier()

    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream

    def make():
        return kvx.Transition(g, t.old_boundaries, old_pools, t.new_boundaries, new_pools, dev,
                              plan.N, plan.max_blocks, plan.dst_blocks, plan.src_bt, epoch=t.epoch,
                              max_sync_rounds=plan.scn.max_sync_rounds,
                              kv_bytes_per_token=plan.kv_bytes_per_token, stream=sp, layer_pull=layer_pull)

    K, Wm = args.steps, args.warmup
    trs = [make() for _ in range(Wm + K)]

    # ---- warm-up
    for s in range(Wm):
        run_step(trs[s], t)
    torch.cuda.synchronize(dev)

    # ---- correctness gate on the warm-up output (device-side payload check);
    #      peers push into our pools, so every rank must be done first
    if world > 1:
        dist.barrier()
    bad = 0
    if not args.no_verify:
        bad = trs[Wm - 1].verify_pattern(SEED, t.live_req, t.live_kv)
    if world > 1:
        tb = torch.tensor([bad], dtype=torch.int64, device=dev)
        dist.all_reduce(tb)
        bad = int(tb.item())
    if bad:
        raise SystemExit(f"bench: destination KV differs from the source payload ({bad} words)")

    # ---- timed region (device-resident KV): K steps
    sampler = ClockSampler(dev)
    sampler.start()
    time.sleep(0.3)
    stall_pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), stream)
                   for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches0 = kvx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    ev0.record(stream)
    for s in range(K):
        # commit without a host sync: the next transition's waves queue right
        # behind it; every result is collected (and checked) after the loop
        run_step(trs[Wm + s], t, stall_pairs[s], wait=False)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    wall1 = time.time()
    launches = kvx.launch_count() - launches0
    for s in range(K):
        res = trs[Wm + s].collect_commit()
        if res.violations != t.violations:
            raise SystemExit(f"bench: step {s} commit reported {res.violations} Eq. 10 violations")
    if world > 1:
        dist.barrier()
    sampler.stop()
    dev_ms = ev0.elapsed_time(ev1)
    stalls = sorted(a.elapsed_time(b) for a, b, _ in stall_pairs)
    stall_med = statistics.median(stalls)
    # dominant kernel: wave-0 move of each timed step
    mv = [trs[Wm + s].move_timings() for s in range(K)]
    w0_ms = [m[0][0] for m in mv if m]
    w0_bytes = mv[0][0][1] if mv and mv[0] else 0
    w0_avg = sum(w0_ms) / len(w0_ms) if w0_ms else float("nan")
    all_move_ms = sum(x[0] for m in mv for x in m)
    n_waves = max((len(m) for m in mv), default=0)
    wave_ms = [round(statistics.median(m[i][0] for m in mv if len(m) > i), 4) for i in range(n_waves)]

    # a rank that launches no mover of its own (N=8 C3: the old-stage GPUs whose
    # layers their receivers pull) reports 0 here and null in rank_wave0_move_ms
    w0_red = w0_avg if w0_ms else 0.0
    tm = torch.tensor([dev_ms, stall_med, float(launches), w0_red, float(w0_bytes)], dtype=torch.float64,
                      device=dev)
    rank_ms = [round(dev_ms / K, 4)]
    rank_w0 = [round(w0_avg, 4) if w0_ms else None]
    if world > 1:
        allv = [torch.zeros(2, dtype=torch.float64, device=dev) for _ in range(world)]
        dist.all_gather(allv, torch.tensor([dev_ms / K, w0_red], dtype=torch.float64, device=dev))
        rank_ms = [round(float(v[0]), 4) for v in allv]
        rank_w0 = [round(float(v[1]), 4) if float(v[1]) > 0 else None for v in allv]
        mx = tm.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = tm.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        dev_ms, stall_med, w0_avg = float(mx[0]), float(mx[1]), float(mx[3])
        launches = int(sm[2])
        w0_bytes_total = int(sm[4])
    else:
        w0_bytes_total = w0_bytes
    for tr in trs:
        tr.close()

    # ---- e2e through the public API (host inputs, results back to host)
    e2e_steps = args.e2e_steps or K
    h2d = d2h = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = time.perf_counter()
    prev = None
    for s in range(e2e_steps + 1):
        # step s is granted and issued (commit async) before step s-1's commit
        # result is collected on the host, as an engine that resumes routing at
        # the commit would (engine.cpp:747-756): the D2H read of every step's
        # result stays inside the timed region, off the device's critical path
        tr = None
        if s < e2e_steps:
            tr = make()  # grant: device state + source block table H2D
            run_step(tr, t, wait=False)
        if prev is not None:
            res = prev.collect_commit()
            if res.violations != t.violations:
                raise SystemExit(f"bench e2e: commit reported {res.violations} Eq. 10 violations")
            prev.close()
            if s == 1:
                n_entries = sum(len(w.req) for w in t.waves)
                h2d = plan.src_bt.nbytes + n_entries * (4 + 8 + 8) + len(t.live_req) * (4 + 8)
                d2h = 3 * 8 + res.row_ptr.nbytes + res.blocks.nbytes + res.free_list.nbytes
        prev = tr
    torch.cuda.synchronize(dev)
    e2e_s = time.perf_counter() - e0
    if world > 1:
        te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())

    # ---- drain-free stall: at the reference's barrier the
    #      in-flight micro-batches are handed to their new owners (hidden x
    #      fp16 rows) instead of drained, the final wave goes out at once over
    #      the barrier's live set, then commit.  Device time barrier -> commit.
    handoff = None
    bar = next((e for e in t.events if isinstance(e, W.Barrier) and e.microbatches), None)
    if bar is not None:
        row = {"llama2-13b": 5120, "llama2-7b": 4096, "llama2-70b": 8192}[CONFIGS[args.config][1]] * 2
        srcs = [torch.full((max(m.tokens, 1) * row,), m.batch % 251, dtype=torch.uint8, device=dev)
                for m in bar.microbatches]
        cap = sum(m.tokens * row + 256 for m in bar.microbatches) + 256
        arenas = [torch.zeros(cap, dtype=torch.uint8, device=dev) for _ in range(len(t.new_boundaries) + 1)]
        htimes, stimes = [], []
        for rep in range(6):
            tr = make()
            tr.set_handoff(True)
            wave0 = t.waves[0]
            tr.begin_refactor((wave0.req, wave0.hi))
            for e in t.events[1:]:  # delta waves before the barrier, as the reference ran them
                if isinstance(e, W.Barrier):
                    break
                tr.on_kv_sync_complete((e.req, e.hi), 1)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            a0, a1, a2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a0.record(stream)
            act, _ = tr.on_kv_sync_complete((bar.req, bar.kv), bar.inflight_batches)
            assert act == kvx.ACT_FINAL, act
            slots = tr.handoff(row, [(m.batch, m.after, m.tokens, s_.data_ptr())
                                     for m, s_ in zip(bar.microbatches, srcs)],
                               [x.data_ptr() for x in arenas], [cap] * len(arenas))
            a1.record(stream)
            res = tr.on_refactor_commit((bar.req, bar.kv))
            a2.record(stream)
            torch.cuda.synchronize(dev)
            assert res.violations == 0
            if rep > 0:
                htimes.append(a0.elapsed_time(a1))
                stimes.append(a0.elapsed_time(a2))
            tr.close()
        hbytes = sum(sl[4] for sl in slots)
        hms, sms = statistics.median(htimes), statistics.median(stimes)
        if world > 1:
            tt = torch.tensor([hms, sms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            hms, sms = [float(x) for x in tt.tolist()]
        handoff = {"batches": len(bar.microbatches), "bytes": int(hbytes),
                   "final_wave_plus_handoff_ms": round(hms, 4), "stall_handoff_ms": round(sms, 4),
                   "note": "drain-free mode: in-flight micro-batches of the reference's barrier moved "
                           "to their new owners (hidden x fp16 rows), final wave over the barrier's "
                           "live set, commit; device time barrier -> commit result on host"}

    # ---- the stall as the reference defines it (engine.cpp:676-686):
    #      host-observed (handler call -> commit result on the host) and under
    #      the reference's conditions (weights loading beside wave 0, commit at
    #      max(final wave, weights ready), drain vs handoff)
    h_med, h_lo, h_hi = host_observed_stall(make, t)
    if world > 1:
        th = torch.tensor([h_med, h_hi], dtype=torch.float64, device=dev)
        dist.all_reduce(th, op=dist.ReduceOp.MAX)
        h_med, h_hi = [float(x) for x in th.tolist()]
    # ---- the device stall with a decode step between wave 0 and the barrier
    #      (the reference's timeline; see serving_stall)
    sv = serving_stall(make, t, old_pools, W.stage_ranges(L, t.old_boundaries), plan.src_bt, stream, dev)
    if sv is not None and world > 1:
        ts = torch.tensor(list(sv), dtype=torch.float64, device=dev)
        dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        sv = tuple(float(x) for x in ts.tolist())
    ref_cond = None
    if world == 1 and not args.no_weights:
        ref_cond = reference_condition_stall(make, t, plan, CONFIGS[args.config][1], stream, dev)

    # ---- stage weight migration: the new stages' parameters
    #      gathered by layer range on the device (N=1; fp16 weights of the shape)
    weights = None
    if world == 1 and not args.no_weights:
        params = {"llama2-13b": 26.0e9, "llama2-7b": 13.5e9, "llama2-70b": 138.0e9}[CONFIGS[args.config][1]]
        lb = int(params / L) // 4096 * 4096
        if lb * L * 2 < 120e9:
            wold = [torch.empty((e - b) * lb, dtype=torch.uint8, device=dev)
                    for b, e in W.stage_ranges(L, t.old_boundaries)]
            wnew = [torch.empty((e - b) * lb, dtype=torch.uint8, device=dev)
                    for b, e in W.stage_ranges(L, t.new_boundaries)]
            wt = []
            for rep in range(4):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                kvx.weights_migrate(dev, L, lb, t.old_boundaries, [x.data_ptr() for x in wold],
                                    t.new_boundaries, [x.data_ptr() for x in wnew], stream=sp)
                b.record(stream)
                torch.cuda.synchronize(dev)
                if rep:
                    wt.append(a.elapsed_time(b))
            wms = statistics.median(wt)
            wbytes = lb * L
            weights = {"bytes": wbytes, "ms": round(wms, 3), "GB_s": round(wbytes / (wms * 1e-3) / 1e9, 1),
                       "hbm_frac": round(2 * wbytes / (wms * 1e-3) / 1e9 / peaks()[0], 4),
                       "reference_load_ms": plan.t.load_ready_ms - plan.t.t_ms,
                       "note": "device-to-device layer-range gather of the new stages' weights; the "
                               "reference models this as host/storage loads (load_ready_ms)"}
            del wold, wnew

    # ---- NVLink under the reference's disjoint grant (N > 1)
    nvl = None
    # (folded ranks share GPUs, so the probe is no measurement there; KVX_BENCH_FOLD_PROBE=1
    # runs it anyway as a functional check of the N=8 path on a 4-GPU box)
    if world > 1 and (not fold or os.environ.get("KVX_BENCH_FOLD_PROBE") == "1") and not args.no_nvlink_probe:
        nvl = nvlink_probe(kvx, torch, dist, plan, g, rank, world, dev, gather)

    # ---- NCCL baseline of the cross-GPU path (N > 1, when bytes cross GPUs)
    nccl = None
    if world > 1 and not args.no_nccl:
        nb_ms = nccl_baseline(kvx, torch, dist, plan, g, old_pools, old_dev, new_dev, rank, world, dev,
                              stream)
        if nb_ms is not None:
            nccl = {"gather_ms": round(nb_ms[0], 4), "nccl_ms": round(nb_ms[1], 4),
                    "total_ms": round(nb_ms[2], 4), "fused_p2p_ms": round(w0_avg, 4),
                    "fused_speedup": round(nb_ms[2] / w0_avg, 3),
                    "note": "wave 0: local gather into a copy of the destination layout + grouped "
                            "NCCL send/recv of each remote layer region, vs the fused gather+push "
                            "kernel over NVLink P2P (max over ranks)"}

    # ---- the roofline denominator re-measured live on this GPU: the same
    #      torch copy MEASURED_PEAKS.json uses (b.copy_(a), 1 Gi bf16, read+write)
    copy_ref = None
    if world == 1:
        a_t = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
        b_t = torch.empty_like(a_t)
        best = float("inf")
        for _ in range(10):
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record()
            b_t.copy_(a_t)
            c1.record()
            torch.cuda.synchronize(dev)
            best = min(best, c0.elapsed_time(c1))
        copy_ref = {"torch_copy_GBps": round(2 * a_t.numel() * 2 / (best * 1e-3) / 1e9, 1),
                    "note": "b.copy_(a) over 1 Gi bf16 (read+write), best of 10, this run"}
        del a_t, b_t

    # ---- roofline of the dominant kernel
    peak, peak_kind = peaks()
    layer_bytes = plan.wave0_tokens * 2 * plan.token_bytes  # K+V bytes per layer in wave 0
    hbm, out, inn = S.link_bytes(L, t.old_boundaries, t.new_boundaries, old_dev, new_dev, layer_bytes,
                               n_gpus)
    nvl_peak = 770.0  # measured peer copy GB/s per direction (B200_PROFILING.md)
    t_roof = max(max(h / (peak * 1e9) for h in hbm), max(o / (nvl_peak * 1e9) for o in out),
                 max(i / (nvl_peak * 1e9) for i in inn))
    if n_gpus == 1:
        achieved = w0_bytes / (w0_avg * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "live_copy_reference": copy_ref,
                "frac": round(achieved / peak, 4), "traffic": None,
                "kernel": "kvx_bulk_kernel<3,64K> (wave 0, TMA bulk mover)", "bytes_per_launch": w0_bytes,
                "launch_ms": round(w0_avg, 4), "peak_source": peak_kind}
    else:
        frac = t_roof * 1e3 / w0_avg
        bound = "nvlink" if max(out + inn) / nvl_peak > max(hbm) / peak else "hbm"
        roof = {"bound": bound, "achieved": round(frac * (peak if bound == "hbm" else nvl_peak), 1),
                "peak": peak if bound == "hbm" else nvl_peak, "unit": "GB/s", "frac": round(frac, 4),
                "traffic": None, "kernel": "kvx_bulk_kernel (wave 0, slowest rank)",
                "algorithmic_bytes_per_gpu": {"hbm_rw": [int(x) for x in hbm], "nvlink_out": [int(x) for x in out],
                                              "nvlink_in": [int(x) for x in inn]},
                "traffic_note": "N>1: rank 0's wave-0 mover under ncu in this run when rank 0 moves no layer "
                                "over NVLink (vs its own hbm_rw); NVLink bytes from ncu: scripts/nvlink_ncu.sh, "
                                "profiles/r02j/",
                "t_roof_ms": round(t_roof * 1e3, 4), "launch_ms": round(w0_avg, 4),
                "peak_source": f"hbm {peak_kind}; nvlink 770 GB/s measured peer copy"}

    # ordered teardown: unmap peers' pools, then free our own
    for p in old_pools + new_pools:
        if p is not None and p.imported:
            p.close()
    if world > 1:
        dist.barrier()
    for p in old_pools + new_pools:
        if p is not None and not p.imported:
            p.close()
    if world > 1:
        dist.barrier()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- DRAM traffic of the dominant launch, from an ncu pass of THIS run
    #      (pools above are freed; the child rebuilds them and issues wave 0)
    if n_gpus == 1 and not args.no_ncu:
        roof["traffic"], roof["traffic_source"] = ncu_traffic(args.config)
        if roof["traffic"]:
            roof["traffic_over_algorithmic"] = round(roof["traffic"] / w0_bytes, 4)
    elif not args.no_ncu and not fold and out[0] == 0 and inn[0] == 0 and dev == 0:
        # rank 0's share is local: the same wave-0 mover over its own layers
        roof["traffic"], roof["traffic_source"] = ncu_traffic(args.config, world=n_gpus, placement=args.placement)
        if roof["traffic"]:
            roof["traffic_rank"] = 0
            roof["traffic_over_algorithmic"] = round(roof["traffic"] / hbm[0], 4)

    value = plan.step_bytes * K / (dev_ms * 1e-3) / 1e9
    e2e_value = plan.step_bytes * e2e_steps / e2e_s / 1e9
    clocks = sampler.summary(wall0, wall1)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": n_gpus, "steps": K,
        "warmup": Wm, "ms_per_step": round(dev_ms / K, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp16 (u16 words)", "data": "synthetic",
        "config": bench_config(plan, args, n_gpus),
        "stall_ms": round(stall_med, 4), "stall_ms_all": [round(x, 4) for x in (stalls[0], stalls[-1])],
        "stall": {"device_ms": round(stall_med, 4),
                  "device_note": "final wave + commit on the device: CUDA events around the barrier handler "
                                 "call that issues the final wave and the commit (timed loop, no host sync)",
                  "host_observed_ms": round(h_med, 4), "host_observed_range_ms": [round(h_lo, 4), round(h_hi, 4)],
                  "host_note": "wall clock from the barrier handler call (after the host saw the earlier waves "
                               "complete) to the commit result on the host (engine.cpp:676-713)",
                  "reference_condition": ref_cond,
                  "device_after_decode_ms": None if sv is None else round(sv[0], 4),
                  "final_wave_after_decode_ms": None if sv is None else round(sv[1], 4),
                  "after_decode_note": "as device_ms, with a decode step between the last pre-barrier wave and "
                                       "the barrier, as in the reference's timeline (the final wave moves what "
                                       "decode appended): the append of the final wave's rows, then 1 GiB of "
                                       "KV-cache reads. device_ms issues the final wave right behind wave 0's "
                                       "17 GB mover and so also pays the write-back of wave 0's dirty L2 lines"},
        "e2e": {"value": round(e2e_value, 2), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                "ms_per_step": round(e2e_s * 1e3 / e2e_steps, 4)},
        "roofline": roof, "gpu_launches": int(launches), "clocks": clocks, "handoff": handoff,
        "weights": weights, "nccl_baseline": nccl, "nvlink_disjoint": nvl,
        "move_kernel_ms_per_step": round(all_move_ms / K, 4), "move_ms_by_wave": wave_ms,
        "rank_ms_per_step": rank_ms, "rank_wave0_move_ms": rank_w0,
        "mover": os.environ.get("KVX_MOVE_IMPL", "bulk") + ":" + os.environ.get("KVX_BULK_CFG", "auto"),
    }
    sim = plan.t.simulated_stall_ms()
    line["stall_reference_simulated_ms"] = round(sim, 3) if sim is not None else None
    if fold:
        line["folded_onto_gpus"] = fold
        line["not_a_measurement"] = "ranks share GPUs (KVX_BENCH_FOLD); functional check of the N-rank path"
    if n_gpus == 1 and not args.no_cpu_baseline:
        threads, model = host_cpu()
        gbs, desc, _, full = cpu_run(plan, None, 1, threads,
                                     target_bytes=args.sample_gb * 1e9 if args.sample_gb else None, seconds=8.0)
        gbs1, desc1, _, _ = cpu_run(plan, None, 1, 1, target_bytes=0.5e9, seconds=3.0)
        line["cpu_baseline"] = {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "cpu_model": model,
                                "kind": "port", "sample": desc, "full_plan": full,
                                "value_1_thread": round(gbs1, 3), "sample_1_thread": desc1,
                                "reference_control_plane": reference_control_plane(plan.golden)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
