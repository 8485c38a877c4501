"""Synthetic inputs of the inflight-refactor KV transition.

* Model shapes of BASELINE.json's configs (Llama-2 7B / 13B / 70B-GQA).
* Transition specs read from the committed golden wave plans
  (tests/golden/*.jsonl, produced by the UNMODIFIED reference engine through
  oracle/extract_waves.cpp): plans, per-wave (req, lo, hi) intervals, the
  live set at commit, and the reference's own accounting.
* Fragmented source block tables: the serving pipeline's blocks for the
  live requests are a seeded permutation of its pool (the realistic case --
  pages of one request are scattered), so the gather is a real gather.

Nothing here moves bytes; it only builds inputs.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")

# (layers, kv_heads, head_dim) -- kv_bytes_per_token = 2 * L * H * D * 2 B
SHAPES = {
    "llama2-7b": (32, 32, 128),
    "llama2-13b": (40, 40, 128),
    "llama2-70b": (80, 8, 128),
}


@dataclass
class Wave:
    index: int
    final: bool
    rounds: int
    req: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    tokens: int
    kv_synced_bytes_total: float  # reference accumulator after this wave
    t_ms: float = 0.0             # simulated dispatch time of the wave (KvSyncComplete / commit schedule)


@dataclass
class MicroBatchRec:
    """An in-flight micro-batch at the barrier (engine.cpp:449-464)."""
    batch: int
    where: str          # current | inbound | transit
    after: int          # last old stage whose output it holds (-1: none)
    tokens: int         # activation rows: prompt for prefill units, 1 per decode unit
    act_bytes: float    # reference's modelled hop size (scale_activation)


@dataclass
class Barrier:
    """engine.cpp:676: the barrier fell; live set + in-flight batches it saw."""
    rounds: int
    inflight_batches: int
    req: np.ndarray
    kv: np.ndarray
    microbatches: list = field(default_factory=list)
    barrier_ms: float = 0.0


@dataclass
class TransitionSpec:
    """One begin -> waves -> commit|abort sequence of the reference engine."""
    scenario: str
    instance: int
    epoch: int
    old_stages: int
    old_boundaries: List[int]
    new_stages: int
    new_boundaries: List[int]
    new_gpus: List[int]
    t_ms: float = 0.0
    load_ready_ms: float = 0.0
    param_loads: list = field(default_factory=list)  # per server: stages, bws, reference latency
    waves: List[Wave] = field(default_factory=list)
    events: list = field(default_factory=list)  # Wave | Barrier, in engine order
    outcome: str = "open"              # commit | abort
    live_req: Optional[np.ndarray] = None
    live_kv: Optional[np.ndarray] = None
    violations: Optional[int] = None
    kv_synced_bytes_total: Optional[float] = None
    commit_ms: Optional[float] = None

    def simulated_stall_ms(self) -> Optional[float]:
        """The reference's own stall for this transition: barrier -> commit in
        simulated time (engine.cpp:676 -> 686), drain and load waits included."""
        bars = [e for e in self.events if isinstance(e, Barrier)]
        if not bars or self.commit_ms is None:
            return None
        return self.commit_ms - bars[0].barrier_ms

    def live_kv_map(self, max_requests: int) -> np.ndarray:
        """kv_tokens at commit per request id (0 for requests not live)."""
        t = np.zeros(max_requests, np.int64)
        if self.live_req is not None:
            t[self.live_req] = self.live_kv
        return t

    def max_tokens(self, max_requests: int) -> np.ndarray:
        """Per-request token count the source must hold (max over waves/commit)."""
        t = np.zeros(max_requests, np.int64)
        for w in self.waves:
            np.maximum.at(t, w.req, w.hi)
        if self.live_req is not None:
            np.maximum.at(t, self.live_req, self.live_kv)
        return t


@dataclass
class Scenario:
    name: str
    note: str
    num_layers: int
    kv_bytes_per_token: float
    max_sync_rounds: int
    num_requests: int
    transitions: List[TransitionSpec]
    result: Dict
    # global order of (transition index, event) across instances, as the
    # reference dispatched them: ("wave", Wave) | ("barrier", Barrier) |
    # ("commit" | "abort", None)
    timeline: list = field(default_factory=list)


def load_golden(name: str, golden_dir: str = GOLDEN_DIR) -> Scenario:
    path = os.path.join(golden_dir, name + ".jsonl")
    with open(path) as f:
        rows = [json.loads(l) for l in f]
    head = rows[0]
    assert head["kind"] == "scenario"
    trans: List[TransitionSpec] = []
    cur: Dict[int, TransitionSpec] = {}
    idx: Dict[int, int] = {}
    timeline = []
    result = {}
    for r in rows[1:]:
        k = r["kind"]
        if k == "begin":
            t = TransitionSpec(head["name"], r["instance"], r["epoch"], r["old"]["stages"],
                               list(r["old"]["boundaries"]), r["new"]["stages"],
                               list(r["new"]["boundaries"]), list(r["new_gpus"]),
                               r.get("begin_ms", r["t_ms"]),
                               r["load_ready_ms"], r.get("param_loads", []))
            cur[r["instance"]] = t
            idx[r["instance"]] = len(trans)
            trans.append(t)
        elif k == "wave":
            e = np.array(r["entries"], dtype=np.int64).reshape(-1, 3)
            w = Wave(r["wave"], r["final"], r["rounds"], e[:, 0].astype(np.int32), e[:, 1].copy(),
                     e[:, 2].copy(), r["tokens"], r["kv_synced_bytes_total"], r.get("t_ms", 0.0))
            cur[r["instance"]].waves.append(w)
            cur[r["instance"]].events.append(w)
            timeline.append((idx[r["instance"]], "wave", w))
        elif k == "barrier":
            e = np.array(r["live"], dtype=np.int64).reshape(-1, 2)
            mbs = [MicroBatchRec(m["batch"], m["where"], m["after"], int(sum(u[2] for u in m["units"])),
                                 m["act_bytes"]) for m in r.get("microbatches", [])]
            b = Barrier(r["rounds"], r["inflight_batches"], e[:, 0].astype(np.int32), e[:, 1].copy(), mbs,
                        r.get("barrier_ms", r["t_ms"]))
            cur[r["instance"]].events.append(b)
            timeline.append((idx[r["instance"]], "barrier", b))
        elif k == "commit_state":
            e = np.array(r["live"], dtype=np.int64).reshape(-1, 2)
            t = cur[r["instance"]]
            t.live_req, t.live_kv = e[:, 0].astype(np.int32), e[:, 1].copy()
            t.commit_ms = r["t_ms"]  # RefactorCommit dispatch time
        elif k in ("commit", "abort", "end_unknown"):
            timeline.append((idx[r["instance"]], k, None))
            t = cur.pop(r["instance"])
            t.outcome = k
            t.violations = r.get("violations")
            t.kv_synced_bytes_total = r["kv_synced_bytes_total"]
        elif k == "result":
            result = r
    return Scenario(head["name"], head["note"], head["num_layers"], head["kv_bytes_per_token"],
                    head["max_sync_rounds"], head["num_requests"], trans, result, timeline)


def golden_names(golden_dir: str = GOLDEN_DIR) -> List[str]:
    return sorted(f[:-6] for f in os.listdir(golden_dir) if f.endswith(".jsonl"))


def shape_for(scn: Scenario) -> Tuple[int, int, int]:
    """Geometry whose kv_bytes_per_token equals the scenario's, when one of
    the BASELINE shapes does; else a small stand-in (the engine_* fixtures use
    1e5 B/token, which no integral geometry reproduces -- the control-plane
    accounting still uses the fixture's own figure)."""
    for L, H, D in SHAPES.values():
        if L == scn.num_layers and 2 * L * H * D * 2 == scn.kv_bytes_per_token:
            return L, H, D
    return scn.num_layers, 2, 64


def fragmented_block_table(tokens: np.ndarray, max_blocks: int, block_tokens: int,
                           pool_blocks: Optional[int] = None, seed: int = 0,
                           slack: float = 0.25) -> Tuple[np.ndarray, int]:
    """Per-request source block table [max_requests, max_blocks] whose ids are
    a seeded permutation of the pool (fragmented pages); -1 = none."""
    nblk = (tokens + block_tokens - 1) // block_tokens
    need = int(nblk.sum())
    if pool_blocks is None:
        pool_blocks = max(1, int(need * (1.0 + slack)) + 1)
    if need > pool_blocks:
        raise ValueError("source pool too small")
    perm = np.random.default_rng(seed).permutation(pool_blocks).astype(np.int32)
    bt = np.full((len(tokens), max_blocks), -1, np.int32)
    k = 0
    for r in np.nonzero(nblk)[0]:
        n = int(nblk[r])
        bt[r, :n] = perm[k:k + n]
        k += n
    return bt, pool_blocks


def stage_ranges(num_layers: int, boundaries) -> List[Tuple[int, int]]:
    cuts = [0, *boundaries, num_layers]
    return [(cuts[k], cuts[k + 1]) for k in range(len(cuts) - 1)]


def synthetic_lengths(n: int, lo: int, hi: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).integers(lo, hi + 1, size=n).astype(np.int64)


def serving_append(pop, table: np.ndarray, have: np.ndarray, want: np.ndarray,
                   block_tokens: int = 16) -> np.ndarray:
    """Emulates the serving pipeline's decode appends between two refactors:
    every request growing from have[r] to want[r] tokens gets the extra
    logical blocks popped from its pool set's block manager (`pop(n) -> ids`)
    and written into `table` (in place).  Returns the grown request ids."""
    grown = []
    for r in np.nonzero(want > have)[0]:
        b0 = int((have[r] + block_tokens - 1) // block_tokens)
        b1 = int((want[r] + block_tokens - 1) // block_tokens)
        if b1 > b0:
            table[r, b0:b1] = pop(b1 - b0)
        grown.append(int(r))
    return np.array(grown, np.int32)
