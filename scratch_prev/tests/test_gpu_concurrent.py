"""Concurrent transitions (engine.cpp:991-998 refactors every active
instance): three replicas' refactors, each on its own private stream, waves
interleaved from one host thread and from three host threads -- every
replica's destination equals the oracle's."""
import threading

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import kvx
from paper_2510_11938_b200 import workload as W

pytestmark = pytest.mark.gpu


class Replica:
    def __init__(self, seed):
        rng = np.random.default_rng(seed)
        self.seed = seed
        self.L, self.H, self.D = 12, 4, 64
        self.ob, self.nb = [3, 6, 9], [6]
        self.N = 40
        self.final = rng.integers(1, 160, self.N).astype(np.int64)
        self.mid = np.minimum(self.final, rng.integers(0, 120, self.N))
        mb = int((self.final.max() + 15) // 16)
        self.mb = mb
        self.src_bt, cap0 = W.fragmented_block_table(self.final, mb, 16, seed=seed)
        cap1 = int(((self.final + 15) // 16).sum())
        g = kvx.geometry(self.L, self.H, self.D)
        req = np.arange(self.N, dtype=np.int32)
        self.old = []
        for b, e in W.stage_ranges(self.L, self.ob):
            p = kvx.Pool(0, g, e - b, cap0)
            p.zero()
            p.fill_pattern(seed, b, req, self.final, self.src_bt)
            self.old.append(p)
        self.new = []
        for b, e in W.stage_ranges(self.L, self.nb):
            p = kvx.Pool(0, g, e - b, cap1)
            p.zero()
            self.new.append(p)
        self.tr = kvx.Transition(g, self.ob, self.old, self.nb, self.new, 0, self.N, mb, cap1, self.src_bt)
        self.dp = O.DataPlane(O.geo(self.L, self.H, self.D), self.ob, self.nb, cap0, cap1, self.N, mb,
                              self.src_bt)
        self.dp.fill_source(seed, req, self.final)
        self.req = req

    def wave(self, k):
        lo, hi = (np.zeros(self.N, np.int64), self.mid) if k == 0 else (self.mid, self.final)
        self.tr.wave(self.req, lo, hi)
        assert self.dp.wave(self.req, lo, hi) == 0

    def check(self):
        self.tr.wait()
        res = self.tr.commit(self.req, self.final)
        assert res.violations == 0
        np.testing.assert_array_equal(self.tr.dst_block_table(), self.dp.bt)
        for k, p in enumerate(self.new):
            np.testing.assert_array_equal(p.read(), self.dp.new_pools[k])

    def close(self):
        self.tr.close()
        for p in self.old + self.new:
            p.close()


def test_interleaved_replicas_one_thread(gpu_count):
    reps = [Replica(s) for s in (1, 2, 3)]
    try:
        for k in (0, 1):
            for r in reps:
                r.wave(k)
        for r in reps:
            r.check()
    finally:
        for r in reps:
            r.close()


def test_replicas_from_host_threads(gpu_count):
    reps = [Replica(s) for s in (4, 5, 6)]
    errors = []

    def run(r):
        try:
            r.wave(0)
            r.wave(1)
            r.check()
        except Exception as e:  # surfaced below
            errors.append(e)

    try:
        th = [threading.Thread(target=run, args=(r,)) for r in reps]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errors, errors
    finally:
        for r in reps:
            r.close()
