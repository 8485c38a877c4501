"""Stage weight migration: the oracle's restatement of the
reference's parameter-load model is pinned to the reference's own numbers,
and the layer routing of the weight gather follows stage_loads."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2510_11938_b200 import workload as W


def begins():
    for name in W.golden_names():
        for t in W.load_golden(name).transitions:
            yield name, t


CASES = list(begins())


@pytest.mark.parametrize("name,t", CASES, ids=[f"{c[0]}-{i}" for i, c in enumerate(CASES)])
def test_warm_start_matches_reference(name, t):
    """warm_start_latency_ms (cluster.cpp:525-536) per server, and
    load_ready_ms = now + max over servers (engine.cpp:621-631), bit-exact."""
    assert t.param_loads
    worst = 0.0
    for srv in t.param_loads:
        stages = srv["stages"]
        ms = O.warm_start_ms([s[2] for s in stages], [s[3] for s in stages], srv["host_bw"],
                             srv["storage_bw"])
        assert ms == srv["latency_ms"]
        worst = max(worst, ms)
    assert t.t_ms + worst == t.load_ready_ms


def test_some_loads_are_host_cached():
    cached = [s[3] for _, t in CASES for srv in t.param_loads for s in srv["stages"]]
    assert any(cached) and not all(cached)


@pytest.mark.parametrize("name,t", CASES[:6], ids=[f"{c[0]}" for c in CASES[:6]])
def test_weight_routing_follows_stage_loads(name, t):
    L = 32 if not name.startswith(("llama13", "bursty", "llama70")) else (80 if "70b" in name else 40)
    ss, so, ds, do = O.weights_plan(L, 1000, t.old_boundaries, t.new_boundaries)
    new_r = W.stage_ranges(L, t.new_boundaries)
    old_r = W.stage_ranges(L, t.old_boundaries)
    for l in range(L):
        assert old_r[ss[l]][0] <= l < old_r[ss[l]][1] and so[l] == (l - old_r[ss[l]][0]) * 1000
        assert new_r[ds[l]][0] <= l < new_r[ds[l]][1] and do[l] == (l - new_r[ds[l]][0]) * 1000
    # new stage k receives exactly its range, contiguous, once
    for k, (b, e) in enumerate(new_r):
        assert sorted(do[ds == k].tolist()) == [i * 1000 for i in range(e - b)]
