"""Shared set-up for the -m gpu parity tests: one golden transition on the
GPU (through the kvx C-ABI) and, optionally, on the CPU oracle with the same
geometry, source block table and payload."""
import numpy as np

from oracle import pyoracle as O
from paper_2510_11938_b200 import kvx
from paper_2510_11938_b200 import workload as W
from tests.replay import replay

SEED = 0x5EED


class GpuCase:
    def __init__(self, scn, t, heads, dim, device=0, oracle=True, oracle_pools=True, slack=0.25,
                 dst_blocks=None, dev_table=False):
        L = scn.num_layers
        self.scn, self.t = scn, t
        self.g = kvx.geometry(L, heads, dim)
        self.N = scn.num_requests
        self.tokens = t.max_tokens(self.N)
        self.max_blocks = int(max(1, (self.tokens.max() + 15) // 16))
        self.src_bt, self.old_blocks = W.fragmented_block_table(self.tokens, self.max_blocks, 16,
                                                                seed=7, slack=slack)
        need = int(((self.tokens + 15) // 16).sum())
        self.dst_blocks = dst_blocks if dst_blocks is not None else max(need, 1)
        self.live = np.nonzero(self.tokens)[0].astype(np.int32)
        self.old_pools = []
        for b, e in W.stage_ranges(L, t.old_boundaries):
            p = kvx.Pool(device, self.g, e - b, self.old_blocks)
            p.zero()
            p.fill_pattern(SEED, b, self.live, self.tokens[self.live], self.src_bt)
            self.old_pools.append(p)
        self.new_pools = []
        for b, e in W.stage_ranges(L, t.new_boundaries):
            p = kvx.Pool(device, self.g, e - b, self.dst_blocks)
            p.zero()
            self.new_pools.append(p)
        self.dev_bt = None
        if dev_table:  # the serving engine's device-resident copy; no host table passed
            import torch
            self.dev_bt = torch.from_numpy(np.ascontiguousarray(self.src_bt, np.int32)).to(f"cuda:{device}")
            torch.cuda.synchronize(device)
        self.tr = kvx.Transition(self.g, t.old_boundaries, self.old_pools, t.new_boundaries,
                                 self.new_pools, device, self.N, self.max_blocks, self.dst_blocks,
                                 None if dev_table else self.src_bt, epoch=t.epoch,
                                 max_sync_rounds=scn.max_sync_rounds,
                                 kv_bytes_per_token=scn.kv_bytes_per_token,
                                 src_block_table_dev=self.dev_bt.data_ptr() if dev_table else 0)
        self.dp = None
        if oracle:
            og = O.geo(L, heads, dim)
            self.dp = O.DataPlane(og, t.old_boundaries, t.new_boundaries, self.old_blocks,
                                  self.dst_blocks, self.N, self.max_blocks, self.src_bt,
                                  with_pools=oracle_pools)
            if oracle_pools:
                self.dp.fill_source(SEED, self.live, self.tokens[self.live])

    def run_ctl(self):
        """Drives the product's control mirror (kvx_ctl_*) through the golden
        transition; the oracle follows the same waves.  Returns (commit, ms)."""
        tr, dp = self.tr, self.dp
        octx = O.ControlCtx(self.N, self.scn.max_sync_rounds, self.scn.kv_bytes_per_token)
        ms = []

        class Shim:
            def begin(self_, req, kv):
                tok = tr.begin_refactor((req, kv))
                r = octx.begin(req, kv)
                assert tok == r[0]
                if dp is not None:
                    assert dp.wave(req, r[1], r[2]) == 0
                ms.append(tr.wait())
                return r

            def on_sync_complete(self_, req, kv, inflight):
                act, tok = tr.on_kv_sync_complete((req, kv), inflight)
                r = octx.on_sync_complete(req, kv, inflight)
                assert (act, tok) == (r[0], r[1])
                if dp is not None and act != kvx.ACT_BARRIER_WAIT:
                    assert dp.wave(req, r[2], r[3]) == 0
                ms.append(tr.wait())
                return r

        for w, _, _ in replay(Shim(), self.t):
            # same additions from 0 as the oracle ctx (itself pinned bit-exact
            # to the reference accumulator by test_golden_control)
            assert tr.ctl_state()["kv_synced_bytes"] == octx.kv_synced_bytes
        self.octx = octx
        return ms

    def compare_tables(self):
        np.testing.assert_array_equal(self.tr.dst_block_table(), self.dp.bt)

    def compare_bytes(self):
        for k, p in enumerate(self.new_pools):
            got = p.read()
            want = self.dp.new_pools[k]
            if not np.array_equal(got, want):
                bad = np.nonzero(got != want)[0]
                raise AssertionError(f"new stage {k}: {bad.size} bytes differ, first at {bad[:5]}")

    def compare_bytes_by_layer(self, seed: int = SEED):
        """Every byte of every destination pool against the oracle, one layer
        at a time, at any size: the expected layer is kvo_fill_layer over the
        ORACLE's destination table and synced marks (its allocation-only
        replay of the block rule), i.e. the payload on rows [0, synced) of
        each request and zeros everywhere else -- partial-block tails, spare
        blocks and never-allocated blocks included.  Does not use the
        product's own verify kernel."""
        L = self.scn.num_layers
        og = O.geo(L, self.g.num_kv_heads, self.g.head_dim)
        req = np.arange(self.N, dtype=np.int32)
        lb = self.dst_blocks * self.g.block_bytes
        want = np.empty(lb, np.uint8)
        for j, (b, e) in enumerate(W.stage_ranges(L, self.t.new_boundaries)):
            for ll in range(e - b):
                got = self.new_pools[j].read(ll * lb, lb)
                O.fill_layer(og, seed, b + ll, self.dst_blocks, req, self.dp.synced_hi, self.dp.bt, out=want)
                if not np.array_equal(got, want):
                    bad = np.nonzero(got != want)[0]
                    raise AssertionError(f"new stage {j} layer {b + ll}: {bad.size} bytes differ, "
                                         f"first at {bad[:5]}")

    def compare_source(self):
        for k, p in enumerate(self.old_pools):
            np.testing.assert_array_equal(p.read(), self.dp.old_pools[k])

    def close(self):
        self.tr.close()
        for p in self.old_pools + self.new_pools:
            p.close()
