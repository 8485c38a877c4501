"""Block-manager restatement (CPU): a fresh free stack reproduces the bump
rule; commit pushes the finished requests' blocks, abort pushes every block,
later allocations reuse them LIFO."""
import numpy as np

from oracle import pyoracle as O
from paper_2510_11938_b200 import workload as W

SEED = 5


def plane(tokens, bm=None, max_blocks=6):
    g = O.geo(4, 1, 8)
    src_bt, old_blocks = W.fragmented_block_table(tokens, max_blocks, 16, seed=1)
    dp = O.DataPlane(g, [2], [1, 3], old_blocks, 64, len(tokens), max_blocks, src_bt, bm=bm)
    live = np.nonzero(tokens)[0]
    dp.fill_source(SEED, live, tokens[live])
    return dp


def test_fresh_stack_equals_bump():
    tokens = np.array([40, 17, 0, 90], np.int64)
    a, b = plane(tokens), plane(tokens, bm=O.StackBM(64))
    req = np.array([0, 1, 3])
    for lo, hi in ((np.zeros(3, np.int64), np.array([20, 16, 33])), (np.array([20, 16, 33]), tokens[req])):
        assert a.wave(req, lo, hi) == 0 and b.wave(req, lo, hi) == 0
    np.testing.assert_array_equal(a.bt, b.bt)
    assert b.bm.top == 64 - int(((tokens + 15) // 16).sum())


def test_commit_pushes_and_lifo_reuse():
    tokens = np.array([40, 17, 33, 0], np.int64)
    bm = O.StackBM(64)
    dp = plane(tokens, bm=bm)
    dp.wave([0, 1, 2], [0, 0, 0], [40, 17, 33])          # blocks 0..2 | 3,4 | 5,6,7
    v, row_ptr, blocks, free = dp.commit([0, 2], [40, 33])  # request 1 finished
    assert v == 0 and free.tolist() == [3, 4]
    assert bm.top == 64 - 8 + 2
    assert bm.pop(3).tolist() == [4, 3, 8]               # LIFO: freed ids first, then fresh


def test_abort_returns_everything():
    tokens = np.array([40, 17, 33, 0], np.int64)
    bm = O.StackBM(16)
    dp = plane(tokens, bm=bm)
    dp.wave([0, 1, 2], [0, 0, 0], [40, 17, 33])
    assert bm.top == 8
    dp.abort()
    assert bm.top == 16 and (dp.bt == -1).all()
    assert sorted(bm.snapshot().tolist()) == list(range(16))


def test_exhaustion_rejects_the_whole_wave():
    tokens = np.array([40, 40, 0, 0], np.int64)
    bm = O.StackBM(5)
    dp = plane(tokens, bm=bm)
    assert dp.wave([0, 1], [0, 0], [40, 40]) == -1       # needs 6 > 5: nothing taken
    assert bm.top == 5 and (dp.bt == -1).all()
