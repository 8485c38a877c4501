"""Probe: does a shared block manager's pop on a busy stream race a push on
another stream?  Prints stream states and the ids transition A received."""
import time
import numpy as np
import torch
from paper_2510_11938_b200 import kvx

g = kvx.geometry(2, 1, 8)
N, mb, cap = 4, 4, 16
src_bt = np.arange(N * mb, dtype=np.int32).reshape(N, mb)
old = [kvx.Pool(0, g, 2, N * mb) for _ in range(2)]
new = [kvx.Pool(0, g, 2, cap)]
for p in old + new:
    p.zero()
bm = kvx.BlockManager(0, cap)
sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
tA = kvx.Transition(g, [], [old[0]], [], new, 0, N, mb, cap, src_bt, stream=sA.cuda_stream, dst_blockmgr=bm)
tB = kvx.Transition(g, [], [old[1]], [], new, 0, N, mb, cap, src_bt, stream=sB.cuda_stream, dst_blockmgr=bm)
tB.wave(np.array([0, 1], np.int32), np.zeros(2, np.int64), np.array([40, 40], np.int64))
tB.wait()
torch.cuda.synchronize()
t0 = time.time()
with torch.cuda.stream(sA):
    torch.cuda._sleep(int(3e8))
print("after sleep launch: sA idle?", sA.query(), round(time.time() - t0, 4))
tA.wave(np.array([0], np.int32), np.zeros(1, np.int64), np.array([50], np.int64))
print("after A.wave: sA idle?", sA.query(), round(time.time() - t0, 4))
res = tB.commit(np.array([0], np.int32), np.array([40], np.int64))
print("after B.commit: sA idle?", sA.query(), "free", res.free_list.tolist(), round(time.time() - t0, 4))
tA.wait()
print("A ids", tA.dst_block_table()[0].tolist(), round(time.time() - t0, 4))
