"""Probe 2: which step of a commit on stream B waits for busy stream A?"""
import ctypes as C
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
use_bm = True
bm = kvx.BlockManager(0, cap)
sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
x = torch.zeros(16, device="cuda")
torch.cuda.synchronize()
# sanity: torch work on sB overtakes a sleeping sA
with torch.cuda.stream(sA):
    torch.cuda._sleep(int(2e8))
with torch.cuda.stream(sB):
    x.add_(1)
t0 = time.time(); sB.synchronize(); print("torch op on sB done after", round(time.time() - t0, 4), "sA idle?", sA.query())
torch.cuda.synchronize()

tA = kvx.Transition(g, [], [old[0]], [], new, 0, N, mb, cap, src_bt, stream=sA.cuda_stream, dst_blockmgr=bm)
tB = kvx.Transition(g, [], [old[1]], [], new, 0, N, mb, cap, src_bt, stream=sB.cuda_stream, dst_blockmgr=bm)
tB.wave(np.array([0, 1], np.int32), np.zeros(2, np.int64), np.array([40, 40], np.int64))
tB.wait()
torch.cuda.synchronize()
t0 = time.time()
with torch.cuda.stream(sA):
    torch.cuda._sleep(int(3e8))
stamp = lambda m: print(f"{m:28s} t={time.time() - t0:.4f} sA idle={sA.query()} sB idle={sB.query()}", flush=True)
stamp("sleep queued")
tB.wave(np.array([2], np.int32), np.zeros(1, np.int64), np.array([5], np.int64))
stamp("B.wave (no A wave yet)")
sB.synchronize()
stamp("B synced")
tA.wave(np.array([0], np.int32), np.zeros(1, np.int64), np.array([50], np.int64))
stamp("A.wave")
req = np.array([0, 2], np.int32); kv = np.array([40, 5], np.int64)
rc = kvx._lib.kvx_commit_async(tB._h, C.c_uint64(tB.epoch), 2, req.ctypes.data_as(C.POINTER(C.c_int32)),
                               kv.ctypes.data_as(C.POINTER(C.c_int64)))
stamp(f"B.commit_async rc={rc}")
sB.synchronize()
stamp("sB synced")
res = kvx._CommitResult()
rc = kvx._lib.kvx_commit_collect(tB._h, C.byref(res))
stamp(f"B.collect rc={rc} nfree={res.n_free}")
tA.wait()
print("A ids", tA.dst_block_table()[0].tolist())
