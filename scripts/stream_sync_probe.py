"""Which operations issued on stream B wait for an unrelated busy stream A?
Stream A runs a ~100 ms spin kernel; each op is issued on B and we time how
long B takes to drain.  ~0 = concurrent, ~100 ms = implicit serialisation.
The block-manager host-array calls (kvx_bm_pop / push / snapshot / reset)
run on the manager's own stream, so they are timed by their host call.
Ends with one JSON line: every kvx op and whether it blocked on stream A."""
import ctypes as C
import glob
import os
import sys
import time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_11938_b200 import kvx

rt = C.CDLL(sorted(glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                          "libcudart.so*")))[0])
sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
x = torch.zeros(1 << 20, device="cuda")
y = torch.zeros(1 << 20, device="cuda")
g = kvx.geometry(2, 1, 8)
N, mb, cap = 4, 4, 16
src_bt = np.arange(N * mb, dtype=np.int32).reshape(N, mb)
old = [kvx.Pool(0, g, 2, N * mb)]
new = [kvx.Pool(0, g, 2, cap)]
for p in old + new:
    p.zero()
torch.cuda.synchronize()


RESULTS = {}


def probe(name, fn):
    torch.cuda.synchronize()
    with torch.cuda.stream(sA):
        torch.cuda._sleep(int(2e8))
    t0 = time.time()
    fn()
    t1 = time.time()
    sB.synchronize()
    t2 = time.time()
    a_busy = not sA.query()
    print(f"{name:40s} host call {1e3 * (t1 - t0):7.2f} ms   B drained after {1e3 * (t2 - t0):7.2f} ms"
          f"   A idle at drain: {not a_busy}", flush=True)
    if name.startswith("kvx"):
        RESULTS[name] = {"host_ms": round(1e3 * (t1 - t0), 3), "drain_ms": round(1e3 * (t2 - t0), 3),
                         "blocked_on_A": not a_busy}


def d2d():
    rt.cudaMemcpyAsync(C.c_void_p(y.data_ptr()), C.c_void_p(x.data_ptr()), C.c_size_t(4096), 3,
                       C.c_void_p(sB.cuda_stream))


def memset():
    rt.cudaMemsetAsync(C.c_void_p(y.data_ptr()), 0, C.c_size_t(4096), C.c_void_p(sB.cuda_stream))


def torch_copy():
    with torch.cuda.stream(sB):
        y.copy_(x)


def torch_add():
    with torch.cuda.stream(sB):
        y.add_(1)


state = {}


def begin(bm=None):
    def f():
        state["t"] = kvx.Transition(g, [], old, [], new, 0, N, mb, cap, src_bt, stream=sB.cuda_stream,
                                    dst_blockmgr=bm)
    return f


def wave():
    state["t"].wave(np.array([0, 1], np.int32), np.zeros(2, np.int64), np.array([40, 40], np.int64))


def commit():
    t = state["t"]
    req, kv = np.array([0], np.int32), np.array([40], np.int64)
    assert kvx._lib.kvx_commit_async(t._h, C.c_uint64(t.epoch), 1, req.ctypes.data_as(C.POINTER(C.c_int32)),
                                     kv.ctypes.data_as(C.POINTER(C.c_int64))) == 0


def collect():
    res = kvx._CommitResult()
    assert kvx._lib.kvx_commit_collect(state["t"]._h, C.byref(res)) == 0


probe("torch add_ (kernel)", torch_add)
probe("torch copy_ same device", torch_copy)
probe("cudaMemcpyAsync D2D 4 KiB", d2d)
probe("cudaMemsetAsync 4 KiB", memset)
probe("kvx_begin (no block manager)", begin())
probe("kvx_wave", wave)
probe("kvx_commit_async (no block manager)", commit)
collect(); state["t"].close()
bm = kvx.BlockManager(0, cap)
probe("kvx_begin (block manager)", begin(bm))
probe("kvx_wave (block manager)", wave)
probe("kvx_commit_async (block manager, 3 freed)", commit)
collect(); state["t"].close()
bm2 = kvx.BlockManager(0, cap)
ids = torch.zeros(4, dtype=torch.int32, device="cuda")
host_ids = {}
probe("kvx_bm_pop (host ids)", lambda: host_ids.setdefault("v", bm2.pop(4)))
probe("kvx_bm_push (host ids)", lambda: bm2.push(host_ids["v"]))
probe("kvx_bm_pop_async (device ids)", lambda: bm2.pop_async(4, ids.data_ptr(), sB.cuda_stream))
probe("kvx_bm_push_async (device ids)", lambda: bm2.push_async(4, ids.data_ptr(), sB.cuda_stream))
probe("kvx_bm_snapshot", lambda: bm2.snapshot())
dev_bt = torch.from_numpy(src_bt).to("cuda")
torch.cuda.synchronize()


def begin_dev():
    state["t"] = kvx.Transition(g, [], old, [], new, 0, N, mb, cap, None, stream=sB.cuda_stream,
                                src_block_table_dev=dev_bt.data_ptr())


probe("kvx_begin (device source table)", begin_dev)
probe("kvx_wave (device source table)", wave)
probe("kvx_commit_async (device source table)", commit)
collect(); state["t"].close()
import json  # noqa: E402
print(json.dumps({"probe": "stream_sync", "ops": RESULTS,
                  "blocked": sorted(k for k, v in RESULTS.items() if v["blocked_on_A"])}), flush=True)
