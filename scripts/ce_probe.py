"""Copy-engine feasibility for two-way NVLink (C3 disjoint N=2 shape).

One process drives two GPUs; each sends 8.4 GB to the other at the same time.
  ce1d      one cudaMemcpyAsync per layer (contiguous 420 MB: the CE ceiling)
  ce2d      the destination-run shape of a staged push: 256 cudaMemcpy2DAsync
            per GPU, each one request's run of full blocks (width) over all
            20 pushed layers (height, pitch = layer stride)
  ce2d_hbm  ce2d with a local 8.4 GB r+w copy on the same GPU beside it (the
            gather into the staging buffer)
  ce1d_runs one 1-D copy per (layer, run): 5,120 cudaMemcpyAsync per GPU
            (host issue time reported: the two GPUs are issued one after the other)
Per-direction GB/s = bytes / max over the two GPUs of the CUDA-event time.
Usage (gpurun --gpus 2): python scripts/ce_probe.py
"""
import json
import sys
import time

import torch
from cuda.bindings import runtime as rt


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    assert int(err) == 0, r
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None


def main():
    L, P = 20, 420 * (1 << 20)
    runs = 256
    width = P // runs // 4096 * 4096
    devs = [0, 1]
    for d in devs:
        torch.cuda.set_device(d)
        ck(rt.cudaSetDevice(d))
        r = rt.cudaDeviceEnablePeerAccess(1 - d, 0)
        assert int(r[0]) in (0, int(rt.cudaError_t.cudaErrorPeerAccessAlreadyEnabled)), r
    S = [torch.ones(L * P, dtype=torch.uint8, device=f"cuda:{d}") for d in devs]
    D = [torch.zeros(L * P, dtype=torch.uint8, device=f"cuda:{d}") for d in devs]
    X = [torch.ones(L * P // 2, dtype=torch.uint8, device=f"cuda:{d}") for d in devs]
    Y = [torch.zeros(L * P // 2, dtype=torch.uint8, device=f"cuda:{d}") for d in devs]
    st = [torch.cuda.Stream(device=d) for d in devs]
    hs = [torch.cuda.Stream(device=d) for d in devs]
    kind = rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice

    def issue(mode, d):
        s = st[d].cuda_stream
        src, dst = S[d].data_ptr(), D[1 - d].data_ptr()
        if mode == "ce1d":
            for l in range(L):
                ck(rt.cudaMemcpyAsync(dst + l * P, src + l * P, P, kind, s))
            return L * P
        if mode.startswith("ce1d_runs"):  # one 1-D copy per (layer, run): 5,120 calls per GPU
            for l in range(L):
                for r in range(runs):
                    o = l * P + r * width
                    ck(rt.cudaMemcpyAsync(dst + o, src + o, width, kind, s))
            return runs * width * L
        for r in range(runs):
            ck(rt.cudaMemcpy2DAsync(dst + r * width, P, src + r * width, P, width, L, kind, s))
        if mode == "ce2d_hbm":
            with torch.cuda.stream(hs[d]):
                Y[d].copy_(X[d])
                Y[d].copy_(X[d])
        return runs * width * L

    out = []
    modes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["ce1d", "ce2d", "ce2d_hbm", "ce1d", "ce2d", "ce2d_hbm"]
    for mode in modes:
        times, hosts = [], []
        for rep in range(4):
            for d in devs:
                torch.cuda.synchronize(d)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in devs]
            for d in devs:
                ev[d][0].record(st[d])
                hs[d].wait_stream(st[d])
            nb = 0
            h0 = time.perf_counter()
            for d in devs:
                torch.cuda.set_device(d)
                nb = issue(mode, d)
            host_ms = (time.perf_counter() - h0) * 1e3
            for d in devs:
                st[d].wait_stream(hs[d])
                ev[d][1].record(st[d])
            for d in devs:
                torch.cuda.synchronize(d)
            t = max(ev[d][0].elapsed_time(ev[d][1]) for d in devs)
            if rep:
                times.append(t)
                hosts.append(host_ms)
        t = sorted(times)[len(times) // 2]
        line = {"mode": mode, "bytes_per_direction": nb, "ms": round(t, 3),
                "GBps_per_direction": round(nb / (t * 1e-3) / 1e9, 1), "frac_770": round(nb / (t * 1e-3) / 770e9, 4),
                "host_issue_ms_both_gpus": round(sorted(hosts)[len(hosts) // 2], 3)}
        print(json.dumps(line), flush=True)
        out.append(line)


if __name__ == "__main__":
    main()
