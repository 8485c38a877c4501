"""NVLink calibration on this box: copy-engine peer copies (torch copy_
between two GPUs in one process), one direction and both directions at
once, 4 GiB per direction.  Prints GB/s per direction."""
import json
import torch

n = 4 << 30
a0 = torch.empty(n, dtype=torch.uint8, device="cuda:0")
b1 = torch.empty(n, dtype=torch.uint8, device="cuda:1")
a1 = torch.empty(n, dtype=torch.uint8, device="cuda:1")
b0 = torch.empty(n, dtype=torch.uint8, device="cuda:0")
s0 = torch.cuda.Stream(device=0)
s1 = torch.cuda.Stream(device=1)
out = {}
for mode in ("uni", "bi"):
    times = []
    for rep in range(4):
        torch.cuda.synchronize(0); torch.cuda.synchronize(1)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        f = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(s0):
            e[0].record(s0)
            b1.copy_(a0, non_blocking=True)     # GPU0 -> GPU1
            e[1].record(s0)
        if mode == "bi":
            with torch.cuda.stream(s1):
                f[0].record(s1)
                b0.copy_(a1, non_blocking=True)  # GPU1 -> GPU0
                f[1].record(s1)
        torch.cuda.synchronize(0); torch.cuda.synchronize(1)
        if rep:
            t = e[0].elapsed_time(e[1])
            if mode == "bi":
                t = max(t, f[0].elapsed_time(f[1]))
            times.append(t)
    ms = min(times)
    out[mode] = round(n / (ms * 1e-3) / 1e9, 1)
print(json.dumps({"ce_peer_copy_GBps_per_direction": out, "bytes": n}))
