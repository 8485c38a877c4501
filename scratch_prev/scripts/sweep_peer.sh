#!/usr/bin/env bash
# Mover variants on the all-NVLink placement (2 GPUs).  Output: gpurun_out/sweep_peer.jsonl
out=gpurun_out/sweep_peer.jsonl
: > $out
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --placement disjoint --no-nccl \
        --e2e-steps 2 2>/dev/null | grep '^{' >> $out; }
for v in 0 1 2 3 4 5 6 7; do KVX_BULK_CFG=$v run; done
KVX_PEER_BULK=0 run
