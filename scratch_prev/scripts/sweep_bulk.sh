#!/usr/bin/env bash
# Mover variant sweep on the C3 bench (1 GPU).  Output: gpurun_out/sweep.jsonl
out=gpurun_out/sweep.jsonl
: > $out
for v in 0 1 2 3 4 5 6 7; do
  KVX_BULK_CFG=$v timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 2 | grep '^{' >> $out
done
KVX_MOVE_IMPL=lsu timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 2 | grep '^{' >> $out
