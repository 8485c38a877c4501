#!/usr/bin/env bash
out=gpurun_out/check4.jsonl
: > $out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu4.log
common="--steps 30 --warmup 3 --no-weights --e2e-steps 2 --no-cpu-baseline"
for c in c3 c2 c4r; do timeout 300 python bench.py --config $c $common 2>/dev/null | grep '^{' >> $out; done
for n in 2 4; do
  for spec in "c3 affinity" "c3 disjoint" "c2 spread" "c3 spread" "c4r disjoint"; do
    set -- $spec
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 29511 bench.py --gpus $n --config $1 --placement $2 $common 2>/dev/null | grep '^{\|bench:' >> $out
  done
done
