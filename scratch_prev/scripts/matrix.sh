#!/usr/bin/env bash
# Results matrix: configs x GPUs x placements (needs a 4-GPU box for the N=4 rows).
out=gpurun_out/matrix.jsonl
: > $out
common="--steps 20 --warmup 3 --no-weights --e2e-steps 2 --no-cpu-baseline"
for c in c1 c2 c3 c4r; do
  timeout 300 python bench.py --config $c $common 2>/dev/null | grep '^{' >> $out
done
for n in 2 4; do
  for c in c2 c3 c4r; do
    for pl in affinity spread disjoint; do
      timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 29511 bench.py --gpus $n --config $c --placement $pl $common 2>/dev/null | grep '^{' >> $out
    done
  done
done
