#!/usr/bin/env bash
# push vs auto movers at N=4
out=gpurun_out/movers4.jsonl; : > $out
run() { timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
          --master-port 29519 bench.py --gpus 4 --steps 20 --no-weights --no-cpu-baseline --e2e-steps 2 "$@" 2>/dev/null \
          | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); d['args']='$*'; print(json.dumps(d))" >> $out; }
for m in push auto; do
  run --placement oneway --move $m
  run --config c2 --placement spread --move $m
  run --placement disjoint --move $m
done
run
