#!/usr/bin/env bash
# NVLink evidence and the two-way push sweep at N GPUs (gpurun --gpus N):
#   1. bench lines: disjoint (two-way, pushed) over peer-CTA counts, oneway (pulled)
#   2. ncu on rank 0 (scripts/ncu_rank0.sh): NVLink tx/rx + DRAM bytes of the
#      wave-0 and final-wave movers, for both placements
# Each ncu command follows the same command run without ncu.
set -u
N=${1:-2}; tag=${2:-r02}
out=gpurun_out; j=$out/${tag}_nvlink_n${N}.jsonl; : > $j
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
B="bench.py --gpus $N --steps 20 --warmup 3 --no-weights --no-cpu-baseline --e2e-steps 2"
run() { timeout 500 $TR $B "$@" 2>>$out/${tag}_nvlink_err.log | grep '^{' | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); d['args']='$* peer_ctas=${KVX_PEER_CTAS:-default}'; print(json.dumps(d))" >> $j; }
run --placement disjoint --move push
for pc in 24 48 64 96; do KVX_PEER_CTAS=$pc run --placement disjoint --move push; done
run --placement oneway --move auto
run --placement oneway --move push
NB="bench.py --gpus $N --steps 2 --warmup 3 --no-weights --no-cpu-baseline --no-nccl --e2e-steps 1 --no-verify"
for pl in "disjoint --move push" "oneway --move auto"; do
  name=$(echo $pl | cut -d' ' -f1)
  timeout 500 $TR $NB --placement $pl > $out/${tag}_nvl_plain_${name}_n${N}.log 2>&1
  timeout 900 $TR --no-python scripts/ncu_rank0.sh $out/${tag}_nvl_ncu_${name}_n${N}.csv 6 2 $NB --placement $pl \
      > $out/${tag}_nvl_ncu_${name}_n${N}.log 2>&1
  echo "$name ncu rc=$?" >> $out/${tag}_nvlink_status.txt
done
