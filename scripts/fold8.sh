#!/usr/bin/env bash
# The driver's N=8 scaling command on a 4-GPU box: 8 ranks folded onto 4 GPUs
# (KVX_BENCH_FOLD=4).  A functional check of the N=8 placement, IPC exchange,
# timing and JSON path -- not a measurement.
out=gpurun_out/${1:-r02}_fold8.jsonl
: > $out
export KVX_BENCH_FOLD=4 KVX_BENCH_FOLD_PROBE=1
run8() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
           --master-port 29513 bench.py --gpus 8 "$@" 2> gpurun_out/fold8_err.log | grep '^{\|bench:' >> $out
         echo "rc=${PIPESTATUS[0]} args=$*" >> gpurun_out/fold8_rc.log; }
: > gpurun_out/fold8_rc.log
run8 --steps 5 --warmup 3
run8 --steps 5 --warmup 3 --config c2 --placement spread --no-weights --no-cpu-baseline
run8 --steps 5 --warmup 3 --config c4r --placement disjoint --no-weights --no-cpu-baseline
run8 --steps 5 --warmup 3 --pull --no-weights --no-cpu-baseline
unset KVX_BENCH_FOLD KVX_BENCH_FOLD_PROBE
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
  --master-port 29514 bench.py --impl reference --gpus 8 --steps 3 --warmup 3 2>>gpurun_out/fold8_err.log | grep '^{' >> $out
echo "rc=${PIPESTATUS[0]} args=reference" >> gpurun_out/fold8_rc.log
