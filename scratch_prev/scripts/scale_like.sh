#!/usr/bin/env bash
# The driver's scaling sequence on one box: N=1,2,4 back to back, both arms.
o=gpurun_out/scale; mkdir -p $o
python bench.py --impl reference > $o/ref_n1.jsonl 2>/dev/null
python bench.py > $o/kvx_n1.jsonl 2>/dev/null
for n in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n \
    bench.py --impl reference --gpus $n > $o/ref_n$n.jsonl 2>/dev/null
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n \
    bench.py --gpus $n > $o/kvx_n$n.jsonl 2>/dev/null
done
