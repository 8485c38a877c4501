#!/usr/bin/env bash
# 4-GPU session: the 2- and 4-rank GPU tests on physical GPUs, the single-process
# multi-device tests, and the driver's scaling sequence (both arms, N=1,2,4).
set -u
tag=${1:-r02o}; o=gpurun_out
nvidia-smi topo -m > $o/${tag}_topo.txt 2>&1
timeout 1800 python -m pytest tests/test_multirank.py tests/test_gpu_multidevice.py -m gpu -q > $o/${tag}_pytest_4gpu.log 2>&1
echo "pytest rc=$?" >> $o/${tag}_pytest_4gpu.log
timeout 900 python bench.py --impl reference > $o/${tag}_ref_n1.jsonl 2>/dev/null
timeout 900 python bench.py > $o/${tag}_kvx_n1.jsonl 2>$o/${tag}_kvx_n1.err
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n \
    bench.py --impl reference --gpus $n > $o/${tag}_ref_n$n.jsonl 2>/dev/null
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n \
    bench.py --gpus $n > $o/${tag}_kvx_n$n.jsonl 2>$o/${tag}_kvx_n$n.err
done
