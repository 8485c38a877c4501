#!/usr/bin/env bash
# push vs pull vs auto movers at N=2 (one-way and two-way placements)
out=gpurun_out/movers2.jsonl; : > $out
timeout 900 python -m pytest tests/test_multirank.py -q -m gpu > gpurun_out/movers2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/movers2_pytest.log
run() { timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
          --master-port 29517 bench.py --gpus 2 --steps 20 --no-weights --no-cpu-baseline --e2e-steps 2 "$@" 2>/dev/null \
          | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); d['args']='$*'; print(json.dumps(d))" >> $out; }
for m in push auto pull; do run --placement oneway --move $m; done
for pc in 48 64 96; do KVX_PEER_CTAS=$pc run --placement oneway --move auto; sed -i "\$s/}\$/, \"peer_ctas\": $pc}/" $out; done
for m in push auto; do run --placement disjoint --move $m; done
