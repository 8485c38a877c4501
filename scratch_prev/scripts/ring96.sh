#!/usr/bin/env bash
out=gpurun_out/ring96.jsonl; : > $out
for pass in 1 2; do for cfg in 0 1 2 3 4 5 6 7; do
  KVX_BULK_CFG=$cfg python bench.py --no-cpu-baseline --no-weights --steps 20 --e2e-steps 1 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':$cfg,'waves':d['move_ms_by_wave'],'value':d['value']}))" >> $out
done; done
