#!/usr/bin/env bash
out=gpurun_out/ab_transpose.txt; : > $out
python -m pytest tests/test_gpu_layouts.py tests/test_gpu_edges.py -q -m gpu 2>&1 | tail -1 >> $out
for i in 1 2; do for l in blocks,heads heads,blocks planes,heads; do for tp in 1 0; do
  KVX_TRANSPOSE=$tp python bench.py --no-cpu-baseline --no-weights --steps 20 --e2e-steps 1 --layouts $l 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print('transposer=$tp $l', d['value'], d['roofline']['frac'], d['move_ms_by_wave'], d['stall_ms'])" >> $out
done; done; done
cat $out
