#!/usr/bin/env bash
# same-box A/B (scratch_prev/ = older tree) for layout-converting refactors
out=gpurun_out/ab_layouts.txt; : > $out
for i in 1 2; do for l in blocks,heads heads,heads; do for side in prev cur; do
  d=.; [ $side = prev ] && d=scratch_prev
  (cd $d && python bench.py --no-cpu-baseline --no-weights --steps 20 --e2e-steps 1 --layouts $l 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$side $l', d['value'], d['move_ms_by_wave'])") >> $out
done; done; done
cat $out
