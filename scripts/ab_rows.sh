#!/usr/bin/env bash
# Row mover (layout-converting moves) on the C3 bench: the build under test, 3 reps.
out=gpurun_out/${1:-r02}_rows.jsonl; : > $out
for rep in 1 2 3; do for lay in blocks,heads heads,blocks planes,heads; do
  timeout 300 python bench.py --layouts $lay --steps 10 --no-cpu-baseline --no-weights --no-ncu --e2e-steps 2 2>/dev/null \
    | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'layouts': '$lay', 'rep': $rep, 'value': d['value'], 'frac': d['roofline']['frac'], 'waves': d['move_ms_by_wave'], 'stall': d['stall_ms']}))" >> $out
done; done
