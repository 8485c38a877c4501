#!/usr/bin/env bash
# TMA transposer grid sweep on C3 layout conversions (CFGS="hc:grid ..."; the hc
# part only took effect with the temporary KVX_TMAP_HC knob of the first sweeps).
out=gpurun_out/tmap_grid.jsonl; : > $out
for rep in 1 2; do
  for lay in blocks,heads heads,blocks; do
    for cfg in ${CFGS:-8:96 8:128}; do
      hc=${cfg%%:*}; grid=${cfg##*:}
      KVX_TMAP_GRID=$grid timeout 300 python bench.py --layouts $lay --steps 10 --no-cpu-baseline --no-weights --no-ncu --e2e-steps 2 2>/dev/null \
       | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'layouts': '$lay', 'hc': $hc, 'grid': $grid, 'rep': $rep, 'frac': d['roofline']['frac'], 'w0_ms': d['roofline']['launch_ms']}))" >> $out
    done
  done
done
