#!/usr/bin/env bash
# TMA transposer vs row mover on C3 layout conversions, same box, interleaved reps.
out=gpurun_out/${1:-r02}_ab_tmap.jsonl; : > $out
run() { timeout 300 python bench.py --layouts $1 --steps 10 --no-cpu-baseline --no-weights --no-ncu --e2e-steps 2 2>/dev/null \
  | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'layouts': '$1', 'tmap': '${KVX_TMAP:-1}', 'rep': $2, 'value': d['value'], 'frac': d['roofline']['frac'], 'w0_ms': d['roofline']['launch_ms'], 'sm_mhz': d['clocks'].get('sm_mhz'), 'reasons': d['clocks'].get('reasons')}))" >> $out; }
for rep in 1 2 3; do
  for lay in blocks,heads heads,blocks; do
    KVX_TMAP=0 run $lay $rep
    KVX_TMAP=1 run $lay $rep
  done
done
