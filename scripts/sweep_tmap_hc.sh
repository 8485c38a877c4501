#!/usr/bin/env bash
# (KVX_TMAP_HC was a temporary knob for this sweep, removed after it: profiles/r02am_tmap_head_chunk_sweep.jsonl)
out=gpurun_out/tmap_hc.jsonl; : > $out
for rep in 1 2; do
  for lay in blocks,heads heads,blocks; do
    for hc in 8 4 2 1; do
      KVX_TMAP_HC=$hc timeout 300 python bench.py --layouts $lay --steps 10 --no-cpu-baseline --no-weights --no-ncu --e2e-steps 2 2>/dev/null \
       | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'layouts': '$lay', 'hc': $hc, 'rep': $rep, 'frac': d['roofline']['frac'], 'w0_ms': d['roofline']['launch_ms']}))" >> $out
    done
  done
done
