#!/usr/bin/env bash
# Same-box A/B of the row mover's index math: plain divisions vs FastDiv
# (KVX_ROW_FASTDIV build flag; the two builds are in paper_2510_11938_b200/_lib_ab/).
out=gpurun_out/${1:-r02}_ab_row_div.jsonl; : > $out
L=paper_2510_11938_b200/_lib
cp $L/libkvx.so /tmp/libkvx_keep.so
for rep in 1 2; do for v in div fast; do
  cp paper_2510_11938_b200/_lib_ab/libkvx_$v.so $L/libkvx.so
  for lay in blocks,heads heads,blocks; do
    timeout 300 python bench.py --layouts $lay --steps 10 --no-cpu-baseline --no-weights --no-ncu --e2e-steps 2 2>/dev/null \
      | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'index_math': '$v', 'layouts': '$lay', 'rep': $rep, 'value': d['value'], 'frac': d['roofline']['frac'], 'waves': d['move_ms_by_wave'], 'stall': d['stall_ms']}))" >> $out
  done
done; done
cp /tmp/libkvx_keep.so $L/libkvx.so
