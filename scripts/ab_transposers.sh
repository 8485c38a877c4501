out=gpurun_out/r02af_ab3.jsonl; : > $out
L=paper_2510_11938_b200/_lib
cp $L/libkvx.so /tmp/keep.so
run() { timeout 300 python bench.py --layouts $1 --steps 10 --no-cpu-baseline --no-weights --no-ncu --e2e-steps 2 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'variant': '$2', 'layouts': '$1', 'frac': d['roofline']['frac'], 'final_ms': d['move_ms_by_wave'][-1], 'sm_mhz': d['clocks'].get('sm_mhz')}))" >> $out; }
for rep in 1 2; do
  cp paper_2510_11938_b200/_lib_ab/libkvx_orig.so $L/libkvx.so
  for lay in blocks,heads heads,blocks; do KVX_TMAP=0 run $lay rows_div; done
  cp paper_2510_11938_b200/_lib_ab/libkvx_fast.so $L/libkvx.so
  for lay in blocks,heads heads,blocks; do KVX_TMAP=0 run $lay rows_fastdiv; KVX_TMAP=1 run $lay tmap; done
done
cp /tmp/keep.so $L/libkvx.so
