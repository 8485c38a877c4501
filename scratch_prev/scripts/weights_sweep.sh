#!/usr/bin/env bash
out=gpurun_out/weights_sweep.jsonl; : > $out
for pass in 1 2; do for spec in "32k 148" "slab 96" "slab 128" "slab 148" "32k 96"; do set -- $spec
  KVX_WEIGHTS_RING=$1 KVX_WEIGHTS_GRID=$2 python bench.py --no-cpu-baseline --steps 5 --e2e-steps 1 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); w=d['weights']; print(json.dumps({'ring':'$1','grid':$2,'ms':w['ms'],'GB_s':w['GB_s'],'frac':w['hbm_frac']}))" >> $out
done; done
cat $out
