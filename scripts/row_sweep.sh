#!/usr/bin/env bash
out=gpurun_out/row_sweep.jsonl; : > $out
for l in blocks,heads heads,blocks; do for o in 0 1; do for c in 0 1 2 3 4; do
  KVX_ROW_ORDER_DST=$o KVX_ROW_CTAS_PER_SM=$c python bench.py --no-cpu-baseline --no-weights --steps 10 --e2e-steps 1 --layouts $l 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'layouts':'$l','order_dst':$o,'ctas_per_sm':$c,'w0':d['move_ms_by_wave'][0],'value':d['value']}))" >> $out
done; done; done
cat $out
