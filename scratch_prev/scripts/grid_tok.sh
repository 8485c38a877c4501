#!/usr/bin/env bash
out=gpurun_out/grid_tok.jsonl; : > $out
for pass in 1 2; do for gt in 96 128 148; do
  KVX_BULK_GRID_TOK=$gt python bench.py --no-cpu-baseline --no-weights --steps 30 --e2e-steps 1 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'grid_tok':$gt,'waves':d['move_ms_by_wave'],'stall':d['stall_ms'],'handoff_stall':d['handoff']['stall_handoff_ms'],'value':d['value']}))" >> $out
done; done
cat $out
