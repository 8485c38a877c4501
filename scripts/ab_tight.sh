#!/usr/bin/env bash
# Same-box A/B of the launch sequence on the stall path (KVX_TIGHT, kvx_transition.cu):
# 0 = timing events around every mover (default), 1 = none, 2 = none and the
# plan kernel adjacent to the mover (programmatic dependent launch).
out=gpurun_out/${1:-r02}_ab_tight.jsonl; : > $out
for rep in 1 2; do for m in 0 1 2; do
  KVX_TIGHT=$m timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-weights --no-ncu --e2e-steps 2 2>/dev/null \
    | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'tight': $m, 'rep': $rep, 'value': d['value'], 'ms_per_step': d['ms_per_step'], 'stall_ms': d['stall_ms'], 'stall_range': d['stall_ms_all'], 'host_stall': d['stall']['host_observed_ms'], 'handoff_stall': (d['handoff'] or {}).get('stall_handoff_ms')}))" >> $out
done; done
