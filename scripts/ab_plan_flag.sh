#!/usr/bin/env bash
# Same-box A/B of the plan -> commit hand-off on the stall path (kvx_transition.cu):
# KVX_PLAN_FLAG=1 (default): the commit kernel waits on the plan kernel's sequence
# word, no event between plan kernel and mover; 0: an event after the plan kernel.
out=gpurun_out/${1:-r02}_ab_plan_flag.jsonl; : > $out
for rep in 1 2 3; do for m in 0 1; do
  KVX_PLAN_FLAG=$m timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-weights --no-ncu --e2e-steps 2 2>/dev/null \
    | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'plan_flag': $m, 'rep': $rep, 'value': d['value'], 'ms_per_step': d['ms_per_step'], 'stall_ms': d['stall_ms'], 'stall_range': d['stall_ms_all'], 'final_wave_ms': d['move_ms_by_wave'][-1], 'host_stall': d['stall']['host_observed_ms'], 'handoff_stall': (d['handoff'] or {}).get('stall_handoff_ms')}))" >> $out
done; done
