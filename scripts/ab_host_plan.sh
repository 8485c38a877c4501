#!/usr/bin/env bash
# Same-box A/B of host-planned waves (kvx_transition.cu, KVX_HOST_PLAN): 1 = the host
# builds the segments into pinned memory and the mover starts at once; 0 = the device
# plan kernel runs before the mover.
out=gpurun_out/${1:-r02}_ab_host_plan.jsonl; : > $out
for rep in 1 2 3; do for m in 0 1; do
  KVX_HOST_PLAN=$m timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-weights --no-ncu --e2e-steps 10 2>/dev/null \
    | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'host_plan': $m, 'rep': $rep, 'value': d['value'], 'e2e': d['e2e']['value'], 'ms_per_step': d['ms_per_step'], 'w0_frac': d['roofline']['frac'], 'stall_ms': d['stall_ms'], 'stall_range': d['stall_ms_all'], 'final_wave_ms': d['move_ms_by_wave'][-1], 'host_stall': d['stall']['host_observed_ms'], 'handoff_stall': (d['handoff'] or {}).get('stall_handoff_ms')}))" >> $out
done; done
