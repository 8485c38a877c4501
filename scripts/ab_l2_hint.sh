#!/usr/bin/env bash
# Same-box A/B of L2 cache-policy hints on the bulk mover's copies (KVX_L2_HINT:
# 0 none, 1 evict_first, 2 evict_unchanged), C3 bench, interleaved reps.
out=gpurun_out/${1:-r02}_ab_l2_hint.jsonl; : > $out
for rep in 1 2 3; do for h in 0 1 2; do
  KVX_L2_HINT=$h timeout 300 python bench.py --steps 30 --no-cpu-baseline --no-weights --no-ncu --e2e-steps 2 2>/dev/null \
    | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'l2_hint': $h, 'rep': $rep, 'value': d['value'], 'w0_frac': d['roofline']['frac'], 'waves': d['move_ms_by_wave'], 'stall': d['stall_ms']}))" >> $out
done; done
