#!/usr/bin/env bash
# same-box A/B of the refactor stall: scratch_prev/ (older tree) vs the current tree
out=gpurun_out/ab_stall.txt; : > $out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_blockmgr.py tests/test_gpu_layouts.py tests/test_gpu_handoff.py -q -m gpu 2>&1 | tail -1 >> $out
for i in 1 2 3; do for side in prev cur; do
  d=.; [ $side = prev ] && d=scratch_prev
  (cd $d && python bench.py --no-cpu-baseline --no-weights --steps 30 --e2e-steps 3 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$side', d['value'], d['e2e']['value'], 'stall', d['stall_ms'], 'handoff', d['handoff']['stall_handoff_ms'], d['move_ms_by_wave'])") >> $out
done; done
cat $out
