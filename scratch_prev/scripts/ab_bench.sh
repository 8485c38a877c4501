#!/usr/bin/env bash
# A/B of the default bench between the current tree and scratch_prev/ (an
# older tree exported next to it), alternating on the same box.
out=gpurun_out/ab.txt; : > $out
for i in 1 2 3; do
  for side in prev cur; do
    d=.; [ $side = prev ] && d=scratch_prev
    (cd $d && python bench.py --no-cpu-baseline --no-weights --steps 30 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$side', d['value'], d['roofline']['launch_ms'], d['roofline']['live_copy_reference']['torch_copy_GBps'])") >> $out
  done
done
cat $out
