#!/usr/bin/env bash
# (the KVX_PLAN_FAST switch was reverted after this A/B: profiles/r02am_ab_plan_fast.jsonl)
# Same-box A/B of the plan kernel's load order (KVX_PLAN_FAST: 1 = the first
# segment's table loads before the scan, 0 = after it), interleaved reps of
# the C3 bench (stall back to back and after a decode step, wave movers).
# Usage (gpurun, 1 GPU): bash scripts/ab_plan_fast.sh <tag> [reps]
set -u
tag=${1:-ab}; reps=${2:-4}
out=gpurun_out/${tag}_ab_plan_fast.jsonl; : > $out
for r in $(seq 1 $reps); do
  for f in 0 1; do
    KVX_PLAN_FAST=$f timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-ncu --no-weights \
      > gpurun_out/${tag}_b.json 2> gpurun_out/${tag}_b.err
    python - "$f" "$r" gpurun_out/${tag}_b.json >> $out <<'PY'
import json, sys
l = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
print(json.dumps({"plan_fast": int(sys.argv[1]), "rep": int(sys.argv[2]), "value": l["value"],
                  "waves": l["move_ms_by_wave"], "stall": l["stall_ms"], "stall_range": l["stall_ms_all"],
                  "stall_after_decode": l["stall"]["device_after_decode_ms"],
                  "host_observed": l["stall"]["host_observed_ms"]}))
PY
  done
done
