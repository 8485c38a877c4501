#!/usr/bin/env bash
# (the KVX_L2_HINT switch was reverted after this A/B: profiles/r02am_ab_l2_store_hint.jsonl)
# Same-box A/B of the bulk mover's L2 policy (KVX_L2_HINT: bit 0 stores,
# bit 1 loads evict_first), interleaved reps: C3 bench (value, wave movers,
# stall back-to-back and after a decode step) and the L2-state probe.
# Usage (gpurun, 1 GPU): bash scripts/ab_l2_store.sh <tag> [hints] [reps]
set -u
tag=${1:-ab}; hints=${2:-"0 1 3"}; reps=${3:-3}
out=gpurun_out/${tag}_ab_l2_store.jsonl; : > $out
for r in $(seq 1 $reps); do
  for h in $hints; do
    KVX_L2_HINT=$h timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-ncu --no-weights \
      > gpurun_out/${tag}_b.json 2> gpurun_out/${tag}_b.err
    python - "$h" "$r" gpurun_out/${tag}_b.json >> $out <<'PY'
import json, sys
l = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
print(json.dumps({"l2_hint": int(sys.argv[1]), "rep": int(sys.argv[2]), "value": l["value"],
                  "w0_frac": l["roofline"]["frac"], "waves": l["move_ms_by_wave"], "stall": l["stall_ms"],
                  "stall_after_decode": l["stall"]["device_after_decode_ms"],
                  "final_after_decode": l["stall"]["final_wave_after_decode_ms"]}))
PY
  done
done
for h in $hints; do
  KVX_L2_HINT=$h timeout 300 python scripts/final_wave_l2.py --reps 10 --modes b2b,clean \
    | sed "s/^{/{\"l2_hint\": $h, /" >> $out
done
