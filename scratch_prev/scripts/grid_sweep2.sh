#!/usr/bin/env bash
# Grid x ring sweep of the wave-0 mover on this box (identified by GPU UUID),
# alternating configurations, two passes.
out=gpurun_out/grid2_$(nvidia-smi --query-gpu=uuid --format=csv,noheader | head -1 | cut -c5-12).jsonl; : > $out
uuid=$(nvidia-smi --query-gpu=uuid,pci.bus_id --format=csv,noheader | head -1)
for pass in 1 2; do
  for g in 64 96 112 128 148; do
    for cfg in auto 0 2; do
      if [ $cfg = auto ]; then e=""; else e="KVX_BULK_CFG=$cfg"; fi
      env KVX_BULK_GRID=$g $e python bench.py --no-cpu-baseline --no-weights --steps 20 --e2e-steps 1 2>/dev/null | tail -1 | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'uuid':'$uuid','pass':$pass,'grid':$g,'cfg':'$cfg','launch_ms':r['launch_ms'],'value':d['value'],'torch_copy':r['live_copy_reference']['torch_copy_GBps']}))" >> $out
    done
  done
done
cat $out
