#!/usr/bin/env bash
# ncu evidence for the stall-critical launch: the C3 FINAL-wave mover (the
# second kvx_bulk_kernel launch of one transition; 256 tokens x 40 layers x
# 20 KiB runs).  Plain run first, then the launch list, then --set full.
# Usage (gpurun, 1 GPU): bash scripts/ncu_final_wave.sh <tag> [extra env...]
set -u
tag=${1:-r02}
out=gpurun_out
P="python bench.py --traffic-probe --probe-all-waves --config c3"
$P > $out/${tag}_final_plain.log 2>&1; echo "plain rc=$?" > $out/${tag}_final_status.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:kvx_bulk_kernel --csv --log-file $out/${tag}_final_launches.csv $P \
    > $out/${tag}_final_ncu1.log 2>&1; echo "launches rc=$?" >> $out/${tag}_final_status.txt
ncu --set full --clock-control none --import-source on -k regex:kvx_bulk_kernel -s 1 -c 1 \
    -o $out/${tag}_final_full $P > $out/${tag}_final_ncu2.log 2>&1; echo "full rc=$?" >> $out/${tag}_final_status.txt
ncu -i $out/${tag}_final_full.ncu-rep --page raw --csv > $out/${tag}_final_full_raw.csv 2>/dev/null
ncu -i $out/${tag}_final_full.ncu-rep --page details --csv > $out/${tag}_final_full_details.csv 2>/dev/null
