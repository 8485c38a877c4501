#!/usr/bin/env bash
# ncu evidence for the bench's dominant kernel (run under gpurun, 1 GPU).
# Each ncu command is preceded by the same command line run without ncu.
set -u
out=gpurun_out
tag=${1:-r01b}
C3="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-verify --no-weights --no-ncu"
C1="python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-verify --no-weights --no-ncu"
: > $out/ncu_status.txt
# 1. launch list of the C3 bench (every kernel, device time; cold-cache, serialised)
$C3 > $out/plain_c3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $out/${tag}_launches_c3.csv $C3 > $out/ncu_launches.log 2>&1
echo "launches rc=$?" >> $out/ncu_status.txt
# 2. DRAM traffic of the C3 wave-0 mover launch (a bench-size launch; 2 movers per step)
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:kvx_bulk_kernel -s 6 -c 1 --csv \
    --log-file $out/${tag}_bulk_traffic_c3.csv $C3 > $out/ncu_traffic.log 2>&1
echo "traffic rc=$?" >> $out/ncu_status.txt
# 3. full section set on the same kernel at the C1 size (2 GiB wave 0)
$C1 > $out/plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:kvx_bulk_kernel -s 6 -c 1 \
    -o $out/${tag}_bulk_c1 $C1 > $out/ncu_full.log 2>&1
echo "full rc=$?" >> $out/ncu_status.txt
