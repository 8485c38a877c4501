#!/usr/bin/env bash
# ncu evidence for the row mover (token-major -> head-major transpose)
out=gpurun_out; tag=${1:-r01}
C1="python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-verify --no-weights --layouts blocks,heads"
C3="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-verify --no-weights --layouts blocks,heads"
$C3 > $out/plain_rows_c3.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:kvx_move_any_kernel -s 6 -c 1 --csv --log-file $out/${tag}_rows_traffic_c3.csv $C3 > $out/ncu_rows_traffic.log 2>&1
echo "rows traffic rc=$?" > $out/ncu_rows_status.txt
$C1 > $out/plain_rows_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:kvx_move_any_kernel -s 6 -c 1 \
    -o $out/${tag}_rows_c1 $C1 > $out/ncu_rows_full.log 2>&1
echo "rows full rc=$?" >> $out/ncu_rows_status.txt
