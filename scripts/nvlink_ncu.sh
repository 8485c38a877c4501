#!/usr/bin/env bash
# NVLink byte counters of the kvx movers (gpurun --gpus 2): one process drives
# both GPUs (scripts/nvlink_1proc.py), so ncu can profile it.  Each ncu command
# follows the same command run without ncu.
set -u
tag=${1:-r02}
out=gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum"
for pm in "disjoint push" "oneway pull" "oneway push"; do
  set -- $pm
  P="python scripts/nvlink_1proc.py --placement $1 --move $2 --reps 1"
  timeout 600 python scripts/nvlink_1proc.py --placement $1 --move $2 --reps 5 --verify >> $out/${tag}_nvlink_1proc.jsonl 2>> $out/${tag}_nvlink_1proc.err
  echo "$1 $2 plain rc=$?" >> $out/${tag}_nvlink_ncu_status.txt
  timeout 900 ncu --metrics $M --clock-control none -k regex:kvx_bulk_kernel --csv \
      --log-file $out/${tag}_nvlink_ncu_$1_$2.csv $P > $out/${tag}_nvlink_ncu_$1_$2.log 2>&1
  echo "$1 $2 ncu rc=$?" >> $out/${tag}_nvlink_ncu_status.txt
done
