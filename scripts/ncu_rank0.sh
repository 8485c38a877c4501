#!/usr/bin/env bash
# torchrun --no-python wrapper: rank 0 runs under ncu with NVLink + DRAM byte
# counters on the kvx bulk mover, the other ranks run plainly.
#   python -m torch.distributed.run ... --no-python scripts/ncu_rank0.sh <csv> <skip> <count> bench.py ARGS
csv=$1; skip=$2; count=$3; shift 3
if [ "${LOCAL_RANK:-0}" = "0" ]; then
  exec ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum \
       --clock-control none -k regex:kvx_bulk_kernel -s "$skip" -c "$count" --csv --log-file "$csv" python "$@"
else
  exec python "$@"
fi
