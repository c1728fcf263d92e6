#!/bin/bash
# Usage (on the GPU box, via gpurun): bash profiles/run_ncu.sh <tag> [bench args...]
# 1) plain bench run (must exit 0), 2) launch list of every kernel with device time and DRAM
# bytes, 3) one --set full capture of the level-0 K-A launch (the dominant kernel).
set -e
tag=$1; shift
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 $*"
KA=${KA_REGEX:-k_segments}
$BENCH > gpurun_out/plain_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_seg|k_rec|k_stream|k_tma|k_zero|k_head|k_rows|k_gather" \
    --csv --log-file gpurun_out/launches_$tag.csv $BENCH > gpurun_out/ncu_list_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$KA -s 0 -c 1 \
    -o gpurun_out/prof_$tag -f $BENCH > gpurun_out/ncu_full_$tag.log 2>&1
