Q="--no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
ARROW_TAIL_STAGE=1 ARROW_TAIL_STAGE_VERBOSE=1 timeout 300 python bench.py $Q > gpurun_out/s2_R128_on.log 2>&1
timeout 300 python bench.py $Q > gpurun_out/s2_R128_off.log 2>&1
ARROW_TAIL_STAGE=1 ARROW_SEG_BS=8 timeout 300 python bench.py $Q > gpurun_out/s2_R128_on_bs8.log 2>&1
ARROW_SEG_BS=8 timeout 300 python bench.py $Q > gpurun_out/s2_R128_off_bs8.log 2>&1
