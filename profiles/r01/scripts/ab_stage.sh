timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_stage.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_stage.log
Q="--no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
timeout 300 python bench.py $Q > gpurun_out/s_R128_on.log 2>&1
ARROW_TAIL_STAGE=0 timeout 300 python bench.py $Q > gpurun_out/s_R128_off.log 2>&1
timeout 300 python bench.py $Q --k 64 --dtype f64 > gpurun_out/s_R64d_on.log 2>&1
ARROW_TAIL_STAGE=0 timeout 300 python bench.py $Q --k 64 --dtype f64 > gpurun_out/s_R64d_off.log 2>&1
timeout 300 python bench.py $Q --k 256 > gpurun_out/s_R256_on.log 2>&1
ARROW_TAIL_STAGE=0 timeout 300 python bench.py $Q --k 256 > gpurun_out/s_R256_off.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_seg|k_zero|k_tail" --csv --log-file gpurun_out/launches_stage_R_k128.csv $B > gpurun_out/ncu_stage.log 2>&1
