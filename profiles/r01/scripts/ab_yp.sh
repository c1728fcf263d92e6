# A/B: Y-row preload for levels >= 1 in k_seg32 (ARROW_SEG32_YP=1) vs default; GPU parity with it on;
# config W (web-like 2^24) at N=1.  Run from the repo root through gpurun.
Q="--no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
ARROW_SEG32_YP=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/yp_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/yp_pytest.log
for r in 1 2; do
  timeout 300 python bench.py $Q > gpurun_out/yp_R128_off_$r.log 2>&1
  ARROW_SEG32_YP=1 timeout 300 python bench.py $Q > gpurun_out/yp_R128_on_$r.log 2>&1
done
ARROW_SEG32_YP=1 timeout 300 python bench.py $Q --k 64 > gpurun_out/yp_R64_on.log 2>&1
timeout 300 python bench.py $Q --k 64 > gpurun_out/yp_R64_off.log 2>&1
ARROW_SEG32_YP=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/yp_launches_on.csv python bench.py $Q --steps 2 --warmup 3 > /dev/null 2>&1
timeout 900 python bench.py --config W --steps 10 --warmup 3 > gpurun_out/W_n1.log 2>&1
echo done
