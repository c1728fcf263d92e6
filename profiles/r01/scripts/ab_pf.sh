timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or layout or strict or iterate or golden" > gpurun_out/pytest_pf.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_pf.log
Q="--no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
for kk in 128 32 8; do
  timeout 300 python bench.py $Q --k $kk > gpurun_out/pf_R${kk}_on.log 2>&1
  ARROW_SEG_PF=0 timeout 300 python bench.py $Q --k $kk > gpurun_out/pf_R${kk}_off.log 2>&1
done
timeout 300 python bench.py $Q --config G > gpurun_out/pf_G_on.log 2>&1
ARROW_SEG_PF=0 timeout 300 python bench.py $Q --config G > gpurun_out/pf_G_off.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_seg|k_zero" --csv --log-file gpurun_out/launches_pf_R_k32.csv $B --k 32 > gpurun_out/ncu_pf32.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_seg|k_zero" --csv --log-file gpurun_out/launches_pf_R_k128.csv $B > gpurun_out/ncu_pf128.log 2>&1
