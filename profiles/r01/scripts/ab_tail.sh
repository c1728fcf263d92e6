timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k_sweep or strict or iterate or golden or config_G" > gpurun_out/pytest_tail.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tail.log
Q="--no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
for kk in 32 8 128; do
  timeout 300 python bench.py $Q --k $kk > gpurun_out/t_R${kk}_base.log 2>&1
  ARROW_SEG_YPF=1 timeout 300 python bench.py $Q --k $kk > gpurun_out/t_R${kk}_ypf.log 2>&1
  ARROW_TAIL_ATOMIC=1 timeout 300 python bench.py $Q --k $kk > gpurun_out/t_R${kk}_atomic.log 2>&1
done
timeout 300 python bench.py $Q --config G > gpurun_out/t_G_base.log 2>&1
ARROW_SEG_YPF=1 timeout 300 python bench.py $Q --config G > gpurun_out/t_G_ypf.log 2>&1
ARROW_TAIL_ATOMIC=1 timeout 300 python bench.py $Q --config G > gpurun_out/t_G_atomic.log 2>&1
