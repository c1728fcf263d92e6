nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rmw profiles/rmw_bw.cu && timeout 120 /tmp/rmw > gpurun_out/rmw_bw.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_ffma.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ffma.log
Q="--no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
for kk in 32 8 16 64; do timeout 300 python bench.py $Q --k $kk > gpurun_out/f_R${kk}.log 2>&1; done
timeout 300 python bench.py $Q --config G > gpurun_out/f_G.log 2>&1
timeout 300 python bench.py $Q --config T > gpurun_out/f_T.log 2>&1
timeout 400 python bench.py > gpurun_out/f_R128_full.log 2>&1
