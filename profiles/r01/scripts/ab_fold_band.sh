set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu2.log
Q="--no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
timeout 300 python bench.py $Q > gpurun_out/b2_R_fold.log 2>&1
ARROW_KZ_FOLD=0 timeout 300 python bench.py $Q > gpurun_out/b2_R_nofold.log 2>&1
timeout 300 python bench.py $Q --band strict > gpurun_out/b2_R_strict.log 2>&1
timeout 300 python bench.py $Q --config G > gpurun_out/b2_G_fold.log 2>&1
ARROW_KZ_FOLD=0 timeout 300 python bench.py $Q --config G > gpurun_out/b2_G_nofold.log 2>&1
timeout 300 python bench.py $Q --config G --band strict > gpurun_out/b2_G_strict.log 2>&1
timeout 300 python bench.py $Q --k 32 > gpurun_out/b2_R32_fold.log 2>&1
ARROW_KZ_FOLD=0 timeout 300 python bench.py $Q --k 32 > gpurun_out/b2_R32_nofold.log 2>&1
