#!/bin/bash
# GPU decomposer parity + timing, deterministic-flag test (one gpurun call)
mkdir -p gpurun_out/r02/gd
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > gpurun_out/r02/gd/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_decompose.py -m gpu -x -q -s -p no:cacheprovider > gpurun_out/r02/gd/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/gd/pytest.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "deterministic" -p no:cacheprovider > gpurun_out/r02/gd/det.log 2>&1
echo "det rc=$?" >> gpurun_out/r02/gd/det.log
