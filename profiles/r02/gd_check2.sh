#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r02/gd2
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > gpurun_out/r02/gd2/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_decompose.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r02/gd2/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02/gd2/pytest.log
timeout 900 python profiles/r02/gd_time.py > gpurun_out/r02/gd2/time.log 2>&1
tail -n 2 gpurun_out/r02/gd2/pytest.log; grep -v "^\[arrow" gpurun_out/r02/gd2/time.log
