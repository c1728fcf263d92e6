timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/verify_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/verify_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/verify_smoke.log 2>&1
/usr/bin/time -v timeout 600 python bench.py > gpurun_out/verify_R128.log 2> gpurun_out/verify_R128.time
timeout 600 python bench.py --impl reference > gpurun_out/verify_ref.log 2>&1
