# arrow_spmm_host_batch: parity tests, then the default bench line (e2e = pipelined batch) and k=32
mkdir -p gpurun_out/hb
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/hb/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/hb/pytest.log
timeout 600 python bench.py > gpurun_out/hb/R128.jsonl 2> gpurun_out/hb/R128.err
timeout 600 python bench.py --k 32 --no-cpu-baseline > gpurun_out/hb/R32.jsonl 2> gpurun_out/hb/R32.err
timeout 300 python bench.py --config G --no-cpu-baseline > gpurun_out/hb/G.jsonl 2> gpurun_out/hb/G.err
echo done
