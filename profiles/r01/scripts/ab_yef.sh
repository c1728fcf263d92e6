# A/B: L2 evict-first policy on the Y read-modify-writes of levels >= 1 (ARROW_SEG32_YEF=1) vs default
mkdir -p gpurun_out/yef
Q="--no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
ARROW_SEG32_YEF=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/yef/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/yef/pytest.log
for r in 1 2 3; do
  timeout 300 python bench.py $Q > gpurun_out/yef/R128_off_$r.jsonl 2>/dev/null
  ARROW_SEG32_YEF=1 timeout 300 python bench.py $Q > gpurun_out/yef/R128_on_$r.jsonl 2>/dev/null
done
echo done
