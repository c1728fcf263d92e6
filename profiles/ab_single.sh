timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for cfg in "1 1" "0 1" "1 0" "0 0"; do set -- $cfg
ARROW_SEG_DEFER=$1 ARROW_KZ_OVERLAP=$2 timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"defer=$1 kz_overlap=$2\", d[\"ms_per_step\"], d[\"roofline\"][\"frac\"], d[\"kernel_ms_per_step\"])"
done
