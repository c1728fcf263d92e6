# A/B of single-GPU K-A switches on config R (usage: VARS="ARROW_X=0 ARROW_X=1" bash profiles/ab_single.sh)
[ "${TEST:-1}" = "1" ] && timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for v in ${VARS:-NONE=0}; do
env $v timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline ${BENCH_ARGS:-} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['roofline']['frac'], d['kernel_ms_per_step'])"
done
