python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --k 32 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('k32', d['ms_per_step'], d['roofline']['frac'], d['kernel_ms_per_step'])"
BENCH="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
ncu --set full --clock-control none --import-source on -k regex:k_seg32 -s 1 -c 1 -o gpurun_out/prof_l1 -f $BENCH > gpurun_out/ncu_l1.log 2>&1
ncu -i gpurun_out/prof_l1.ncu-rep --page details --csv > gpurun_out/prof_l1_details.csv 2>&1
ncu -i gpurun_out/prof_l1.ncu-rep --page raw --csv > gpurun_out/prof_l1_raw.csv 2>&1
