B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0 --k 32"
timeout 300 $B > gpurun_out/plain_k32b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_segsmall -s 0 -c 2 \
    -o gpurun_out/prof_k32 -f $B > gpurun_out/ncu_full_k32.log 2>&1
