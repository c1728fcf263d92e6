nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gbw2 profiles/gather_bw2.cu && timeout 120 /tmp/gbw2 > gpurun_out/gather_bw2.txt 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0 --k 32"
timeout 300 $B > gpurun_out/plain_k32.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_seg|k_zero" --csv --log-file gpurun_out/launches_R_k32.csv $B > gpurun_out/ncu_k32.log 2>&1
