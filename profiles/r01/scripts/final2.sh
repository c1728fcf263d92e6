# round-1 closing evidence (2 GPUs: single-GPU tests + world-2 multi-GPU parity): tests, smoke,
# default bench line (cpu_baseline incl. one-core), reference arm, ncu launch list, one --set full capture
mkdir -p gpurun_out/f2
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/f2/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/f2/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f2/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/f2/R128.jsonl 2> gpurun_out/f2/R128.err
timeout 600 python bench.py --k 32 --no-cpu-baseline > gpurun_out/f2/R32.jsonl 2> gpurun_out/f2/R32.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f2/reference.jsonl 2> gpurun_out/f2/reference.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/f2/launches_R_k128.csv $B > gpurun_out/f2/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_seg32 -s 0 -c 1 \
    -o gpurun_out/f2/full_R128_L0 -f $B > gpurun_out/f2/ncu_full.log 2>&1
ncu -i gpurun_out/f2/full_R128_L0.ncu-rep --page details --csv > gpurun_out/f2/full_R128_L0_details.csv 2>/dev/null
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 > gpurun_out/f2/n2_R128.jsonl 2> gpurun_out/f2/n2_R128.err
echo done
