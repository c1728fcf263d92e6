# final round-1 evidence: tests, smoke, bench lines, ncu launch lists + one --set full capture
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final_R128.log 2>&1
timeout 600 python bench.py --k 32 --no-cpu-baseline > gpurun_out/final_R32.log 2>&1
timeout 300 python bench.py --config G --no-cpu-baseline > gpurun_out/final_G.log 2>&1
timeout 300 python bench.py --config T --no-cpu-baseline > gpurun_out/final_T.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_seg|k_zero|k_tail" --csv --log-file gpurun_out/final_launches_R_k128.csv $B > gpurun_out/final_ncu_list128.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_seg|k_zero|k_tail" --csv --log-file gpurun_out/final_launches_R_k32.csv $B --k 32 > gpurun_out/final_ncu_list32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_seg32 -s 0 -c 2 \
    -o gpurun_out/final_prof_R128 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0 > gpurun_out/final_ncu_full.log 2>&1
Q="--no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
ARROW_SEG_DEFER=1 timeout 300 python bench.py $Q > gpurun_out/final_R128_defer.log 2>&1
timeout 300 python bench.py $Q --band strict > gpurun_out/final_R128_strict.log 2>&1
