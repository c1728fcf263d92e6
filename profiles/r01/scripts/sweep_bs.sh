start=$(date +%s); timeout 600 python bench.py > gpurun_out/verify_R128.log 2>&1; echo "bench wall s: $(( $(date +%s) - start ))" > gpurun_out/verify_R128.time
Q="--no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
timeout 300 python bench.py $Q > gpurun_out/bs_R128_base.log 2>&1
for bs in 8 32; do ARROW_SEG_BS_TAIL=$bs timeout 300 python bench.py $Q > gpurun_out/bs_R128_tail$bs.log 2>&1; done
for bs in 12 24 32; do ARROW_SEG_BS=$bs timeout 300 python bench.py $Q > gpurun_out/bs_R128_all$bs.log 2>&1; done
for w in 8192 32768; do timeout 300 python bench.py $Q --window-rows $w > gpurun_out/w_R128_$w.log 2>&1; done
