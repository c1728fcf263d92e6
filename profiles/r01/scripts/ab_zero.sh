Q="--no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
for kk in 32 8 128; do
  timeout 300 python bench.py $Q --k $kk > gpurun_out/z_R${kk}_fold.log 2>&1
  ARROW_KZ_FOLD=0 timeout 300 python bench.py $Q --k $kk > gpurun_out/z_R${kk}_nofold.log 2>&1
done
timeout 300 python bench.py $Q --config G > gpurun_out/z_G_fold.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0 --k 32"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_segsmall -s 0 -c 1 \
    -o gpurun_out/prof_k32b -f $B > gpurun_out/ncu_full_k32b.log 2>&1
