# segments per batch: levels >= 1 (ARROW_SEG_BS_TAIL) and level 0 (ARROW_SEG_BS), config R k=128 / 32
mkdir -p gpurun_out/bst
Q="--no-cpu-baseline --e2e-steps 0 --no-lib-baseline --iterate 0"
for r in 1 2; do
for t in 0 4 8 24 32; do
  ARROW_SEG_BS_TAIL=$t timeout 300 python bench.py $Q > gpurun_out/bst/R128_tail$t.r$r.jsonl 2>/dev/null
done
done
for t in 0 8 32; do
  ARROW_SEG_BS_TAIL=$t timeout 300 python bench.py $Q --k 32 > gpurun_out/bst/R32_tail$t.jsonl 2>/dev/null
done
for b in 24 32; do
  ARROW_SEG_BS=$b ARROW_SEG_BS_TAIL=16 timeout 300 python bench.py $Q > gpurun_out/bst/R128_l0bs$b.jsonl 2>/dev/null
done
echo done
