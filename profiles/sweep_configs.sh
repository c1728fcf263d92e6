# Per-config bench lines (1 GPU): bash profiles/sweep_configs.sh > gpurun_out/sweep.jsonl
for a in "--config G" "--config T" "--config R --k 32" "--config R --k 8" "--config R --k 128 --order permuted"; do
  timeout 300 python bench.py $a --steps 20 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1
done
