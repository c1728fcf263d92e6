# Usage (GPU box, >= 4 GPUs): bash profiles/dist_trace.sh -- per-phase traces of the distributed step
timeout 300 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/dist_t4.log 2>&1; tail -1 gpurun_out/dist_t4.log
for G in ${GS:-2 4}; do
for pk in ${PACKS:-compute comm}; do
  ARROW_DIST_PACK=$pk ARROW_DIST_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
    --master-addr 127.0.0.1 --master-port 2951$G bench.py --gpus $G --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
    > gpurun_out/b${G}_$pk.log 2>&1
  echo "== G=$G pack=$pk"; grep -v "^\[arrow dist" gpurun_out/b${G}_$pk.log | tail -1 | grep -o '"ms_per_step": [0-9.]*'
  grep "^\[arrow dist" gpurun_out/b${G}_$pk.log | tail -$G | cut -c1-420
done; done
