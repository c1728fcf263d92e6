# config W (web-like 2^24, k=32) at G = 2 and 4 (P2P transport), with the 1D and 1.5D comparators
for G in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2952$G bench.py --gpus $G --config W --steps 10 --warmup 3 > gpurun_out/W_n$G.jsonl 2> gpurun_out/W_n$G.err
  echo "G=$G exit $?"
done
