timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_dist4.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_dist4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29721 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29722 bench.py --gpus 4 --steps 20 --warmup 5 --k 32 > gpurun_out/bench_n4_k32.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29723 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2b.log 2>&1
