# round-1 closing run on 4 GPUs: full GPU suite (incl. world-4 multi-GPU parity), smoke, bench N=1 and N=4
mkdir -p gpurun_out/f3
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f3/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/f3/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f3/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/f3/R128.jsonl 2> gpurun_out/f3/R128.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 > gpurun_out/f3/n4_R128.jsonl 2> gpurun_out/f3/n4_R128.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --impl reference --gpus 4 --steps 2 --warmup 3 > gpurun_out/f3/n4_reference.jsonl 2> gpurun_out/f3/n4_reference.err
echo done
