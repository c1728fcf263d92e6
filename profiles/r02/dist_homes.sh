#!/bin/bash
# home-aware arrangement (R25) on N GPUs: parity (GPU decomposer + distributed) and bench lines
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-homes}
mkdir -p $OUT
N=$(nvidia-smi -L | wc -l)
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_decompose.py -q -x -p no:cacheprovider > $OUT/pytest_gd.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gd.log
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider > $OUT/pytest_dist.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_dist.log
tail -n 2 $OUT/pytest_gd.log $OUT/pytest_dist.log
run() {  # name, bench args
  local name=$1; shift
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
     bench.py --gpus $N --steps 20 --warmup 5 --e2e-steps 0 --no-lib-baseline "$@" > $OUT/bench_n${N}_$name.jsonl 2> $OUT/bench_n${N}_$name.err
  python - $OUT/bench_n${N}_$name.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d=json.loads(l); print(sys.argv[1], d["ms_per_step"], d["value"], d["config"].get("levels"), d["config"].get("sum_n_i"), (d.get("nvlink") or {}).get("bytes_per_gpu_per_direction_max"), d.get("decompose_seconds"), d.get("clocks"))
PY
}
trace() {  # name, bench args: a short run with the per-phase trace (host-synchronised; not a bench value)
  local name=$1; shift
  ARROW_DIST_TRACE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
     bench.py --gpus $N --steps 3 --warmup 3 --e2e-steps 0 --no-lib-baseline --no-cpu-baseline "$@" > $OUT/trace_n${N}_$name.jsonl 2> $OUT/trace_n${N}_$name.err
  grep "arrow dist rank" $OUT/trace_n${N}_$name.err | tail -$N
}
run k128 --k 128
run k128_hl1 --k 128 --home-aware --home-levels 1 --gpu-decompose
run k128_hl2 --k 128 --home-aware --home-levels 2 --gpu-decompose
run k128_nccl --k 128 --transport nccl
run k128_strict --k 128 --band strict
run k32 --k 32
run k32_hl1 --k 32 --home-aware --home-levels 1 --gpu-decompose
trace k128 --k 128
trace k128_hl1 --k 128 --home-aware --home-levels 1 --gpu-decompose
