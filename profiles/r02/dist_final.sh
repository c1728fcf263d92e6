#!/bin/bash
# multi-GPU closing check at N GPUs: parity, then the bench defaults (home-aware, GPU decomposition)
# and the variants they replace
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-dist_final}
mkdir -p $OUT
N=$(nvidia-smi -L | wc -l)
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider > $OUT/pytest_dist.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_dist.log
tail -n 2 $OUT/pytest_dist.log
run() {
  local name=$1; shift
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
     bench.py --gpus $N "$@" > $OUT/bench_n${N}_$name.jsonl 2> $OUT/bench_n${N}_$name.err
  python - $OUT/bench_n${N}_$name.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d=json.loads(l); print(sys.argv[1], d["ms_per_step"], d["value"], d["config"].get("levels"), d["config"].get("arrangement"), (d.get("nvlink") or {}).get("bytes_per_gpu_per_direction_max"), (d.get("e2e") or {}).get("value"), d.get("clocks"))
PY
}
run default_k128 --steps 20 --warmup 5
run default_k32 --steps 20 --warmup 5 --k 32 --e2e-steps 0 --no-lib-baseline
run plain_k128 --steps 20 --warmup 5 --no-home-aware --e2e-steps 0 --no-lib-baseline
run strict_k128 --steps 20 --warmup 5 --band strict --e2e-steps 0 --no-lib-baseline
ARROW_DIST_TRACE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
     bench.py --gpus $N --steps 3 --warmup 3 --e2e-steps 0 --no-lib-baseline --no-cpu-baseline > $OUT/trace.jsonl 2> $OUT/trace.err
grep "arrow dist rank" $OUT/trace.err | tail -$N
