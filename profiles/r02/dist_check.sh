#!/bin/bash
# multi-GPU check: distributed parity (P2P + NCCL transports, block and strict band) and bench lines at N GPUs
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-dist}
mkdir -p $OUT
N=$(nvidia-smi -L | wc -l)
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dist.py -q > $OUT/pytest_dist.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_dist.log
tail -3 $OUT/pytest_dist.log
run() {  # name, bench args
  local name=$1; shift
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
     bench.py --gpus $N --steps 20 --warmup 5 --e2e-steps 0 "$@" > $OUT/bench_n${N}_$name.jsonl 2> $OUT/bench_n${N}_$name.err
  python - $OUT/bench_n${N}_$name.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d=json.loads(l); print(sys.argv[1], d["ms_per_step"], d["value"], d["config"].get("levels"), (d.get("library_baseline") or {}).get("ms_per_step"), (d.get("baseline_1_5d") or {}).get("ms_per_step"), (d.get("nvlink") or {}).get("bytes_per_gpu_per_direction_max"), d.get("clocks"))
PY
}
run k128 --k 128 ${EXTRA}
run k32 --k 32 ${EXTRA}
run k128_nccl --k 128 --transport nccl ${EXTRA}
run k128_strict --k 128 --band strict ${EXTRA}
run k128_strict_nccl --k 128 --band strict --transport nccl ${EXTRA}
