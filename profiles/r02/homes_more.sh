#!/bin/bash
# more home-aware points at N GPUs (config R), then the weak-scaling points (default and home-aware)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-homes_more}
mkdir -p $OUT
N=$(nvidia-smi -L | wc -l)
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
run() {
  local name=$1; shift
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 \
     bench.py --gpus $N --steps 20 --warmup 5 --e2e-steps 0 --no-lib-baseline --gpu-decompose "$@" > $OUT/bench_n${N}_$name.jsonl 2> $OUT/bench_n${N}_$name.err
  python - $OUT/bench_n${N}_$name.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d=json.loads(l); print(sys.argv[1], d["ms_per_step"], d["value"], d["config"].get("levels"), d["config"].get("sum_n_i"), (d.get("nvlink") or {}).get("bytes_per_gpu_per_direction_max"), d.get("clocks"))
PY
}
run k128_hl3 --k 128 --home-aware --home-levels 3
run k128_hl4 --k 128 --home-aware --home-levels 4
run k128_hl2_strict --k 128 --home-aware --home-levels 2 --band strict
run k32_hl2 --k 32 --home-aware --home-levels 2
run k8 --k 8
run k8_hl2 --k 8 --home-aware --home-levels 2
TAG=$TAG bash profiles/r02/weak.sh
TAG=$TAG EXTRA="--home-aware --home-levels 2" SUF=_hl2 bash profiles/r02/weak.sh
