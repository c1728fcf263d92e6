#!/bin/bash
# home_levels re-check with the 4-blocks/SM distributed kernels, R k=128
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-hl2}
mkdir -p $OUT
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
Q="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
for N in 2 4; do
  for hl in 1 2 3; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N \
       bench.py --gpus $N $Q --home-levels $hl > $OUT/n${N}_hl$hl.jsonl 2> $OUT/n${N}_hl$hl.err
  done
done
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ["OUT"]+"/*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["ms_per_step"], d["config"].get("arrangement"))
PY
