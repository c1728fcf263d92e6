#!/bin/bash
# distributed: level-0 window 65536 (default) vs 16384, R k=128 at N = 2 and 4; parity
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-win_dist}
mkdir -p $OUT
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider > $OUT/pytest_dist.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_dist.log
Q="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
for N in 4 2; do
  for rep in 1 2; do
    for w in 0 16384; do
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N \
         bench.py --gpus $N $Q --window-rows $w > $OUT/n${N}_w${w}_$rep.jsonl 2> $OUT/n${N}_w${w}_$rep.err
    done
  done
done
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ["OUT"]+"/*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["ms_per_step"], d["config"].get("window_rows"))
PY
tail -n 2 $OUT/pytest_dist.log
