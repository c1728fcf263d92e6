#!/bin/bash
# tile-window size (rows) at k = 8 / 32 / 128, config R, one GPU
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-win}
mkdir -p $OUT
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
Q="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
for k in 32 8 128; do
  for w in 16384 32768 65536 131072; do
    timeout 600 python bench.py $Q --k $k --window-rows $w > $OUT/k${k}_w$w.jsonl 2> $OUT/k${k}_w$w.err
  done
done
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ["OUT"]+"/*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["ms_per_step"], d.get("per_launch_ms"))
PY
