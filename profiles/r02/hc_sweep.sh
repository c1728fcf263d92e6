#!/bin/bash
# head-row chunk (entries per segment) with the round-2 windows, R k=128 and k=32
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-hc}
mkdir -p $OUT
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
Q="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
for rep in 1 2; do
  for k in 128 32; do
    for hc in 16 32 64; do
      timeout 600 python bench.py $Q --k $k --head-chunk $hc > $OUT/k${k}_hc${hc}_$rep.jsonl 2> $OUT/k${k}_hc${hc}_$rep.err
    done
  done
done
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ["OUT"]+"/*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["ms_per_step"], (d.get("per_launch_ms") or [0,0])[1])
PY
