#!/bin/bash
# A/B: Y rows of level >= 1 read-modify-writes loaded L2-only (ld.global.cg; build/v7) vs the head
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-v7}
mkdir -p $OUT
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
(cd build/v7 && python -c "import paper_2402_19364_b200 as ab; ab.lib()") >> $OUT/build.log 2>&1
Q="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
for rep in 1 2 3; do
  timeout 600 python bench.py $Q > $OUT/main_$rep.jsonl 2> $OUT/main_$rep.err
  (cd build/v7 && timeout 600 python bench.py $Q > ../../$OUT/v7_$rep.jsonl 2> ../../$OUT/v7_$rep.err)
done
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ["OUT"]+"/*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["ms_per_step"], d.get("per_launch_ms"))
PY
