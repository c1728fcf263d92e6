#!/bin/bash
# level-0 window 65536 by default (levels >= 1 16384) vs 16384 everywhere, R k=128 (3 reps each), and
# the parity suite
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-win3}
mkdir -p $OUT
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
Q="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
for rep in 1 2 3; do
  timeout 600 python bench.py $Q > $OUT/default_$rep.jsonl 2> $OUT/default_$rep.err
  timeout 600 python bench.py $Q --window-rows 16384 > $OUT/w16384_$rep.jsonl 2> $OUT/w16384_$rep.err
done
timeout 600 python bench.py $Q --flags 2 > $OUT/det.jsonl 2> $OUT/det.err
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ["OUT"]+"/*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["ms_per_step"], d["config"].get("window_rows"), d.get("per_launch_ms"))
PY
tail -n 2 $OUT/pytest.log
