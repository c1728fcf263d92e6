#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-det2}
mkdir -p $OUT
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
Q="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
for rep in 1 2; do
  timeout 600 python bench.py $Q --flags 2 > $OUT/det128_$rep.jsonl 2> $OUT/det128_$rep.err
  timeout 600 python bench.py $Q --flags 2 --head-chunk 64 > $OUT/det64_$rep.jsonl 2> $OUT/det64_$rep.err
  timeout 600 python bench.py $Q --flags 2 --head-chunk 256 > $OUT/det256_$rep.jsonl 2> $OUT/det256_$rep.err
  timeout 600 python bench.py $Q > $OUT/main_$rep.jsonl 2> $OUT/main_$rep.err
done
timeout 600 python bench.py $Q --flags 2 --k 32 > $OUT/det_k32.jsonl 2> $OUT/det_k32.err
timeout 600 python bench.py $Q --k 32 > $OUT/main_k32.jsonl 2> $OUT/main_k32.err
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "determin or host or iterate" -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ["OUT"]+"/*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["ms_per_step"], d.get("per_launch_ms"))
PY
tail -n 2 $OUT/pytest.log
