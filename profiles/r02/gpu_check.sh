#!/bin/bash
# round-2 GPU check: parity suite, then the default bench line (short) and per-level K-A times
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r02
export OUT=gpurun_out/r02/${TAG:-a}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline > $OUT/bench_R128.jsonl 2> $OUT/bench_R128.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline --k 32 > $OUT/bench_R32.jsonl 2> $OUT/bench_R32.err
tail -3 $OUT/pytest.log
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ.get("OUT","gpurun_out/r02/a")+"/bench_*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["ms_per_step"], d["value"], d["roofline"]["ms_per_step"], d["hbm_roofline"]["frac_of_measured"])
PY
