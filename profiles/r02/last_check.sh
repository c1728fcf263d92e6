#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/last
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
tail -n 2 $OUT/pytest.log $OUT/smoke.log
python - <<'PY'
import json
for l in open("gpurun_out/r02/last/bench_default.jsonl"):
    if l.startswith("{"):
        d=json.loads(l); print(d["ms_per_step"], d["value"], d["roofline"]["frac"], d["e2e"]["value"], d["create_seconds"], d["clocks"])
PY
