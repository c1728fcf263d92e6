#!/bin/bash
# bench sweep: one JSON line per setting (quick: no CPU baseline, e2e, iterate or cuSPARSE)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-s}
mkdir -p $OUT
Q="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
IFS=';' read -ra RUNS <<< "$SWEEP"
i=0
for args in "${RUNS[@]}"; do
  timeout 600 python bench.py $Q $args > $OUT/run$i.jsonl 2> $OUT/run$i.err
  python - "$OUT/run$i.jsonl" "$args" <<'PY'
import json,sys
try:
    d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][-1]
    print(f"{sys.argv[2]:45s} {d['ms_per_step']:8.4f} ms  {d['value']:9.1f} GFLOP/s  launches {d['per_launch_ms']}  clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
  i=$((i+1))
done
