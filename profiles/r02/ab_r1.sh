#!/bin/bash
# same-box A/B against the round-1 head (git worktree build/r1ref at ff917c1, built in-tree) and
# the round-2 variants given in SWEEP (';'-separated bench.py argument lists)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-ab}
mkdir -p $OUT
Q="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
summ() { python - "$1" "$2" <<'PY'
import json,sys
try:
    d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][-1]
    print(f"{sys.argv[2]:36s} {d['ms_per_step']:8.4f} ms {d['value']:9.1f} GFLOP/s per-launch {d.get('per_launch_ms', d.get('kernel_ms_per_step'))}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
}
IFS=';' read -ra RUNS <<< "$SWEEP"
for rep in 1 2; do
  (cd build/r1ref && timeout 600 python bench.py $Q $EXTRA > ../../$OUT/r1_$rep.jsonl 2> ../../$OUT/r1_$rep.err); summ $OUT/r1_$rep.jsonl "round1 $EXTRA"
  i=0
  for args in "${RUNS[@]}"; do
    timeout 600 python bench.py $Q $EXTRA $args > $OUT/r2_${rep}_$i.jsonl 2> $OUT/r2_${rep}_$i.err; summ $OUT/r2_${rep}_$i.jsonl "round2 $EXTRA $args"
    i=$((i+1))
  done
done
