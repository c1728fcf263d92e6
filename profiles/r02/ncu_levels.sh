#!/bin/bash
# ncu --set full of the first two K-A launches (level 0, level 1) of config R k=128 (one GPU)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-n}
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline ${BENCH_ARGS}"
$CMD > $OUT/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_ka} -c ${NCOUNT:-2} -o $OUT/prof $CMD > $OUT/ncu.log 2>&1
echo "rc=$?"
tail -3 $OUT/ncu.log
