#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r02/probe
O=gpurun_out/r02/probe/tma_unit.txt
: > $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tu profiles/r02/tma_unit.cu -lcuda || exit 1
for args in "0 128" "1 128" "2 128" "1 32" "3 32" "3 128"; do
  timeout 20 /tmp/tu $args >> $O 2>&1; rc=$?; echo "  rc=$rc" >> $O
  if [ $rc -ne 0 ]; then break; fi
done
cat $O
