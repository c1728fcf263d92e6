#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r02/probe
O=gpurun_out/r02/probe/tma_gather.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tg profiles/r02/tma_gather.cu -lcuda || exit 1
for args in "3 128 0" "1 128 0" "1 32 0"; do
  timeout 60 /tmp/tg $args >> $O 2>&1; rc=$?; echo "args=$args rc=$rc" >> $O
  if [ $rc -ne 0 ]; then break; fi
done
cat $O
