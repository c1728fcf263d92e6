#!/bin/bash
# closing multi-GPU evidence on a 4-GPU box: distributed parity, bench defaults at N = 2 and 4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-close4}
mkdir -p $OUT
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider > $OUT/pytest_dist.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_dist.log
tail -n 2 $OUT/pytest_dist.log
for N in 2 4; do
  for k in 128 32; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N \
       bench.py --gpus $N --steps 20 --warmup 5 --k $k $( [ $k = 32 ] && echo "--e2e-steps 0 --no-lib-baseline" ) > $OUT/bench_n${N}_k$k.jsonl 2> $OUT/bench_n${N}_k$k.err
    python - $OUT/bench_n${N}_k$k.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d=json.loads(l); print(sys.argv[1], d["ms_per_step"], d["value"], d["config"].get("arrangement"), (d.get("nvlink") or {}).get("bytes_per_gpu_per_direction_max"), (d.get("e2e") or {}).get("value"), (d.get("library_baseline") or {}).get("ms_per_step"), (d.get("baseline_1_5d") or {}).get("ms_per_step"), d.get("decompose_seconds"), d.get("clocks"))
PY
  done
done
