#!/bin/bash
# A/B at N = 4 and 2: distributed K-A kernels at 4 blocks/SM (build/v8; 64 / 60 registers, no spills)
# vs 3 blocks/SM (the head)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-v8}
mkdir -p $OUT
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
(cd build/v8 && python -c "import paper_2402_19364_b200 as ab; ab.lib()") >> $OUT/build.log 2>&1
Q="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
for N in 4 2; do
  for rep in 1 2; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N \
       bench.py --gpus $N $Q > $OUT/main_n${N}_$rep.jsonl 2> $OUT/main_n${N}_$rep.err
    (cd build/v8 && timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N \
       bench.py --gpus $N $Q > ../../$OUT/v8_n${N}_$rep.jsonl 2> ../../$OUT/v8_n${N}_$rep.err)
  done
done
(cd build/v8 && timeout 1200 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider > ../../$OUT/v8_pytest_dist.log 2>&1; echo "pytest rc=$?" >> ../../$OUT/v8_pytest_dist.log)
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ["OUT"]+"/*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["ms_per_step"])
PY
tail -n 2 $OUT/v8_pytest_dist.log
