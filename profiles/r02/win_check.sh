#!/bin/bash
# the bench's k-dependent window default against 16384 rows: R k=64/32, G; and N=4 k=32
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-win2}
mkdir -p $OUT
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
Q="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
for a in "--k 64" "--k 32" "--config G"; do
  n=$(echo $a | tr -d ' -')
  timeout 600 python bench.py $Q $a > $OUT/${n}_default.jsonl 2> $OUT/${n}_default.err
  timeout 600 python bench.py $Q $a --window-rows 16384 > $OUT/${n}_w16384.jsonl 2> $OUT/${n}_w16384.err
done
for w in 0 16384; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 \
     bench.py --gpus 4 $Q --k 32 --window-rows $w > $OUT/n4_k32_w$w.jsonl 2> $OUT/n4_k32_w$w.err
done
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ["OUT"]+"/*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["ms_per_step"], d["config"].get("window_rows"), d.get("per_launch_ms"))
PY
