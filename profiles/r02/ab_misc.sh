#!/bin/bash
# PCIe copy probe; deterministic mode after the head-chunk fix; A/B of 5 blocks/SM for levels >= 1 (build/v5)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-misc}
mkdir -p $OUT
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
timeout 300 python profiles/r02/pcie_bw.py > $OUT/pcie.jsonl 2> $OUT/pcie.err
Q="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
timeout 600 python bench.py $Q --flags 2 > $OUT/det.jsonl 2> $OUT/det.err
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k deterministic -p no:cacheprovider > $OUT/det_pytest.log 2>&1
for rep in 1 2; do
  timeout 600 python bench.py $Q > $OUT/main_$rep.jsonl 2> $OUT/main_$rep.err
  (cd build/v5 && timeout 600 python bench.py $Q > ../../$OUT/v5_$rep.jsonl 2> ../../$OUT/v5_$rep.err)
done
python - <<'PY'
import json,glob,os
o=os.environ["OUT"]
for l in open(o+"/pcie.jsonl"): print(l.strip())
for f in sorted(glob.glob(o+"/*.jsonl")):
    if "pcie" in f: continue
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["ms_per_step"], d.get("per_launch_ms"))
PY
tail -n 2 $OUT/det_pytest.log
