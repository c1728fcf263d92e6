#!/bin/bash
# round-2 closing evidence on one B200: parity suite, smoke, bench lines, launch lists with DRAM bytes,
# ncu --set full of the first two K-A launches (level 0, level 1) at config R k=128
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-final}
mkdir -p $OUT
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
Q="--steps 20 --warmup 5 --e2e-steps 0 --iterate 0"
timeout 600 python bench.py $Q --k 32 > $OUT/bench_R32.jsonl 2> $OUT/bench_R32.err
timeout 600 python bench.py $Q --no-cpu-baseline --no-lib-baseline --flags 2 > $OUT/bench_R128_det.jsonl 2> $OUT/bench_R128_det.err
timeout 600 python bench.py $Q --no-cpu-baseline --no-lib-baseline --band strict > $OUT/bench_R128_strict.jsonl 2> $OUT/bench_R128_strict.err
timeout 600 python bench.py $Q --config G > $OUT/bench_G.jsonl 2> $OUT/bench_G.err
timeout 600 python bench.py $Q --config T > $OUT/bench_T.jsonl 2> $OUT/bench_T.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.jsonl 2> $OUT/bench_reference.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --iterate 0 --no-lib-baseline"
for k in 128 32; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_" \
      --csv --log-file $OUT/launches_R_k$k.csv $B --k $k > $OUT/ncu_list_k$k.log 2>&1
done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ka -c 2 -o $OUT/prof_R128 -f $B > $OUT/ncu_full.log 2>&1
echo "ncu rc=$?" >> $OUT/ncu_full.log
tail -n 2 $OUT/pytest.log $OUT/smoke.log
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ["OUT"]+"/bench_*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d.get("ms_per_step"), d.get("value"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), d.get("clocks"))
PY
