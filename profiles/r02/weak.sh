#!/bin/bash
# weak scaling (§8(d) config 5, Fig. 6 analogue): RMAT scale 21 + log2(G) at G GPUs, b = n/256, fp32;
# the G = 1 point (S21) is in profiles/r02/S/.  G = N of this box.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export OUT=gpurun_out/r02/${TAG:-weak}
mkdir -p $OUT
N=$(nvidia-smi -L | wc -l)
case $N in 2) C=R;; 4) C=S23;; *) C=S21;; esac
python -c "import paper_2402_19364_b200 as ab; ab.lib()" > $OUT/build.log 2>&1
for k in 128 32 8; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29557 \
     bench.py --gpus $N --config $C --k $k --steps 20 --warmup 5 --e2e-steps 0 --no-lib-baseline --gpu-decompose ${EXTRA} \
     > $OUT/weak_n${N}_${C}_k$k${SUF}.jsonl 2> $OUT/weak_n${N}_${C}_k$k${SUF}.err
  python - $OUT/weak_n${N}_${C}_k$k${SUF}.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d=json.loads(l); print(sys.argv[1], d["ms_per_step"], d["value"], d["config"]["workload"], (d.get("nvlink") or {}).get("bytes_per_gpu_per_direction_max"), d.get("clocks"))
PY
done
