set -x
for i in 1 2; do
  for d in 0 1; do
    TPR_K1_DYNAMIC=$d timeout 400 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/ab6_cfg2_d${d}_$i.json 2>&1
    TPR_K1_DYNAMIC=$d timeout 400 python bench.py --config 3 --no-cpu --no-e2e --steps 10 > gpurun_out/ab6_cfg4_d${d}_$i.json 2>&1
    TPR_K1_DYNAMIC=$d timeout 400 python tools/sweep.py --modes trace --only 4:8:256,1:2:16 --reps 4 --k1-reps 4 --out gpurun_out/ab6_trace_d${d}_$i.jsonl > /dev/null 2>&1
  done
done
