set -x
for b in 4 8 16 32; do
  TPR_K1_DYNAMIC=$b timeout 400 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/ab8_cfg2_b${b}.json 2>&1
  TPR_K1_DYNAMIC=$b timeout 400 python bench.py --config 3 --no-cpu --no-e2e --steps 8 > gpurun_out/ab8_cfg4_b${b}.json 2>&1
  TPR_K1_DYNAMIC=$b timeout 400 python tools/sweep.py --modes trace --only 4:8:256,1:2:16 --reps 4 --k1-reps 4 --out gpurun_out/ab8_trace_b${b}.jsonl > /dev/null 2>&1
done
TPR_K1_DYNAMIC=8 timeout 400 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/ab8_cfg2_b8_again.json 2>&1
