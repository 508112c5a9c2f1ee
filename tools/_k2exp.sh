set -x
mkdir -p gpurun_out/k2exp
for cfg in 4x16384 6x16384 3x32768 8x8192 12x8192 6x32768; do
  TPR_BULK_K2=$cfg timeout 300 python tools/weight_sweep.py --reps 5 --only 8:2:4,8:2:8,4:2:4,8:4:2,8:8:4 --out gpurun_out/k2exp/ws_$cfg.jsonl > gpurun_out/k2exp/ws_$cfg.log 2>&1
done
timeout 300 python tools/weight_sweep.py --engine vector --reps 5 --only 8:2:4,8:2:8,4:2:4,8:4:2,8:8:4 --out gpurun_out/k2exp/ws_vector.jsonl > gpurun_out/k2exp/ws_vector.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tpr_k2 --launch-skip 2 -c 1 -o gpurun_out/k2exp/k2_fwd_8_2_4 python tools/weight_sweep.py --reps 1 --only 8:2:4 --out gpurun_out/k2exp/ncu_ws.jsonl > gpurun_out/k2exp/ncu.log 2>&1
timeout 900 python tools/sweep.py --out gpurun_out/k2exp/sweep2.jsonl > gpurun_out/k2exp/sweep2.log 2>&1
