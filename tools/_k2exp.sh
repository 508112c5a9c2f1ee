set -x
mkdir -p gpurun_out/k2dyn
timeout 600 python -m pytest tests/test_bulk_engine_gpu.py tests/test_weights_gpu.py -q -m gpu > gpurun_out/k2dyn/pytest.log 2>&1; echo rc=$? >> gpurun_out/k2dyn/pytest.log
for cfg in 4x16384 6x16384 3x32768 8x16384 4x32768; do
  TPR_BULK_K2=$cfg timeout 300 python tools/weight_sweep.py --reps 5 --only 8:2:4,8:2:8,4:2:4,4:4:2,8:4:2,8:8:4 --out gpurun_out/k2dyn/ws_$cfg.jsonl > gpurun_out/k2dyn/ws_$cfg.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tpr_k2 --launch-skip 2 -c 1 -o gpurun_out/k2dyn/k2_fwd_8_2_4 python tools/weight_sweep.py --reps 1 --only 8:2:4 --out gpurun_out/k2dyn/ncu_ws.jsonl > gpurun_out/k2dyn/ncu.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/k2dyn/bench_cfg2.json 2> gpurun_out/k2dyn/bench_cfg2.err
