# Re-measure everything the docs cite (one B200). Outputs under gpurun_out/.
set -x
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/final_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/final_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err
timeout 600 python bench.py --config 4 > gpurun_out/final_bench_headline.json 2> gpurun_out/final_bench_headline.err
for c in 0 2 3; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/final_bench_cfg$c.json 2> gpurun_out/final_bench_cfg$c.err; done
timeout 600 python bench.py --weights-mode full_copy_per_gpu --no-cpu > gpurun_out/final_bench_fullcopy.json 2> gpurun_out/final_bench_fullcopy.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
timeout 900 python tools/sweep.py --out gpurun_out/final_sweep.jsonl > gpurun_out/final_sweep.log 2>&1
