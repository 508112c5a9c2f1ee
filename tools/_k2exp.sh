set -x
mkdir -p gpurun_out/r4
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/r4/pytest.log 2>&1; echo rc=$? >> gpurun_out/r4/pytest.log
timeout 300 python tools/host_overhead.py > gpurun_out/r4/host_overhead.log 2>&1
timeout 300 python tools/host_phases.py > gpurun_out/r4/host_phases.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/r4/bench_cfg2.json 2> gpurun_out/r4/bench_cfg2.err
timeout 600 python bench.py --config 0 --no-cpu > gpurun_out/r4/bench_cfg0.json 2> gpurun_out/r4/bench_cfg0.err
timeout 900 python tools/sweep.py --modes trace --out gpurun_out/r4/sweep_trace.jsonl > gpurun_out/r4/sweep.log 2>&1
