set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 9 python __graft_entry__.py > gpurun_out/sanitize_memcheck_smoke.log 2>&1; echo rc=$? >> gpurun_out/sanitize_memcheck_smoke.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --error-exitcode 9 python __graft_entry__.py > gpurun_out/sanitize_racecheck_smoke.log 2>&1; echo rc=$? >> gpurun_out/sanitize_racecheck_smoke.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_kv_gpu.py tests/test_bulk_engine_gpu.py tests/test_weights_gpu.py -q -x -k "not full_size and not cfg" > gpurun_out/sanitize_memcheck_tests.log 2>&1; echo rc=$? >> gpurun_out/sanitize_memcheck_tests.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --error-exitcode 9 python __graft_entry__.py > gpurun_out/sanitize_synccheck_smoke.log 2>&1; echo rc=$? >> gpurun_out/sanitize_synccheck_smoke.log
# the fused K3's shared-memory scan and record copies, across plan sizes (one-warp blocks included)
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_kv_gpu.py -q -x -k "not full_size and not cfg and not large" > gpurun_out/sanitize_racecheck_k3.log 2>&1; echo rc=$? >> gpurun_out/sanitize_racecheck_k3.log
# K31, both schedules (item shares: cross-CTA reader counters; dynamic: owner
# decisions, cooperative grid-wide wait, dynamic claims)
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_kv_gpu.py -q -x -k "k31 or launch_paths" > gpurun_out/sanitize_${tool}_k31.log 2>&1; echo rc=$? >> gpurun_out/sanitize_${tool}_k31.log
done
