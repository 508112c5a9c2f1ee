# same-box A/B of K1/K2 (bench cfg2): session-start code (exp_old worktree, if
# present) vs the current lean and forced-tensor K1 kernels
set -x
for i in 1 2; do
  [ -d exp_old ] && (cd exp_old && timeout 400 python bench.py --no-cpu --no-e2e --steps 20 > ../gpurun_out/ab_old_$i.json 2>&1)
  timeout 400 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/ab_new_$i.json 2>&1
  TPR_TENSOR_PARTIAL=2 timeout 400 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/ab_tensor_$i.json 2>&1
done
