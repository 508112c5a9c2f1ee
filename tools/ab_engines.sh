# usage: git worktree add exp_old <commit> && (cd exp_old && python -m paper_2605_05467_b200.build); bash tools/ab_engines.sh
# same-box A/B of K1/K2 (bench cfg2) and the trace sweep's K1: session-start
# code (exp_old worktree, if present), current default, warp-specialised
set -x
for i in 1 2; do
  [ -d exp_old ] && (cd exp_old && timeout 400 python bench.py --no-cpu --no-e2e --steps 20 > ../gpurun_out/ab_old_$i.json 2>&1)
  timeout 400 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/ab_new_$i.json 2>&1
done
timeout 600 python tools/sweep.py --modes trace --max-seqs 1 --reps 2 --out gpurun_out/ab_sweep_new.jsonl > /dev/null 2>&1
