# Re-measure everything the docs cite (one B200). Outputs under gpurun_out/.
#   bash tools/refresh_round.sh [tag]     (default tag: final); then tools/refresh_extra.sh [tag]
#   then copy the outputs the docs cite into profiles/rNN/
T=${1:-final}
O=gpurun_out
set -x
timeout 1200 python -m pytest tests -q -m gpu > $O/${T}_pytest_gpu.log 2>&1; echo rc=$? >> $O/${T}_pytest_gpu.log
timeout 600 python bench.py > $O/${T}_bench_n1.json 2> $O/${T}_bench_n1.err
timeout 600 python bench.py --config 4 --no-headline > $O/${T}_bench_headline.json 2> $O/${T}_bench_headline.err
for c in 0 2 3; do timeout 600 python bench.py --config $c --no-cpu --no-headline > $O/${T}_bench_cfg$c.json 2> $O/${T}_bench_cfg$c.err; done
timeout 600 python bench.py --weights-mode full_copy_per_gpu --no-cpu --no-headline > $O/${T}_bench_fullcopy.json 2> $O/${T}_bench_fullcopy.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err
timeout 300 python tools/small_switch.py --out $O/${T}_small_switch.jsonl > $O/${T}_small_switch.log 2>&1
timeout 900 python tools/weight_sweep.py --out $O/${T}_weight_sweep.jsonl > $O/${T}_weight_sweep.log 2>&1
timeout 900 python tools/weight_sweep.py --model 70b --layers 20 --sets 8:4,8 --sets 4:2,4 --out $O/${T}_weight_sweep_70b.jsonl > $O/${T}_weight_sweep_70b.log 2>&1
# ncu: launch lists (cfg2, cfg1) and full captures of K1 (cfg2; trace contexts), K2 (cfg2) and K31
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tpr_k[0-9] -c 200 --csv --log-file $O/${T}_launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-headline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tpr_k[0-9] -c 200 --csv --log-file $O/${T}_launches_cfg1.csv python bench.py --config 0 --steps 4 --warmup 3 --no-cpu --no-e2e --no-headline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tpr_k1_kv_migrate_bulk --launch-skip 1 -c 1 -o $O/${T}_k1_cfg2 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-headline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tpr_k2 --launch-skip 1 -c 1 -o $O/${T}_k2_cfg2 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-headline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tpr_k1_kv_migrate_bulk --launch-skip 2 -c 1 -o $O/${T}_k1_tensor_trace python tools/sweep.py --modes trace --only 4:8:256 --reps 1 --k1-reps 1 --out /dev/null > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tpr_k31 --launch-skip 4 -c 1 -o $O/${T}_k31_1seq python tools/k31_trace.py --case 1seq --reps 8 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tpr_k31 --launch-skip 4 -c 1 -o $O/${T}_k31_cfg1 python tools/k31_trace.py --case cfg1 --reps 8 > /dev/null 2>&1
