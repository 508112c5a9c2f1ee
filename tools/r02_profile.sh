# Round-2 small-switch and ncu evidence (one B200). Outputs under gpurun_out/.
#   bash tools/r02_profile.sh [tag]
T=${1:-r02}
O=gpurun_out
set -x
timeout 300 python tools/copy_floor.py --out $O/${T}_copy_floor.jsonl > $O/${T}_copy_floor.log 2>&1
for c in 1seq cfg1 1seq4096; do timeout 200 python tools/k31_trace.py --case $c --out $O/${T}_k31_trace.jsonl >> $O/${T}_k31_trace.log 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tpr_ -c 200 --csv --log-file $O/${T}_launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-headline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tpr_ -c 200 --csv --log-file $O/${T}_launches_cfg1.csv python bench.py --config 0 --steps 4 --warmup 3 --no-cpu --no-e2e --no-headline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tpr_k1_kv_migrate_bulk --launch-skip 1 -c 1 -o $O/${T}_k1_cfg2 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-headline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tpr_k2 --launch-skip 1 -c 1 -o $O/${T}_k2_cfg2 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-headline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tpr_k31 --launch-skip 4 -c 1 -o $O/${T}_k31_1seq python tools/k31_trace.py --case 1seq --reps 8 > /dev/null 2>&1
ls -la $O
