# The rest of the measurements the docs cite (one B200), after refresh_round.sh.
#   bash tools/refresh_extra.sh [tag]     (default tag: final)
T=${1:-final}
O=gpurun_out
set -x
timeout 1500 python tools/sweep.py --out $O/${T}_sweep.jsonl > $O/${T}_sweep.log 2>&1
timeout 300 python tools/copy_floor.py --out $O/${T}_copy_floor.jsonl > $O/${T}_copy_floor.log 2>&1
for c in 1seq cfg1 1seq4096; do timeout 200 python tools/k31_trace.py --case $c --out $O/${T}_k31_trace.jsonl >> $O/${T}_k31_trace.log 2>&1; done
timeout 300 python tools/host_profile.py > $O/${T}_host_profile_1seq.log 2>&1
timeout 900 python tools/reuse_order.py --measure --out $O/${T}_reuse_order.jsonl > $O/${T}_reuse_order.log 2>&1
timeout 900 python tools/kv_microbench.py --out $O/${T}_kv_microbench.jsonl > $O/${T}_kv_microbench.log 2>&1
timeout 600 python tools/replay_engine.py --out $O/${T}_engine_replay.jsonl > $O/${T}_engine_replay.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tpr_k1_kv_migrate_bulk --launch-skip 1 -c 1 -o $O/${T}_k1_cfg4_70b python bench.py --config 3 --steps 2 --warmup 1 --no-cpu --no-e2e --no-headline > /dev/null 2>&1
