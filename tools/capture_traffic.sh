#!/bin/bash
# ncu --set full captures of selected launches of one training step (run under gpurun).
# Reports stay in /tmp on the box; summaries go to gpurun_out/ncu/ncu_<model>_<step>.txt and
# DRAM bytes per launch are merged into gpurun_out/traffic.json (copy both into profiles/).
#   tools/capture_traffic.sh alexnet 128 "d_pool1 conv2 d_conv2_w"
set -e
model=$1; batch=$2; steps=$3
mkdir -p gpurun_out/ncu /tmp/ncu
[ -f gpurun_out/traffic.json ] || { [ -f profiles/traffic.json ] && cp profiles/traffic.json gpurun_out/traffic.json; } || true
for st in $steps; do
  tag=$(echo "$st" | tr '/()' '___')
  rep=/tmp/ncu/prof_${model}_${tag}
  ncu --profile-from-start off --clock-control none --set full --import-source on -c 1 -f -o $rep \
      python tools/profile_step.py --model $model --batch $batch --only "$st" --reps 2 > /dev/null 2>&1 || true
  python tools/ncu_summary.py $rep.ncu-rep > gpurun_out/ncu/ncu_${model}_${tag}.txt
  python tools/traffic_json.py gpurun_out/traffic.json $model "$st" $rep.ncu-rep
done
