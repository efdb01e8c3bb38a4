mkdir -p gpurun_out
cp paper_1811_01532_b200/profiles/gemm_plans_b200.json gpurun_out/plans_committed.json
timeout 900 python tools/tune_plans.py --out gpurun_out/plans_r12.json > gpurun_out/tune_r12.log 2>&1; tail -1 gpurun_out/tune_r12.log
for rep in 1 2; do
for cfg in "committed:X=1" "r12:WAP_PLAN_FILE=gpurun_out/plans_r12.json"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 500 python bench.py --no-cpu-baseline > gpurun_out/b_$name.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_$name.json').read().splitlines()[-1]); print('$name', d['value'], d['vgg16']['value'], d['clocks']['reasons'], d['vgg16']['clocks']['reasons'])"
done
done
