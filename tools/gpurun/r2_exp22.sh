mkdir -p gpurun_out
WAP_AUTOTUNE_SPLITK=1 timeout 900 python tools/tune_plans.py --out gpurun_out/plans_splitk.json > gpurun_out/tune_splitk.log 2>&1; tail -2 gpurun_out/tune_splitk.log
for cfg in "committed:X=1" "splitk:WAP_PLAN_FILE=gpurun_out/plans_splitk.json"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 500 python bench.py --no-cpu-baseline > gpurun_out/b_$name.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_$name.json').read().splitlines()[-1]); print('$name', d['value'], d['vgg16']['value'], d['clocks']['reasons'], d['vgg16']['clocks']['reasons'])"
done
