mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_ops_gpu.py -m gpu -q -x 2>&1 | tail -2
for cfg in "band:X=1" "noband:WAP_LRN_POOL_BAND=0"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 200 python bench.py --model alexnet --no-cpu-baseline --breakdown > gpurun_out/b_$name.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_$name.json').read().splitlines()[-1]); b=d['breakdown_ms']; print('$name', d['value'], 'pool1', b.get('pool1'), 'pool2', b.get('pool2'))"
done
