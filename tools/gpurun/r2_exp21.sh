mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_ops_gpu.py tests/test_runtime_gpu.py -m gpu -q -x 2>&1 | tail -2
for cfg in "direct:X=1" "gemm:WAP_WGRAD_DIRECT=0"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 400 python bench.py --model vgg16 --no-cpu-baseline --breakdown > gpurun_out/b_$name.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_$name.json').read().splitlines()[-1]); b=d['breakdown_ms']; print('$name', d['value'], {k:v for k,v in b.items() if k.startswith('d_conv1_w')})"
done
