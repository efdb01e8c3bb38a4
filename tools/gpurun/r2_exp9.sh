mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x > gpurun_out/t.log 2>&1; echo "EXIT $?" >> gpurun_out/t.log; tail -3 gpurun_out/t.log
if grep -q "EXIT 0" gpurun_out/t.log; then
  for net in alexnet vgg16; do
    WAP_PLAN_CACHE=0 WAP_AUTOTUNE_FREE=1 WAP_AUTOTUNE_LOG=1 timeout 400 python tools/gemm_times.py --model $net > gpurun_out/times_$net.log 2>&1
    grep -E "bn= 64|total" gpurun_out/times_$net.log
    grep -E "autotune d_pool1 " gpurun_out/times_$net.log
  done
  WAP_PLAN_CACHE=0 WAP_AUTOTUNE_FREE=1 timeout 500 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2>gpurun_out/bench.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['vgg16']['value'], d['roofline']['kernel'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
fi
