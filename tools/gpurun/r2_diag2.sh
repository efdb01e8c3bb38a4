mkdir -p gpurun_out
./tools/desc_shift_probe.bin > gpurun_out/desc_shift.log 2>&1
for cfg in "default:" "nocache:WAP_PLAN_CACHE=0" "noauto:WAP_AUTOTUNE=0" "nosacc:WAP_LIB_VARIANT=nosacc WAP_PLAN_CACHE=0"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name ($envs)" >> gpurun_out/smoke_diag.log
  env $envs timeout 300 python tools/smoke_diag.py >> gpurun_out/smoke_diag.log 2>&1
done
for cfg in "nocache:WAP_PLAN_CACHE=0" "nosacc:WAP_LIB_VARIANT=nosacc WAP_PLAN_CACHE=0" "nosaccfree:WAP_LIB_VARIANT=nosacc WAP_PLAN_CACHE=0 WAP_AUTOTUNE_FREE=1"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 400 python bench.py --model alexnet --no-cpu-baseline --breakdown > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
done
for k in d_pool1 conv3 d_conv3 conv2; do
  echo "== $k" >> gpurun_out/trace.log
  WAP_LIB_VARIANT=trace WAP_AUTOTUNE=0 timeout 200 python tools/gemm_trace.py --model alexnet --batch 128 --only $k >> gpurun_out/trace.log 2>&1
done
cat gpurun_out/desc_shift.log gpurun_out/smoke_diag.log gpurun_out/trace.log
for f in nocache nosacc nosaccfree; do python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$f.json').read().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['kernel_ms'])"; done
