mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_ops_gpu.py tests/test_runtime_gpu.py -m gpu -q -x > gpurun_out/gemmtests.log 2>&1; echo "EXIT $?" >> gpurun_out/gemmtests.log
for v in default nosplit; do
  if [ $v = default ]; then e=""; else e="WAP_LIB_VARIANT=$v"; fi
  env $e WAP_AUTOTUNE=0 timeout 300 python tools/gemm_times.py --model alexnet > gpurun_out/times_$v.log 2>&1
done
WAP_PLAN_CACHE=0 timeout 400 python bench.py --model alexnet --no-cpu-baseline > gpurun_out/bench_ss.json 2> gpurun_out/bench_ss.err
tail -1 gpurun_out/smoke.log; tail -5 gpurun_out/gemmtests.log; for v in default nosplit; do echo "== $v"; cat gpurun_out/times_$v.log; done
python -c "
import json; d=json.loads(open('gpurun_out/bench_ss.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['kernel_ms'])"
