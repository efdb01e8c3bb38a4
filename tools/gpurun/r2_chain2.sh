mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_ops_gpu.py tests/test_runtime_gpu.py tests/test_determinism_gpu.py -m gpu -q -x > gpurun_out/gemmtests.log 2>&1; echo "EXIT $?" >> gpurun_out/gemmtests.log
WAP_AUTOTUNE=0 timeout 300 python tools/gemm_times.py --model alexnet > gpurun_out/times_auto.log 2>&1
WAP_PLAN_CACHE=0 WAP_AUTOTUNE_FREE=1 WAP_AUTOTUNE_LOG=1 timeout 400 python bench.py --model alexnet --no-cpu-baseline --breakdown > gpurun_out/bench_free.json 2> gpurun_out/bench_free.err
timeout 600 python tools/wgrad_diag.py --net vgg16 --batch 32 > gpurun_out/wgrad_diag.log 2>&1
tail -1 gpurun_out/smoke.log; tail -3 gpurun_out/gemmtests.log; cat gpurun_out/times_auto.log
python -c "
import json; d=json.loads(open('gpurun_out/bench_free.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['kernel_ms'], d['gemm_summary'])"
cat gpurun_out/wgrad_diag.log | tail -8
