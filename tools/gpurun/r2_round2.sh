mkdir -p gpurun_out
timeout 900 python tools/tune_plans.py > gpurun_out/tune.log 2>&1; echo "EXIT $?" >> gpurun_out/tune.log
cp paper_1811_01532_b200/profiles/gemm_plans_b200.json gpurun_out/
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --breakdown > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1200 python -m pytest tests/test_bench_parity_gpu.py -m gpu -q -s > gpurun_out/parity.log 2>&1; echo "EXIT $?" >> gpurun_out/parity.log
tail -2 gpurun_out/tune.log; tail -1 gpurun_out/smoke.log
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['vgg16']['value'], d['roofline']['kernel'], d['roofline']['kernel_ms'], d['gemm_summary'])"
grep -E "decisions|plain fp32|passed|failed|FAILED|AssertionError" gpurun_out/parity.log
