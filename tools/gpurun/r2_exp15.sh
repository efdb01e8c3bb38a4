mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_ops_gpu.py tests/test_runtime_gpu.py tests/test_determinism_gpu.py -m gpu -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 200 python tools/gemm_times.py --model alexnet 2>&1 | grep -E "total"
timeout 300 python tools/gemm_times.py --model vgg16 2>&1 | grep -E "total"
timeout 500 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['vgg16']['value'], d['roofline']['kernel'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
