mkdir -p gpurun_out
timeout 600 python tools/tune_plans.py > gpurun_out/tune.log 2>&1; echo "EXIT $?" >> gpurun_out/tune.log
cp paper_1811_01532_b200/profiles/gemm_plans_b200.json gpurun_out/
timeout 900 python -m pytest tests/test_determinism_gpu.py tests/test_runtime_gpu.py tests/test_bench_parity_gpu.py -m gpu -q -s -k "bitwise or byte_identical or add_n or alexnet_b128" > gpurun_out/det_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/det_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -5 gpurun_out/tune.log; tail -15 gpurun_out/det_tests.log; head -c 1500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
