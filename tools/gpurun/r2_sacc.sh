mkdir -p gpurun_out
timeout 300 python tools/gemm_accuracy.py > gpurun_out/gemm_accuracy.log 2>&1
timeout 600 python tools/tune_plans.py > gpurun_out/tune.log 2>&1; echo "EXIT $?" >> gpurun_out/tune.log
cp paper_1811_01532_b200/profiles/gemm_plans_b200.json gpurun_out/
timeout 1500 python -m pytest tests/test_gemm_gpu.py tests/test_determinism_gpu.py tests/test_bench_parity_gpu.py tests/test_runtime_gpu.py -m gpu -q -s > gpurun_out/sacc_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/sacc_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/gemm_accuracy.log; tail -3 gpurun_out/tune.log; grep -E "decisions|passed|failed|FAIL" gpurun_out/sacc_tests.log | tail -20; head -c 400 gpurun_out/bench.json
