mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_determinism_gpu.py tests/test_runtime_gpu.py -m gpu -q -k "bitwise or byte_identical or add_n" > gpurun_out/det_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/det_tests.log
tail -30 gpurun_out/det_tests.log; tail -3 gpurun_out/tune.log
