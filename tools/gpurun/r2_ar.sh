mkdir -p gpurun_out
timeout 300 python tools/gemm_accuracy.py > gpurun_out/gemm_accuracy.log 2>&1
timeout 900 python -m pytest tests/test_allreduce_gpu.py -m gpu -q -x > gpurun_out/allreduce_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/allreduce_tests.log
cat gpurun_out/gemm_accuracy.log; tail -30 gpurun_out/allreduce_tests.log
