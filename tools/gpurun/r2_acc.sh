mkdir -p gpurun_out
timeout 300 python tools/gemm_accuracy.py > gpurun_out/gemm_accuracy.log 2>&1
cat gpurun_out/gemm_accuracy.log
