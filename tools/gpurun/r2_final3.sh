mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x > gpurun_out/pre.log 2>&1; echo "EXIT $?" >> gpurun_out/pre.log; tail -2 gpurun_out/pre.log
grep -q "EXIT 0" gpurun_out/pre.log || exit 1
WAP_AUTOTUNE=0 timeout 200 python tools/gemm_times.py --model alexnet > gpurun_out/auto_alexnet.log 2>&1; tail -1 gpurun_out/auto_alexnet.log
bash tools/gpurun/r2_final2.sh
