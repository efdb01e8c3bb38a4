mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x -k "n64" > gpurun_out/pair2_test.log 2>&1; echo "EXIT $?" >> gpurun_out/pair2_test.log
tail -15 gpurun_out/pair2_test.log
if grep -q "EXIT 0" gpurun_out/pair2_test.log; then
  timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_ops_gpu.py tests/test_runtime_gpu.py tests/test_determinism_gpu.py -m gpu -q -x > gpurun_out/gemmtests.log 2>&1; echo "EXIT $?" >> gpurun_out/gemmtests.log
  tail -3 gpurun_out/gemmtests.log
  python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
  for net in alexnet vgg16; do
    WAP_PLAN_CACHE=0 WAP_AUTOTUNE_FREE=1 WAP_AUTOTUNE_LOG=1 timeout 400 python tools/gemm_times.py --model $net > gpurun_out/times_$net.log 2>&1
    grep -E "bn= 64|total" gpurun_out/times_$net.log
  done
fi
