mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_ops_gpu.py -m gpu -q -x > gpurun_out/gemmtests.log 2>&1; echo "EXIT $?" >> gpurun_out/gemmtests.log
tail -3 gpurun_out/gemmtests.log
WAP_AUTOTUNE=0 timeout 300 python tools/gemm_times.py --model alexnet > gpurun_out/times_auto.log 2>&1
cat gpurun_out/times_auto.log | grep -v "fc"
for k in conv4 d_conv3_relu; do
  echo "== $k" >> gpurun_out/trace.log
  WAP_LIB_VARIANT=trace WAP_AUTOTUNE=0 timeout 200 python tools/gemm_trace.py --model alexnet --batch 128 --only $k >> gpurun_out/trace.log 2>&1
done
cat gpurun_out/trace.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
