mkdir -p gpurun_out
for k in d_fc6_w fc6 d_pool1 d_conv4_w; do
  echo "== $k" >> gpurun_out/trace.log
  WAP_LIB_VARIANT=trace timeout 200 python tools/gemm_trace.py --model alexnet --batch 128 --only $k >> gpurun_out/trace.log 2>&1
done
cat gpurun_out/trace.log
