mkdir -p gpurun_out
for spec in "alexnet 128 d_fc6_w" "alexnet 128 d_pool1" "vgg16 32 conv2" "vgg16 32 d_conv1_relu"; do
  set -- $spec
  echo "== $1 $3" >> gpurun_out/epitrace.log
  WAP_LIB_VARIANT=epitrace timeout 300 python tools/gemm_trace.py --model $1 --batch $2 --only $3 >> gpurun_out/epitrace.log 2>&1
done
cat gpurun_out/epitrace.log
