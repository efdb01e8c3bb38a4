for cfg in "rolled:X=1" "unrolled:WAP_LIB_VARIANT=epiunroll"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name"
  env $envs timeout 200 python tools/gemm_times.py --model alexnet 2>&1 | grep -E "conv4 |conv2 |d_conv3_relu|total"
  env $envs timeout 300 python tools/gemm_times.py --model vgg16 2>&1 | grep -E "total"
done
