WAP_LIB_VARIANT=asms timeout 200 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x 2>&1 | tail -1
for cfg in "default:X=1" "asms:WAP_LIB_VARIANT=asms"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name"
  env $envs WAP_AUTOTUNE=0 timeout 200 python tools/gemm_times.py --model alexnet 2>&1 | grep -vE "bn= 64"
  env $envs WAP_AUTOTUNE=0 timeout 300 python tools/gemm_times.py --model vgg16 2>&1 | grep -E "total"
done
