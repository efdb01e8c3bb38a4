WAP_LIB_VARIANT=sg3 timeout 200 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x 2>&1 | tail -1
for cfg in "sg2:X=1" "sg3:WAP_LIB_VARIANT=sg3"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name"
  env $envs WAP_AUTOTUNE=0 timeout 200 python tools/gemm_times.py --model alexnet 2>&1 | grep -v "fc"
  env $envs WAP_AUTOTUNE=0 timeout 250 python tools/gemm_times.py --model vgg16 2>&1 | grep -E "total"
done
