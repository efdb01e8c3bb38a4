for cfg in "default:X=1" "nohop:WAP_LIB_VARIANT=nohop"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name"
  env $envs WAP_AUTOTUNE=0 timeout 200 python tools/gemm_times.py --model alexnet 2>&1 | grep -vE "fc"
  env $envs WAP_AUTOTUNE=0 timeout 300 python tools/gemm_times.py --model vgg16 2>&1 | grep -E "total"
done
