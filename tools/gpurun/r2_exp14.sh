for cfg in "default:X=1" "noepimath:WAP_LIB_VARIANT=noepimath"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name"
  env $envs timeout 200 python tools/gemm_times.py --model alexnet 2>&1 | grep -E "_w |total"
done
