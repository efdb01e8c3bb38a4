mkdir -p gpurun_out
for cfg in "default_c8:X=1" "slots8_c8:WAP_LIB_VARIANT=slots8" "slots8_c16:WAP_LIB_VARIANT=slots8 WAP_CHAIN_CHUNKS=16" "default_c16:WAP_CHAIN_CHUNKS=16"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name" >> gpurun_out/exp3.log
  env $envs WAP_AUTOTUNE=0 WAP_GEMM_CG=2 timeout 300 python tools/gemm_times.py --model alexnet 2>&1 | grep -E "bn=128|total" >> gpurun_out/exp3.log
done
cat gpurun_out/exp3.log
