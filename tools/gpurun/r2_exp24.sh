# timing-only diagnostics (results are wrong): splitter without its TMEM A store, splitter without any work
for cfg in "default:X=1" "noasplit:WAP_LIB_VARIANT=noasplit" "nosplit:WAP_LIB_VARIANT=nosplit"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  echo "== $name"
  env $envs WAP_AUTOTUNE=0 timeout 200 python tools/gemm_times.py --model alexnet 2>&1 | grep -E "conv3 |conv4 |d_conv3_relu|d_conv4_w|d_pool1|total"
done
