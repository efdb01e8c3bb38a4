mkdir -p gpurun_out
run() { # name env...
  name=$1; shift
  echo "== $name" >> gpurun_out/exp1.log
  env "$@" WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 200 python tools/gemm_times.py --model alexnet --only d_pool1 2>&1 | grep -v total >> gpurun_out/exp1.log
  env "$@" WAP_AUTOTUNE=0 timeout 200 python tools/gemm_times.py --model alexnet 2>&1 | grep -E "conv2 |conv4 |d_conv3_relu|d_conv2_w|total" >> gpurun_out/exp1.log
}
run ss_c8 WAP_CHAIN_CHUNKS=8
run ss_c0 WAP_CHAIN_CHUNKS=0
run ss_c16 WAP_CHAIN_CHUNKS=16
run ss_c4 WAP_CHAIN_CHUNKS=4
run ts_c8 WAP_LIB_VARIANT=tsa WAP_CHAIN_CHUNKS=8
run ts_c0 WAP_LIB_VARIANT=tsa WAP_CHAIN_CHUNKS=0
cat gpurun_out/exp1.log
