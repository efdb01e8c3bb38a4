mkdir -p gpurun_out
for v in default blate; do
  if [ $v = default ]; then e="X=1"; else e="WAP_LIB_VARIANT=$v"; fi
  echo "== $v" >> gpurun_out/exp2.log
  env $e timeout 300 python tools/gemm_times.py --model alexnet >> gpurun_out/exp2.log 2>&1
done
for c in 8 16 32 0; do
  echo "== d_pool1 pair chain $c" >> gpurun_out/exp2.log
  WAP_CHAIN_CHUNKS=$c WAP_AUTOTUNE=0 WAP_GEMM_CG=1 timeout 200 python tools/gemm_times.py --model alexnet --only d_pool1 2>&1 | grep -v total >> gpurun_out/exp2.log
done
cat gpurun_out/exp2.log
