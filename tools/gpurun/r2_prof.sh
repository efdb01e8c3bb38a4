mkdir -p gpurun_out/ncu
for k in conv4 d_pool1 conv2 d_conv4_w d_conv3_relu; do
  echo "== $k" >> gpurun_out/trace.log
  WAP_LIB_VARIANT=trace timeout 200 python tools/gemm_trace.py --model alexnet --batch 128 --only $k >> gpurun_out/trace.log 2>&1
done
for st in conv4 d_pool1; do
  ncu --profile-from-start off --clock-control none --set full --import-source on -c 1 -f -o gpurun_out/ncu/prof_alexnet_$st \
      python tools/profile_step.py --model alexnet --batch 128 --only "$st" --reps 2 > gpurun_out/ncu/run_$st.log 2>&1
  python tools/ncu_summary.py gpurun_out/ncu/prof_alexnet_$st.ncu-rep > gpurun_out/ncu/ncu_alexnet_$st.txt
done
cat gpurun_out/trace.log; cat gpurun_out/ncu/*.txt
