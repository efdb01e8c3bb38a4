mkdir -p gpurun_out
timeout 900 bash tools/capture_traffic.sh alexnet 128 "d_conv1_relu pool1"
cat gpurun_out/ncu/*.txt
for st in d_conv1_relu pool1; do
  ncu -i /tmp/ncu/prof_alexnet_${st}.ncu-rep --page details --csv 2>/dev/null | grep -iE "Issue Slot|Warp Cycles Per Issued|No Eligible|Achieved Occupancy|Theoretical Occupancy|Registers Per|Stall" | head -20
done
