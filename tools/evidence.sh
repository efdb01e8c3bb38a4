#!/bin/bash
# Round evidence on one B200 (run under gpurun): GPU tests, smoke, bench lines of both
# nets + the reference arm, per-step ncu launch lists, ncu --set full traffic captures
# of the dominant GEMMs. Everything lands in gpurun_out/ (copy what is judged to profiles/).
#   tools/evidence.sh "d_pool1 conv2" "d_conv2_w conv3"
mkdir -p gpurun_out
ALEX_STEPS=$1; VGG_STEPS=$2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "EXIT $?" >> gpurun_out/gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_alexnet.json 2> gpurun_out/bench_alexnet.err
timeout 400 python bench.py --model vgg16 > gpurun_out/bench_vgg16.json 2> gpurun_out/bench_vgg16.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for mb in "alexnet 128" "vgg16 32"; do
  set -- $mb
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/$1_b$2_launches.csv python tools/profile_step.py --model $1 --batch $2 --reps 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/$1_b$2_launches.csv > gpurun_out/$1_b$2_launches.txt
done
[ -n "$ALEX_STEPS" ] && timeout 900 bash tools/capture_traffic.sh alexnet 128 "$ALEX_STEPS"
[ -n "$VGG_STEPS" ] && timeout 900 bash tools/capture_traffic.sh vgg16 32 "$VGG_STEPS"
true
