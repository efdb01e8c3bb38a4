# final r02 evidence at HEAD with the committed plan file: GPU tests, smoke, bench, reference arm, launch lists
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/gputests.log 2>&1; echo "EXIT $?" >> gpurun_out/gputests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --breakdown > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for mb in "alexnet 128" "vgg16 32"; do
  set -- $mb
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/$1_b$2_launches.csv python tools/profile_step.py --model $1 --batch $2 --reps 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/$1_b$2_launches.csv > gpurun_out/$1_b$2_launches.txt
done
timeout 900 bash tools/capture_traffic.sh alexnet 128 "d_pool1 conv2"
timeout 900 bash tools/capture_traffic.sh vgg16 32 "d_conv1_relu d_conv2_w"
tail -1 gpurun_out/smoke.log; grep -E "decisions|plain fp32|passed|failed|FAILED" gpurun_out/gputests.log
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['vgg16']['value'], d['vgg16']['e2e']['value'], d['roofline']['kernel'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks'], d['vgg16']['clocks'])"
