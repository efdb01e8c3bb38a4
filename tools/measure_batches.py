"""Measure single-GPU training-step time vs per-GPU batch (input to the WAU
calibration and the small-minibatch sweep, BASELINE config 4).

    python tools/measure_batches.py --out gpurun_out/batch_times.json
"""
import argparse
import gc
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import he_init, synthetic_batch  # noqa: E402
from paper_1811_01532_b200 import models, planner, trainer  # noqa: E402

BATCHES = {
    "alexnet": [2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512],
    "vgg16": [2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512],
}


def time_step(net, b, precision, steps, warmup):
    g = models.MODELS[net](b)
    tp = trainer.plan_training(g, 1, planner.load_profile("b200"), force_d=1)
    tr = trainer.Trainer(tp, precision=precision, variables=he_init(g))
    tr.load(synthetic_batch(g, 0, b))
    for _ in range(warmup):
        tr.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        tr.run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del tr
    gc.collect()
    torch.cuda.empty_cache()
    return ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/batch_times.json")
    ap.add_argument("--precision", type=int, default=3)
    ap.add_argument("--nets", default="alexnet,vgg16")
    args = ap.parse_args()
    res = {"precision": args.precision, "device": torch.cuda.get_device_name(0), "ms": {}}
    for net in args.nets.split(","):
        res["ms"][net] = {}
        for b in BATCHES[net]:
            t0 = time.time()
            steps = 10 if (net == "alexnet" or b <= 64) else 4
            ms = time_step(net, b, args.precision, steps, 3)
            res["ms"][net][b] = ms
            print(f"{net} b={b}: {ms:.3f} ms/step ({b / ms * 1e3:.0f} img/s) [{time.time() - t0:.1f}s]", flush=True)
            Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
