"""Per-rank step time of the WAP data-parallel program at every (G, d) of the
small-minibatch sweep (BASELINE config 4), on ONE B200 (input to tools/wau_sweep.py).

For each global batch G and each degree d <= 8 dividing G, the transformed graph's
rank-0 program (trainer.rank_view: its contiguous b = G/d shard, the bucketed
gradient allreduces with their SGD, the whole step one CUDA graph) runs on this GPU
inside a world-size-1 NCCL process group, so every collective is issued and
captured but moves no bytes. The time is therefore the rank's compute plus the
collective launch overhead; the NVLink transfer itself is modeled by wau_sweep.py.

    python tools/measure_rank_steps.py --out gpurun_out/rank_steps.json
"""
import argparse
import gc
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import he_init, synthetic_batch  # noqa: E402
from paper_1811_01532_b200 import models, planner, trainer  # noqa: E402

SWEEP = (16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512)


def time_rank(net, G, d, steps, warmup):
    g = models.MODELS[net](G)
    tp = trainer.plan_training(g, 8, planner.load_profile("b200"), force_d=d)
    tr = trainer.Trainer(tp, rank=0, variables=he_init(g), process_group=dist.group.WORLD if d > 1 else None)
    b = G // d
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
    captured = tr._captured
    del tr
    gc.collect()
    torch.cuda.empty_cache()
    return ms, captured


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/rank_steps.json")
    ap.add_argument("--nets", default="alexnet,vgg16")
    args = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    res = {"device": torch.cuda.get_device_name(0), "how": __doc__.split("\n\n")[1].replace("\n", " "),
           "autotune": os.environ.get("WAP_AUTOTUNE", "1"), "ms": {}}
    for net in args.nets.split(","):
        res["ms"][net] = {}
        for G in SWEEP:
            for d in range(1, 9):
                if G % d:
                    continue
                t0 = time.time()
                steps = 10 if net == "alexnet" or G // d <= 64 else 4
                ms, cap = time_rank(net, G, d, steps, 3)
                res["ms"][net].setdefault(str(G), {})[str(d)] = ms
                print(f"{net} G={G} d={d} b={G // d}: {ms:.3f} ms/step (graph {cap}) [{time.time() - t0:.1f}s]",
                      flush=True)
                Path(args.out).write_text(json.dumps(res, indent=1))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
