"""Isolated CUDA-event time of every GEMM of one training step (diagnostic).

Builds the bench Trainer (AlexNet b=128 / VGG-16 b=32), runs a few steps, then
re-launches each GEMM step alone `--reps` times and prints its shape, the plan
(BN, CTA group, splits, window boxes), the time and the tensor-pipe TFLOP/s
(3 x algorithmic for 3xTF32). Use with WAP_LIB_VARIANT to compare builds.

    WAP_AUTOTUNE=0 python tools/gemm_times.py --model alexnet
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import he_init, synthetic_batch  # noqa: E402
from paper_1811_01532_b200 import _native as N  # noqa: E402
from paper_1811_01532_b200 import models, planner, trainer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="alexnet")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    b = args.batch or (128 if args.model == "alexnet" else 32)
    g = models.MODELS[args.model](b)
    tp = trainer.plan_training(g, 1, planner.load_profile("b200"), force_d=1)
    tr = trainer.Trainer(tp, precision=3, use_graph=False, variables=he_init(g))
    tr.load(synthetic_batch(g, 0, b))
    for _ in range(3):
        tr.run()
    torch.cuda.synchronize()
    L = N.lib()
    stream = torch.cuda.current_stream()
    tot = 0.0
    for st in tr.prog.steps + tr.prog.update_steps:
        inner = getattr(st, "inner", st)
        desc = getattr(inner, "desc", None)
        if desc is None or (args.only and args.only not in inner.name):
            continue
        info = (C.c_int64 * 8)()
        L.wap_gemm_plan_info(inner.call._plan, info)
        inner(N.stream_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.reps):
            inner(N.stream_ptr())
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        tot += ms
        fl = 2.0 * desc.M * desc.N * desc.K * 3
        print(f"{inner.name:22s} M={desc.M:8d} N={desc.N:5d} K={desc.K:8d} bn={info[0]:3d} cg={info[1]} "
              f"splits={info[2]:3d} win={info[4]} pair={info[6]} chain={info[7]} {ms:7.4f} ms  pipe {fl / ms / 1e9:7.1f} TF/s",
              flush=True)
    print(f"total {tot:.3f} ms")


if __name__ == "__main__":
    main()
