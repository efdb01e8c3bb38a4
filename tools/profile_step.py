"""Run selected launches of a lowered training step (for ncu captures).

    python tools/profile_step.py --model alexnet --batch 128 --only d_conv2_w --reps 3
runs the whole step once (warm-up), then `--reps` times only the steps whose
name matches `--only` (substring), so `ncu --profile-from-start off` catches exactly those launches.
"""
import argparse
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
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--precision", type=int, default=3)
    args = ap.parse_args()
    g = models.MODELS[args.model](args.batch)
    tp = trainer.plan_training(g, 1, planner.load_profile("b200"), force_d=1)
    tr = trainer.Trainer(tp, precision=args.precision, use_graph=False, variables=he_init(g))
    tr.load(synthetic_batch(g, 0, args.batch))
    if not args.only:
        tr.run()
    torch.cuda.synchronize()
    names = args.only.split(",")
    steps = [getattr(s, "inner", s) for s in tr.prog.steps]
    sel = [s for s in steps if s.name in names] or [s for s in steps if args.only in s.name]
    print("selected:", [s.name for s in sel], flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # ncu --profile-from-start off captures only this region (autotuning and
    # warm-up launches stay outside it)
    torch.cuda.profiler.start()
    for i in range(args.reps):
        if i == 1:
            e0.record()
        for s in sel:
            s(N.stream_ptr())
    e1.record()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    if args.reps > 1:
        print(f"avg ms per rep: {e0.elapsed_time(e1) / (args.reps - 1):.4f}", flush=True)


if __name__ == "__main__":
    main()
