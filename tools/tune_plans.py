"""Write the committed GEMM plan file (paper_1811_01532_b200/profiles/gemm_plans_b200.json).

Runs the unrestricted autotuner (WAP_AUTOTUNE_FREE=1: CTA vs CTA pair, halo window,
BN, explicit K splits, whatever their rounding) over every GEMM of the benchmark
training programs on this B200 and pins the winners. Programs built later look their
GEMMs up in the file and skip timing, so their results are identical run to run
(plan_cache.py). Run on a GPU box:  python tools/tune_plans.py [--nets alexnet:128 vgg16:32]
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ["WAP_AUTOTUNE_FREE"] = "1"
os.environ["WAP_AUTOTUNE"] = "1"
os.environ.setdefault("WAP_AUTOTUNE_REPS", "12")  # 12 timed launches per candidate (3 by default at run time)


def main():
    import torch

    from bench import he_init
    from paper_1811_01532_b200 import models, plan_cache, planner, trainer

    ap = argparse.ArgumentParser()
    ap.add_argument("--nets", nargs="*", default=["alexnet:128", "vgg16:32"])
    ap.add_argument("--out", default=str(plan_cache.PLAN_FILE))
    ap.add_argument("--merge", action="store_true", help="keep entries of the existing file (default: rewrite)")
    args = ap.parse_args()
    if not args.merge and Path(args.out).exists():
        Path(args.out).unlink()  # plans of another kernel build may not be valid any more
    plans = {}
    prof = planner.load_profile("b200")
    for spec in args.nets:
        net, b = spec.split(":")
        b = int(b)
        g = models.MODELS[net](b)
        tp = trainer.plan_training(g, 1, prof, force_d=1)
        t0 = time.time()
        tr = trainer.Trainer(tp, precision=3, variables=he_init(g), use_graph=False)
        torch.cuda.synchronize()
        n = len(tr.prog.tuned_plans)
        plans.update(tr.prog.tuned_plans)
        print(f"{spec}: {n} GEMM plans tuned in {time.time() - t0:.1f} s", flush=True)
        del tr
        torch.cuda.empty_cache()
    meta = {"device": torch.cuda.get_device_name(), "written_by": "tools/tune_plans.py",
            "nets": args.nets, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    plan_cache.save(plans, args.out, meta)
    print(f"wrote {len(plans)} plans -> {args.out}")


if __name__ == "__main__":
    main()
