"""Per-rep CUDA-event times of selected launches inside the full training step
(the bench's instrumented pass, without averaging), after K graph steps.

    python tools/step_reps.py --model alexnet --only conv3,conv4,conv5 --steps 20 --reps 5
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
    ap.add_argument("--only", default="conv4")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--async-steps", type=int, default=0, help="Trainer.step_async steps after --steps")
    args = ap.parse_args()
    g = models.MODELS[args.model](args.batch)
    tp = trainer.plan_training(g, 1, planner.load_profile("b200"), force_d=1)
    tr = trainer.Trainer(tp, precision=3, use_graph=not args.no_graph, variables=he_init(g))
    tr.load(synthetic_batch(g, 0, args.batch))
    for _ in range(args.steps):
        tr.run()
    batch = synthetic_batch(g, 0, args.batch)
    for _ in range(args.async_steps):
        tr.step_async(batch)
    if args.async_steps:
        print("loss", tr.last_loss())
    torch.cuda.synchronize()
    names = set(args.only.split(","))
    stream = torch.cuda.current_stream()
    steps = [getattr(s, "inner", s) for s in tr.prog.steps]
    for r in range(args.reps):
        evs = []
        prev = None
        for st in steps:
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st(N.stream_ptr())
            z.record(stream)
            if st.name in names:
                evs.append((st.name, prev, a, z))
            prev = st.name
        torch.cuda.synchronize()
        print(f"rep {r}: " + "  ".join(f"{n}(after {p}) {a.elapsed_time(z):.4f}" for n, p, a, z in evs), flush=True)


if __name__ == "__main__":
    main()
