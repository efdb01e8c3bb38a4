"""Per-GEMM timing of one training step, for comparing library variants
(tools/build_variant.sh): e.g. the full kernel vs a TMA(+split)-only build.

    WAP_AUTOTUNE=0 WAP_LIB_VARIANT=tmaonly python tools/gemm_diag.py --model vgg16 --batch 32
prints `name  M N K  config  ms  pipe-TFLOP/s` for every tcgen05 GEMM launch.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import he_init, synthetic_batch  # noqa: E402
from paper_1811_01532_b200 import _native as N  # noqa: E402
from paper_1811_01532_b200 import models, planner, trainer  # noqa: E402
from paper_1811_01532_b200.runtime import _GemmStep  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="alexnet")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--precision", type=int, default=3)
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    g = models.MODELS[args.model](args.batch)
    tp = trainer.plan_training(g, 1, planner.load_profile("b200"), force_d=1)
    tr = trainer.Trainer(tp, precision=args.precision, use_graph=False, variables=he_init(g))
    tr.load(synthetic_batch(g, 0, args.batch))
    torch.cuda.synchronize()
    s = N.stream_ptr()
    rows = []
    for st in tr.prog.steps:
        st = getattr(st, "inner", st)
        if not isinstance(st, _GemmStep):
            continue
        st(s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            st(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        pipe = st.alg_flops * (3 if args.precision == 3 else 1) / (ms * 1e-3) / 1e12
        rows.append({"name": st.name, "MNK": list(st.shape), "ms": round(ms, 4), "pipe_tflops": round(pipe, 1)})
        print(f"{st.name:18s} {str(st.shape):26s} {ms:8.4f} ms {pipe:7.1f} TF/s", flush=True)
    print(f"total {sum(r['ms'] for r in rows):.3f} ms")
    if args.json:
        Path(args.json).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
