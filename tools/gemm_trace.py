"""Role/wait breakdown of one GEMM launch (needs a -DWAP_GEMM_TRACE build):
    WAP_NVCC_EXTRA=-DWAP_GEMM_TRACE python -m paper_1811_01532_b200.build --force
    WAP_AUTOTUNE=0 python tools/gemm_trace.py --model vgg16 --batch 32 --only conv2
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

ROLES = ["producer(empty-win / empty / tma-issue)", "mma(tempty / conv|full)", "epilogue(tfull / drain / drain-bar)",
         "splitter0(full / win+aslot / st-wait+bar)", "splitter1(full / win+aslot / st-wait+bar)"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="vgg16")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--only", default="conv2")
    ap.add_argument("--precision", type=int, default=3)
    args = ap.parse_args()
    g = models.MODELS[args.model](args.batch)
    tp = trainer.plan_training(g, 1, planner.load_profile("b200"), force_d=1)
    tr = trainer.Trainer(tp, precision=args.precision, use_graph=False, variables=he_init(g))
    tr.load(synthetic_batch(g, 0, args.batch))
    sel = [getattr(s, "inner", s) for s in tr.prog.steps if s.name == args.only]
    for _ in range(2):
        for s in sel:
            s(N.stream_ptr())
    torch.cuda.synchronize()
    L = N.lib()
    buf = (C.c_ulonglong * 20)()
    L.wap_gemm_trace_read.argtypes = [C.c_void_p, C.c_int]
    L.wap_gemm_trace_read(C.cast(buf, C.c_void_p), 20)
    for r in range(5):
        tot = buf[4 * r] or 1
        print(f"{ROLES[r]:44s} total {buf[4 * r]:>10d} cyc  waits: " +
              ", ".join(f"{100 * buf[4 * r + i] / tot:5.1f}%" for i in range(1, 4)))


if __name__ == "__main__":
    main()
