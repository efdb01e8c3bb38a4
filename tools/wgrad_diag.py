"""Is the first-layer weight-gradient deviation made by the wgrad GEMM or
inherited from its upstream gradient dY? (diagnostic)

One VGG-16 / AlexNet step on the GPU (runtime.Program) and through the
decision-pinned fp64 oracle (tests/pinned_oracle.py). For the first conv:
  gemm      = dev(dW_gpu, dW64(x, dY_gpu))    the wgrad GEMM's own error
  inherited = dev(dW64(x, dY_gpu), dW_oracle) the error carried in by dY
plus dev(dY_gpu, dY_oracle) and the cancellation ratio sum|x*dy| / |sum x*dy|.
    python tools/wgrad_diag.py --net vgg16 --batch 32
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="vgg16")
    ap.add_argument("--batch", type=int, default=32)
    args = ap.parse_args()
    import torch

    from bench_parity_util import batch, variables
    from oracle import interp_ref as O
    from paper_1811_01532_b200 import models
    from paper_1811_01532_b200.runtime import Program
    from pinned_oracle import PinnedHooks, gpu_decisions

    g = models.MODELS[args.net](args.batch, lr=1e-3) if args.net == "vgg16" else models.MODELS[args.net](args.batch)
    w0 = variables(g)
    inp = batch(g, 0)
    prog = Program(g)
    prog.bind({**inp, **w0})
    prog.run()
    torch.cuda.synchronize()
    dec = gpu_decisions(prog, g)
    dy_id, dw_id = "d_conv1_zb", "d_conv1_w"
    dy_gpu = prog.fetch(dy_id).astype(np.float64)
    dw_gpu = prog.fetch(dw_id).astype(np.float64)
    hooks = PinnedHooks(g, dec)
    ref = O.execute(g, {**{k: v.astype(np.float64) for k, v in inp.items()},
                        **{k: v.astype(np.float64) for k, v in w0.items()}}, 0, keep={dy_id, dw_id},
                    hooks=hooks.hooks())
    conv = g.node("conv1")
    k = g.node("conv1_w").attr("shape")[0]
    s, p = O._geom(conv.attrs, k)
    x = inp["images"].astype(np.float64)
    dw64 = O.conv2d_grad_w(x, dy_gpu, k, s, p)
    absw = O.conv2d_grad_w(np.abs(x), np.abs(dy_gpu), k, s, p)
    print(f"{args.net} b={args.batch}: dY dev {O.relative_deviation(dy_gpu, ref[dy_id]):.3e}")
    print(f"  gemm      dev(dW_gpu, dW64(x, dY_gpu))   {O.relative_deviation(dw_gpu, dw64):.3e}")
    print(f"  inherited dev(dW64(x, dY_gpu), dW_oracle) {O.relative_deviation(dw64, ref[dw_id]):.3e}")
    print(f"  total     dev(dW_gpu, dW_oracle)          {O.relative_deviation(dw_gpu, ref[dw_id]):.3e}")
    print(f"  cancellation max(sum|x dy|) / max|dW| = {absw.max() / np.abs(ref[dw_id]).max():.1f}")


if __name__ == "__main__":
    main()
