"""Small launches of every kernel family, for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize_kernels.py
    compute-sanitizer --tool synccheck python tools/sanitize_kernels.py
    compute-sanitizer --tool memcheck  python tools/sanitize_kernels.py

Covers the tcgen05 GEMM variants (PREC 1 / 3, CTA / CTA pair, halo window,
split-K, N = 64 pair mode, mask bits), the fused LRN+MaxPool forward and MaxPool+LRN
backward, the pool / LRN / xent / SGD kernels through one small AlexNet training
step, and the fused allreduce + SGD (world 1). Shapes are tiny: the sanitizers
slow kernels down by 10-100x.
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1811_01532_b200 import _native as N  # noqa: E402
from paper_1811_01532_b200 import interp, kernels as K, models  # noqa: E402


def gemms():
    g = torch.Generator(device="cuda").manual_seed(0)
    B, H, Ci, Co, k, pad = 1, 13, 64, 192, 3, 1
    xp = torch.zeros(B, H + pad, H + pad, Ci, device="cuda")
    xp[:, :H, :H] = torch.randn(B, H, H, Ci, device="cuda", generator=g)
    w = torch.randn(k, k, Ci, Co, device="cuda", generator=g)
    y = torch.zeros(B, H + pad, H + pad, Co, device="cuda")
    n = 0
    for prec in (1, 3):
        for cluster in (1, 2):
            for window in (0, -1):
                for bn in (0, 64, 128):
                    call = K.conv_fprop(xp, w, y, B=B, H=H, W=H, Ci=Ci, Co=Co, k=k, pad=pad, precision=prec,
                                        run=False)
                    d = type(call.desc).from_buffer_copy(call.desc)
                    d.cluster, d.window, d.block_n = cluster, window, bn
                    d.workspace, d.workspace_bytes = None, 0
                    try:
                        c = K.GemmCall(d)
                    except Exception:
                        continue
                    c()
                    n += 1
    dw = torch.zeros(k * k * Ci, Co, device="cuda")
    for prec in (1, 3):
        for sp in (0, 3):
            K.conv_wgrad(xp, y, dw, B=B, H=H, W=H, Ci=Ci, Co=Co, k=k, pad=pad, precision=prec, splits=sp)
            n += 1
    torch.cuda.synchronize()
    return n


def training_step():
    g = models.alexnet(2, image=67)
    rs = np.random.default_rng(0)
    bind = {}
    for nd in g:
        shape = tuple(nd.attr("shape") or ())
        if nd.kind.value == "Variable":
            bind[nd.id] = 0.05 * rs.standard_normal(shape)
        elif nd.id == "labels":
            lab = np.zeros(shape)
            lab[np.arange(shape[0]), rs.integers(0, shape[1], shape[0])] = 1
            bind[nd.id] = lab
        elif nd.kind.value == "Input":
            bind[nd.id] = rs.standard_normal(shape)
    out = interp.execute(g, bind, 0)
    torch.cuda.synchronize()
    return len(out)


def allreduce():
    from paper_1811_01532_b200.peer_memory import FusedAllReduce

    fr = FusedAllReduce(0, 1, 0, "p2p")
    var, grad = fr.allocate(4096 + 3)
    grad.fill_(1.0)
    fr.launch(0, 4099, 0.1, 0, N.stream_ptr())
    torch.cuda.synchronize()
    assert fr.status() == 0


if __name__ == "__main__":
    torch.cuda.set_device(0)
    N.lib()
    print("gemm launches:", gemms(), flush=True)
    print("training-step outputs:", training_step(), flush=True)
    allreduce()
    print("allreduce ok", flush=True)
