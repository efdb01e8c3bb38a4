"""Plain-PyTorch fp32 reference of the WAP training step (test infrastructure).

The same graph rules as oracle/interp_ref.py (which restates wap.interp,
interp.py:122-215), evaluated in fp32 with cuDNN / cuBLAS on the GPU with TF32
disabled: the "what does ordinary fp32 arithmetic give" yardstick for the
full-size multi-step parity test (tests/test_bench_parity_gpu.py). At AlexNet /
VGG-16 scale the first layers' weight gradients sum 10^5..10^6 products through
a dozen stacked layers, so fp32 itself deviates from the fp64 oracle by a
measurable amount; the test states its tolerance relative to this yardstick as
well as in absolute terms.

Decisions (ReLU masks, MaxPool argmaxes) can be pinned to a given set (the GPU
run's, tests/pinned_oracle.gpu_decisions) exactly as the oracle is pinned, so the
comparison measures arithmetic only. Never used by the product path.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F


def _nchw(x):
    return x.permute(0, 3, 1, 2)


def _nhwc(x):
    return x.permute(0, 2, 3, 1)


def _geom(attrs: dict, k: int) -> tuple[int, int]:
    return int(attrs.get("stride", 1)), int(attrs.get("padding", k // 2))


def _pool_windows(x, window: int, stride: int):
    """[window*window, B, Ho, Wo, C] stack of the pooling windows (row-major taps)."""
    b, h, w, c = x.shape
    ho, wo = (h - window) // stride + 1, (w - window) // stride + 1
    return torch.stack([x[:, i:i + stride * (ho - 1) + 1:stride, j:j + stride * (wo - 1) + 1:stride, :]
                        for i in range(window) for j in range(window)], 0)


def _lrn_scale(x, size, alpha, k):
    c = x.shape[-1]
    half = size // 2
    sq = F.pad(x * x, (half, half))
    acc = torch.zeros_like(x)
    for j in range(size):
        acc = acc + sq[..., j:j + c]
    return k + alpha * acc


def execute(graph, inputs: dict, decisions: dict | None = None, device="cuda") -> dict[str, np.ndarray]:
    """fp32 evaluation of `graph` (single device); returns the graph outputs as
    float64 numpy arrays. decisions: {"relu": {relu_input_id: bool mask},
    "pool": {pool_id: uint8 argmax (0xFF = no gradient)}} or None (own decisions)."""
    tf32 = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    try:
        return _execute(graph, inputs, decisions, device)
    finally:
        torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = tf32


def _execute(graph, inputs, decisions, device):
    from oracle.interp_ref import _topo

    nodes = {n.id: n for n in graph}
    pool_of = {(n.inputs[0], n.attrs["window"], n.attrs["stride"]): n.id for n in graph if n.kind.value == "MaxPool"}
    vals: dict[str, torch.Tensor] = {}
    argmax: dict[str, torch.Tensor] = {}

    def t(a):
        return torch.as_tensor(np.asarray(a, dtype=np.float32), device=device)

    def relu_mask(x_id, x):
        if decisions is not None:
            return torch.as_tensor(decisions["relu"][x_id], device=device)
        return x > 0

    for nid in _topo(graph):
        n = nodes[nid]
        kind, a = n.kind.value, n.attrs
        if kind in ("Input", "Variable"):
            vals[nid] = t(inputs[nid])
            continue
        ins = [vals[i] for i in n.inputs]
        if kind == "MatMul":
            x = ins[0].reshape(ins[0].shape[0], -1) if a.get("flatten_lhs") else ins[0]
            out = x @ ins[1]
        elif kind == "Conv2D":
            s, p = _geom(a, ins[1].shape[0])
            out = _nhwc(F.conv2d(_nchw(ins[0]), ins[1].permute(3, 2, 0, 1), stride=s, padding=p)).contiguous()
        elif kind == "BiasAdd":
            out = ins[0] + ins[1]
        elif kind == "ReLU":
            out = torch.where(relu_mask(n.inputs[0], ins[0]), ins[0], torch.zeros_like(ins[0]))
        elif kind == "SoftmaxXentLoss":
            z = ins[0] - ins[0].max(dim=1, keepdim=True).values
            logp = z - torch.log(torch.exp(z).sum(dim=1, keepdim=True))
            out = (-(ins[1] * logp).sum(dim=1)).sum().reshape(1) / ins[0].shape[0]
        elif kind in ("AddN", "AllReduceSum"):
            out = ins[0].clone()
            for v in ins[1:]:
                out = out + v
        elif kind == "GradMatMulW":
            x = ins[0].reshape(ins[0].shape[0], -1) if a.get("flatten_lhs") else ins[0]
            out = x.T @ ins[1]
        elif kind == "GradMatMulX":
            out = ins[0] @ ins[1].T
            if a.get("lhs_dims") is not None:
                out = out.reshape((out.shape[0], *a["lhs_dims"]))
        elif kind == "GradConv2DW":
            k = a["kernel_size"]
            s, p = _geom(a, k)
            x, dy = ins
            wsz = (dy.shape[3], x.shape[3], k, k)
            out = torch.nn.grad.conv2d_weight(_nchw(x), wsz, _nchw(dy), stride=s, padding=p).permute(2, 3, 1, 0)
            out = out.contiguous()
        elif kind == "GradConv2DX":
            dy, w = ins
            k = w.shape[0]
            s, p = _geom(a, k)
            hw = a.get("input_hw") or (dy.shape[1], dy.shape[2])
            isz = (dy.shape[0], w.shape[2], int(hw[0]), int(hw[1]))
            out = _nhwc(torch.nn.grad.conv2d_input(isz, w.permute(3, 2, 0, 1), _nchw(dy), stride=s, padding=p))
            out = out.contiguous()
        elif kind == "GradBias":
            out = ins[0].reshape(-1, ins[0].shape[-1]).sum(dim=0)
        elif kind == "GradReLU":
            out = ins[1] * relu_mask(n.inputs[0], ins[0])
        elif kind == "GradSoftmaxXent":
            out = (torch.softmax(ins[0], dim=1) - ins[1]) / a.get("denominator", ins[0].shape[0])
        elif kind == "SgdUpdate":
            out = ins[0] - a["learning_rate"] * ins[1]
        elif kind == "MaxPool":
            win = _pool_windows(ins[0], a["window"], a["stride"])
            if decisions is not None:
                g = torch.as_tensor(decisions["pool"][nid].astype(np.int64), device=device)
                own = win.argmax(dim=0)
                g = torch.where(g == 0xFF, own, g)
            else:
                g = win.argmax(dim=0)  # first maximum
            argmax[nid] = g
            out = torch.take_along_dim(win, g[None], dim=0)[0]
        elif kind == "GradMaxPool":
            x, dy = ins
            w_, s_ = a["window"], a["stride"]
            pid = pool_of[(n.inputs[0], w_, s_)]
            g = argmax[pid]
            if decisions is not None:  # 0xFF routes nowhere
                g = torch.where(torch.as_tensor(decisions["pool"][pid].astype(np.int64), device=device) == 0xFF,
                                torch.full_like(g, -1), g)
            _, ho, wo, _ = dy.shape
            out = torch.zeros_like(x)
            for i in range(w_):
                for j in range(w_):
                    sel = g == i * w_ + j
                    out[:, i:i + s_ * (ho - 1) + 1:s_, j:j + s_ * (wo - 1) + 1:s_, :] += torch.where(
                        sel, dy, torch.zeros_like(dy))
        elif kind == "LRN":
            out = ins[0] * _lrn_scale(ins[0], a["size"], a["alpha"], a["bias"]) ** (-a["beta"])
        elif kind == "GradLRN":
            x, dy = ins
            size, alpha, beta = a["size"], a["alpha"], a["beta"]
            s = _lrn_scale(x, size, alpha, a["bias"])
            tt = dy * x * s ** (-beta - 1.0)
            c = x.shape[-1]
            half = size // 2
            tp = F.pad(tt, (half, half))
            acc = torch.zeros_like(x)
            for j in range(size):
                acc = acc + tp[..., j:j + c]
            out = dy * s ** (-beta) - 2.0 * alpha * beta * x * acc
        else:
            raise ValueError(f"no torch fp32 rule for kind {kind}")
        vals[nid] = out
    return {o: vals[o].double().cpu().numpy() for o in graph.outputs}
