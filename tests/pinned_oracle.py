"""Decision-pinned oracle hooks for full-size parity (test infrastructure).

ReLU masks and MaxPool argmaxes make the training step a piecewise-linear
function of its inputs: at AlexNet-224 b=128, ~1e-6 of the ReLU pre-activations
and of the pooling windows sit within fp32 rounding (~1e-6 relative) of their
decision threshold, so ANY fp32 implementation takes a few hundred different
branches than the fp64 oracle (interp.py:168-169,197-198 and the MaxPool
extension), and the gradient of each flipped unit changes by O(1). Elementwise
comparison of gradients against the unpinned oracle therefore measures those
flips, not the arithmetic (measured: tools/parity_diag.py, profiles/r02).

The check is split in two, each against a stated bound:
1. Decisions: every ReLU / MaxPool decision the GPU took either equals the
   oracle's own, or is a near-tie: the pre-activation of a flipped ReLU is within
   `TIE` x max|x| of 0, the oracle's max of a flipped window beats the GPU's
   choice by at most `TIE` x max|x| (fractions and margins are reported).
   TIE = 1e-3 is ten times the forward drift the arithmetic bound below admits
   (after k steps the GPU's fp32 weights and the oracle's fp64 weights differ by
   up to ~1e-4 of max|w|, measured r02); a wrong mask or argmax anywhere in the
   step would show margins of O(1).
2. Arithmetic: the fp64 oracle evaluated ON THE GPU'S DECISIONS (these hooks:
   ReLU / GradReLU take the GPU mask, MaxPool / GradMaxPool the GPU argmax)
   must match loss, weights and updates to 1e-4 on the reference metric.
"""

from __future__ import annotations

import numpy as np

from oracle import interp_ref as O

TIE = 1e-3


def gpu_decisions(prog, graph) -> dict:
    """ReLU masks keyed by the ReLU's input id, MaxPool argmax (window index, 0xFF =
    no gradient) keyed by the MaxPool id, read from a Program after a step."""
    import torch

    relu, pool = {}, {}
    for n in graph:
        if n.kind.value == "ReLU":
            if n.id not in prog.t:
                raise KeyError(f"ReLU output {n.id!r} not materialized")
            relu[n.inputs[0]] = prog.fetch(n.id) > 0
        elif n.kind.value == "MaxPool":
            t = prog.t[f"{n.id}::argmax"]
            b, h, w, c = t.dims
            a = t.buf.view(b, h + t.pad, w + t.pad, t.ld)[:, :h, :w, :c]
            torch.cuda.synchronize()
            pool[n.id] = a.cpu().numpy().copy()
    return {"relu": relu, "pool": pool}


class PinnedHooks:
    """oracle.execute hooks that follow the GPU's decisions and record how the
    oracle's own decisions differ."""

    def __init__(self, graph, decisions: dict):
        self.d = decisions
        self.pool_of = {}
        for n in graph:
            if n.kind.value == "MaxPool":
                self.pool_of[(n.inputs[0], n.attrs["window"], n.attrs["stride"])] = n.id
        self.stats: dict[str, dict] = {}

    def hooks(self) -> dict:
        return {"ReLU": self._relu, "GradReLU": self._grad_relu, "MaxPool": self._pool,
                "GradMaxPool": self._grad_pool}

    def _relu(self, node, ins):
        x = ins[0]
        m = self.d["relu"][node.inputs[0]]
        own = x > 0
        flips = m != own
        scale = float(np.abs(x).max(initial=0.0)) or 1.0
        margin = float(np.abs(x[flips]).max(initial=0.0)) / scale
        self.stats[node.id] = {"kind": "ReLU", "flips": int(flips.sum()), "frac": float(flips.mean()),
                               "max_margin": margin}
        return np.where(m, x, 0.0)

    def _grad_relu(self, node, ins):
        return ins[1] * self.d["relu"][node.inputs[0]]

    def _arg(self, node_id, x, window, stride):
        vals, own = O.maxpool(x, window, stride)
        gpu = self.d["pool"][node_id].astype(np.int64)
        none = gpu == 0xFF
        g = np.where(none, own, gpu)
        return vals, own, g, none

    def _pool(self, node, ins):
        x = ins[0]
        w, s = node.attrs["window"], node.attrs["stride"]
        vals, own, g, none = self._arg(node.id, x, w, s)
        _, ho, wo, _ = vals.shape
        stack = np.stack([O._win(x, i, j, s, ho, wo) for i in range(w) for j in range(w)], axis=0)
        picked = np.take_along_axis(stack, g[None], axis=0)[0]
        flips = (g != own) & ~none
        scale = float(np.abs(x).max(initial=0.0)) or 1.0
        gap = float((vals - picked)[flips].max(initial=0.0)) / scale
        self.stats[node.id] = {"kind": "MaxPool", "flips": int(flips.sum()), "frac": float(flips.mean()),
                               "max_margin": gap}
        return picked

    def _grad_pool(self, node, ins):
        x, dy = ins
        w, s = node.attrs["window"], node.attrs["stride"]
        pid = self.pool_of[(node.inputs[0], w, s)]
        gpu = self.d["pool"][pid].astype(np.int64)
        _, ho, wo, _ = dy.shape
        dx = np.zeros_like(x)
        for i in range(w):
            for j in range(w):
                sel = gpu == i * w + j  # 0xFF routes nowhere (its GradReLU mask is 0)
                dx[:, i:i + s * (ho - 1) + 1:s, j:j + s * (wo - 1) + 1:s, :] += np.where(sel, dy, 0.0)
        return dx
