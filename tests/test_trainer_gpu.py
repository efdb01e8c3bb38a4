"""Single-GPU Trainer (in-place arenas, fused arena SGD, weight/bias gradients on a
parallel stream, whole step captured as one CUDA graph) against interp.execute of
the same training graph (fresh output buffers, one stream, no graph). Both run
the same kernels, so the loss and every updated variable must agree to fp32
rounding of identical arithmetic; the tolerance is kept tight (1e-6)."""

import numpy as np
import pytest
import torch

from oracle import interp_ref as O
from paper_1811_01532_b200 import interp, models, planner, trainer

pytestmark = pytest.mark.gpu


def _bindings(graph, seed=5):
    rs = np.random.default_rng(seed)
    out = {}
    for n in graph:
        shape = tuple(n.attr("shape") or ())
        if n.kind.value == "Variable":
            fan = int(np.prod(shape[:-1])) if len(shape) > 1 else 1
            out[n.id] = ((np.sqrt(2.0 / fan) if len(shape) > 1 else 0.01) * rs.standard_normal(shape)).astype(np.float32)
        elif n.id == "labels":
            lab = np.zeros(shape, np.float32)
            lab[np.arange(shape[0]), rs.integers(0, shape[1], shape[0])] = 1
            out[n.id] = lab
        elif n.kind.value == "Input":
            out[n.id] = rs.standard_normal(shape).astype(np.float32)
    return out


@pytest.mark.parametrize("net,kw", [("alexnet", {"batch": 4, "image": 99}), ("vgg16", {"batch": 2, "image": 32}),
                                    ("alexnet_like", {"batch": 8})])
def test_trainer_graph_step_matches_execute(cuda, net, kw, monkeypatch):
    # both sides use the default GEMM plans: independently autotuned Programs may pick
    # different split-K partitions, whose fp32 rounding differs by more than 1e-6
    monkeypatch.setenv("WAP_AUTOTUNE", "0")
    g = models.MODELS[net](**kw)
    bind = _bindings(g)
    tp = trainer.plan_training(g, 1, planner.load_profile("b200"), force_d=1)
    variables = {k: v for k, v in bind.items() if k not in ("images", "labels")}
    tr = trainer.Trainer(tp, variables=variables, use_graph=True)
    batch = {k: torch.from_numpy(bind[k]) for k in ("images", "labels")}
    loss = tr.step(batch, fetch=True)
    assert tr._captured
    ref = interp.execute(g, {k: v.astype(np.float64) for k, v in bind.items()}, 0)
    assert abs(loss - float(ref["loss"][0])) <= 1e-6 * max(1.0, abs(loss))
    got = tr.variables()
    for vid, val in got.items():
        dev = O.relative_deviation(val, ref[f"{vid}_upd"])
        assert dev < 1e-6, (vid, dev)


def test_step_async_matches_step(cuda, monkeypatch):
    """The overlapped input path (H2D on a copy stream, async loss D2H) computes the
    same three consecutive steps as the synchronous Trainer.step (to fp32 rounding)."""
    monkeypatch.setenv("WAP_AUTOTUNE", "0")
    g = models.MODELS["alexnet"](batch=4, image=99)
    b1, b2, b3 = _bindings(g, seed=11), _bindings(g, seed=12), _bindings(g, seed=13)
    variables = {k: v for k, v in b1.items() if k not in ("images", "labels")}
    tp = trainer.plan_training(g, 1, planner.load_profile("b200"), force_d=1)
    pinned = [{k: torch.from_numpy(b[k]).pin_memory() for k in ("images", "labels")} for b in (b1, b2, b3)]
    ta = trainer.Trainer(tp, variables=variables, use_graph=True)
    ta.step_async(pinned[0])
    ta.step_async(pinned[1])
    ta.step_async(pinned[2])  # staging slot 0 and its graph again
    la = ta.last_loss()
    tb = trainer.Trainer(tp, variables=variables, use_graph=True)
    tb.step(pinned[0])
    tb.step(pinned[1])
    lb = tb.step(pinned[2], fetch=True)
    # same default GEMM plans on both sides; agreement to rounding
    assert abs(la - lb) <= 1e-6 * max(1.0, abs(lb))
    va, vb = ta.variables(), tb.variables()
    for k in va:
        assert O.relative_deviation(va[k], vb[k]) < 1e-6, k
