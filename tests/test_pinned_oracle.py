"""The decision-pinned oracle hooks (tests/pinned_oracle.py) are a faithful
re-parameterisation of the oracle: fed the oracle's own ReLU masks and max-pool
argmaxes they reproduce its outputs bit for bit and count no flips, and fed a
flipped decision they follow it (CPU)."""

import numpy as np

from oracle import interp_ref as O
from paper_1811_01532_b200 import models

from .bench_parity_util import batch, variables
from .pinned_oracle import PinnedHooks


def _setup():
    g = models.alexnet(2, image=99)
    w = {k: v.astype(np.float64) for k, v in variables(g).items()}
    inp = {k: v.astype(np.float64) for k, v in batch(g, 0).items()}
    ref = O.execute(g, {**inp, **w}, 0, keep={n.id for n in g})
    relu = {n.inputs[0]: ref[n.id] > 0 for n in g if n.kind.value == "ReLU"}
    pool = {}
    for n in g:
        if n.kind.value == "MaxPool":
            pool[n.id] = O.maxpool(ref[n.inputs[0]], n.attrs["window"], n.attrs["stride"])[1].astype(np.uint8)
    return g, w, inp, ref, relu, pool


def test_own_decisions_reproduce_oracle_exactly():
    g, w, inp, ref, relu, pool = _setup()
    h = PinnedHooks(g, {"relu": relu, "pool": pool})
    out = O.execute(g, {**inp, **w}, 0, hooks=h.hooks())
    for k in out:
        assert np.array_equal(out[k], ref[k]), k
    assert sum(s["flips"] for s in h.stats.values()) == 0


def test_flipped_decisions_are_followed_and_counted():
    g, w, inp, ref, relu, pool = _setup()
    key = next(iter(relu))
    m = relu[key].copy()
    m[tuple(np.argwhere(~m)[0])] = True  # force one inactive unit on
    h = PinnedHooks(g, {"relu": {**relu, key: m}, "pool": pool})
    O.execute(g, {**inp, **w}, 0, hooks=h.hooks())
    relu_node = next(n.id for n in g if n.kind.value == "ReLU" and n.inputs[0] == key)
    assert h.stats[relu_node]["flips"] == 1
    assert h.stats[relu_node]["max_margin"] > 0
