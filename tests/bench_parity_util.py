"""Deterministic inputs of the benchmark-shape multi-step parity check
(tests/test_bench_parity_gpu.py, tools/parity_diag.py).

Per step k the batch is fresh: N(0,1) NHWC images and one-hot labels from
default_rng((seed, 1000 + k)). Weights are He-scaled (the reference's 0.1*N(0,1)
init saturates a 224x224 net's softmax, SURVEY §7 hard part 7), biases
0.01*N(0,1), all rounded to fp32 once; the oracle runs on those fp32 values in
fp64 and carries its own fp64 weights from step to step (interp.py:203-204).
"""

from __future__ import annotations

import numpy as np

SEED = 42


def variables(g, seed: int = SEED) -> dict[str, np.ndarray]:
    rs = np.random.default_rng(seed)
    out = {}
    for n in g:
        if n.kind.value != "Variable":
            continue
        shape = tuple(n.attr("shape"))
        if len(shape) > 1:
            out[n.id] = (np.sqrt(2.0 / np.prod(shape[:-1])) * rs.standard_normal(shape)).astype(np.float32)
        else:
            out[n.id] = (0.01 * rs.standard_normal(shape)).astype(np.float32)
    return out


def batch(g, step: int, seed: int = SEED) -> dict[str, np.ndarray]:
    shp = tuple(g.node("images").attr("shape"))
    classes = g.node("labels").attr("shape")[1]
    rs = np.random.default_rng((seed, 1000 + step))
    images = rs.standard_normal(shp, dtype=np.float32)
    labels = np.zeros((shp[0], classes), dtype=np.float32)
    labels[np.arange(shp[0]), rs.integers(0, classes, shp[0])] = 1.0
    return {"images": images, "labels": labels}
