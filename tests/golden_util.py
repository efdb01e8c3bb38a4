"""Loading and checking the reference-generated golden fixtures."""
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
SEED = 42


@lru_cache(maxsize=1)
def ref_outputs() -> dict:
    with np.load(GOLDEN / "ref_outputs.npz") as z:
        return {k: z[k] for k in z.files}


def cases():
    """(model, batch, d) triples present in the fixture."""
    out = sorted({tuple(k.split("|")[:3]) for k in ref_outputs()})
    return [(m, int(b), int(d)) for m, b, d in out]


def expected(model: str, batch: int, d: int) -> dict:
    """output id -> ndarray, or (sample, moments) for large tensors."""
    res = {}
    prefix = f"{model}|{batch}|{d}|"
    for k, v in ref_outputs().items():
        if not k.startswith(prefix):
            continue
        rest = k[len(prefix):]
        if rest.endswith("|sample") or rest.endswith("|moments"):
            name, part = rest.rsplit("|", 1)
            res.setdefault(name, {})[part] = v
        else:
            res[rest] = v
    return res


def deviation_vs_golden(value: np.ndarray, golden) -> float:
    """Reference-style relative deviation (interp.py:242-246) against a golden entry."""
    value = np.asarray(value, dtype=np.float64)
    if isinstance(golden, dict):
        flat = value.reshape(-1)
        idx = np.linspace(0, flat.size - 1, golden["sample"].size).astype(np.int64)
        s = golden["sample"]
        scale = max(np.abs(s).max(), np.abs(flat[idx]).max(), 1e-30)
        dev = np.abs(flat[idx] - s).max() / scale
        m = golden["moments"]
        dev_sum = abs(flat.sum() - m[0]) / max(np.abs(flat).sum(), 1e-30)
        dev_sq = abs((flat * flat).sum() - m[1]) / max(m[1], 1e-30)
        return float(max(dev, dev_sum, dev_sq))
    g = np.asarray(golden, dtype=np.float64)
    scale = max(np.abs(value).max(initial=0), np.abs(g).max(initial=0), 1e-30)
    return float(np.abs(value - g).max(initial=0) / scale)


@lru_cache(maxsize=1)
def planner_cases() -> dict:
    return json.loads((GOLDEN / "planner.json").read_text())
