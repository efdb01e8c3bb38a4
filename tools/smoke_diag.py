"""Per-output deviation of the smoke() case (AlexNet topology, 99x99, b=2) against
the oracle, to localise a parity failure (test infrastructure / diagnostics)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from oracle import interp_ref as O  # noqa: E402
from paper_1811_01532_b200 import interp, models  # noqa: E402


def main():
    g = models.alexnet(2, image=99)
    rs = np.random.default_rng(0)
    bind = {}
    for n in g:
        shape = tuple(n.attr("shape") or ())
        if n.kind.value == "Variable":
            fan_in = int(np.prod(shape[:-1])) if len(shape) > 1 else 1
            bind[n.id] = (np.sqrt(2.0 / fan_in) if len(shape) > 1 else 0.01) * rs.standard_normal(shape)
        elif n.id == "labels":
            lab = np.zeros(shape)
            lab[np.arange(shape[0]), rs.integers(0, shape[1], shape[0])] = 1
            bind[n.id] = lab
        elif n.kind.value == "Input":
            bind[n.id] = rs.standard_normal(shape)
    got = interp.execute(g, bind, seed=0)
    ref = O.execute(g, bind, seed=0)
    rows = []
    for k in ref:
        dev = O.relative_deviation(got[k], ref[k])
        gd = ""
        base = k[:-4] if k.endswith("_upd") else None
        if base and base in bind:
            gd = f" grad-part {O.relative_deviation(got[k] - bind[base], ref[k] - bind[base]):.3e}"
        rows.append((dev, k, gd))
    for dev, k, gd in sorted(rows, reverse=True)[:12]:
        print(f"{k:24s} {dev:.3e}{gd}")


if __name__ == "__main__":
    main()
