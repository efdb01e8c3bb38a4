"""Where does a benchmark-shape step deviate from the fp64 oracle? (diagnostic)

Runs one training step of AlexNet-224 / VGG-16-224 at batch B on the GPU
(runtime.Program, every materialized tensor fetched) and through the oracle
(oracle/interp_ref.py with every node kept), on the bench-parity inputs
(tests/bench_parity_util.py), and prints the reference deviation metric per node
in topological order, plus for each GradMaxPool the fraction of input positions
whose "receives gradient" pattern differs (argmax flips between fp32 and fp64).

    python tools/parity_diag.py --net alexnet --batch 128
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="alexnet")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--top", type=int, default=200)
    args = ap.parse_args()
    import torch

    from bench_parity_util import batch, variables
    from oracle import interp_ref as O
    from paper_1811_01532_b200 import models
    from paper_1811_01532_b200.ir import topo_order
    from paper_1811_01532_b200.runtime import Program

    g = models.MODELS[args.net](args.batch)
    w0 = variables(g)
    inp = batch(g, 0)
    prog = Program(g)
    prog.bind({**{k: v for k, v in inp.items()}, **w0})
    prog.run()
    torch.cuda.synchronize()
    t0 = time.time()
    ref = O.execute(g, {**{k: v.astype(np.float64) for k, v in inp.items()},
                        **{k: v.astype(np.float64) for k, v in w0.items()}}, 0, keep={n.id for n in g})
    print(f"oracle {time.time() - t0:.1f} s", flush=True)
    rows = []
    for nid in topo_order(g):
        n = g.node(nid)
        if nid not in prog.t or n.kind.value in ("Input", "Variable"):
            continue
        got = prog.fetch(nid).astype(np.float64)
        r = np.asarray(ref[nid], dtype=np.float64)
        if got.shape != r.shape:
            continue
        dev = O.relative_deviation(got, r)
        l2 = float(np.linalg.norm(got - r) / max(np.linalg.norm(r), 1e-300))
        extra = ""
        if n.kind.value == "GradMaxPool":
            flips = np.mean((got != 0) != (r != 0))
            extra = f" nonzero-pattern mismatch {flips:.2e}"
        if n.kind.value in ("ReLU",):
            flips = np.mean((got > 0) != (r > 0))
            extra = f" sign mismatch {flips:.2e}"
        rows.append((nid, n.kind.value, dev, l2, extra))
    for nid, kind, dev, l2, extra in rows[: args.top]:
        print(f"{nid:28s} {kind:16s} max-dev {dev:.3e}  l2 {l2:.3e}{extra}")


if __name__ == "__main__":
    main()
