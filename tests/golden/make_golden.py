"""Generate golden fixtures from the REFERENCE implementation (run in the build
container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/ref_outputs.npz (reference `wap.interp.execute` outputs on
reference models, single-device and transformed, seed 42, reference-generated
inputs) and tests/golden/planner.json (reference `select_parallelism` on the
224x224 AlexNet / VGG-16 workloads over the small-to-large batch sweep, every
float as its exact hex string). The GPU box has no /root/reference; these
files let the oracle and the device WAU be pinned there too.
"""
import json
import sys
from importlib import import_module
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

import wap  # noqa: E402  (the reference)

from paper_1811_01532_b200 import ir, models, workloads  # noqa: E402

SEED = 42
CASES = [("mlp", 64, (1, 4)), ("alexnet_like", 16, (1, 2, 4)), ("vgg16_like", 8, (1, 2))]
BIG = 20000
SAMPLE = 2048
SWEEP = (16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512)


def ref_outputs():
    tf = import_module("wap.transform")
    arrays = {}
    for name, batch, ds in CASES:
        g = getattr(import_module("wap.models"), name)(batch)
        inputs = wap.generate_inputs(g, SEED)
        for d in ds:
            gg = g if d == 1 else tf.transform(g, wap.ParallelPlan(d, tuple(range(d)), (), 0.0))[0]
            outs = wap.execute(gg, inputs, SEED)
            for k, v in outs.items():
                # replicas of an update are copies of one tensor: keep dev0 (+ every loss)
                if d > 1 and not (k.endswith("/dev0") or k.startswith("loss")):
                    continue
                key = f"{name}|{batch}|{d}|{k}"
                if v.size > BIG:  # large tensors: a fixed sample plus exact moments
                    flat = v.reshape(-1)
                    idx = np.linspace(0, flat.size - 1, SAMPLE).astype(np.int64)
                    arrays[key + "|sample"] = flat[idx]
                    arrays[key + "|moments"] = np.array([flat.sum(), (flat * flat).sum(), float(flat.size)])
                else:
                    arrays[key] = v
    np.savez_compressed(HERE / "ref_outputs.npz", **arrays)
    return len(arrays)


def planner_sweep():
    doc = {"python": list(sys.version_info[:3]), "numpy": np.__version__, "cases": []}
    profs = {p: wap.load_profile(p) for p in ("pcie-box", "nvlink-box")}
    profs["b200"] = wap.load_profile(str(HERE.parents[1] / "paper_1811_01532_b200" / "profiles" / "b200.json"))
    for net in ("alexnet", "vgg16"):
        for G in SWEEP:
            mine = workloads.extract_workloads(ir.infer_shapes(models.MODELS[net](G)))
            # feed the reference planner the same per-layer counts (plain dataclasses)
            rw = wap.NetworkWorkload(
                tuple(wap.LayerWorkload(l.layer, wap.OpKind(l.kind.value), l.flops_fwd, l.flops_bwd,
                                        l.weight_bytes, l.activation_bytes, l.batch) for l in mine.layers),
                mine.global_batch, mine.total_weight_bytes)
            for pname, prof in profs.items():
                for algo in ("ring", "naive_all_to_all"):
                    plan = wap.select_parallelism(rw, tuple(range(8)), prof, algo)
                    doc["cases"].append({
                        "net": net, "G": G, "profile": pname, "algo": algo, "d": plan.d,
                        "power": plan.predicted_power.hex(),
                        "estimates": [[e.d, e.t_c_total.hex(), e.t_s_total.hex(), e.predicted_throughput.hex()]
                                      for e in plan.estimates],
                        "layers": [[l.flops_fwd, l.flops_bwd, l.weight_bytes] for l in mine.layers],
                    })
    (HERE / "planner.json").write_text(json.dumps(doc, indent=1) + "\n")
    return len(doc["cases"])


if __name__ == "__main__":
    print("ref outputs:", ref_outputs())
    print("planner cases:", planner_sweep())
