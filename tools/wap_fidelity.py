"""WAP cost-model fidelity: estimate_total's compute term at d = 1
vs the measured single-B200 step time per batch (profiles/r01/batch_times.json, from
tools/measure_batches.py), for the calibrated b200 profile and the reference's shipped
profiles. Writes a markdown table to stdout.

    python tools/wap_fidelity.py > profiles/r01/wap_fidelity.md
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1811_01532_b200 import ir, models, planner, workloads  # noqa: E402

meas = json.loads((ROOT / "profiles" / "r01" / "batch_times.json").read_text())["ms"]
profiles = ["b200"] + [p.stem for p in sorted((ROOT / "paper_1811_01532_b200" / "profiles").glob("*.json"))
                       if p.stem != "b200"]
print("# WAP Eq. (1) compute term vs measured single-B200 step time\n")
print("Predicted = `estimate_total(...).t_c_total` at d = 1 (planner.py, the reference's model); "
      "measured = CUDA-graph step time, 3xTF32 (profiles/r01/batch_times.json). The b200 profile "
      "was least-squares fitted to these times (tools/wau_sweep.py), so its column shows the "
      "model's residual shape error; the reference's own profiles show how far its toy "
      "hardware numbers are from a B200.\n")
print("| net | batch | GFLOP | measured ms | " + " | ".join(f"{p} pred ms (meas/pred)" for p in profiles) + " |")
print("|---|---|---|---|" + "---|" * len(profiles))
for net in ("alexnet", "vgg16"):
    for b, ms in sorted(meas[net].items(), key=lambda x: int(x[0])):
        wl = workloads.extract_workloads(ir.infer_shapes(models.MODELS[net](int(b))))
        cells = []
        for p in profiles:
            prof = planner.load_profile(p)
            est = planner.estimate_total(wl, 1, prof)
            pred = est.t_c_total * 1e3
            cells.append(f"{pred:.4g} ({ms / pred:.3g})")
        print(f"| {net} | {b} | {wl.total_flops / 1e9:.1f} | {ms:.3f} | " + " | ".join(cells) + " |")
