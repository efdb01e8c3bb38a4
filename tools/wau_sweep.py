"""Calibrate the b200 DeviceProfile and evaluate WAP's GPU-count choice
(BASELINE config 4: small-to-large minibatch sweep, G = 16..512).

Inputs: measured single-GPU step times vs per-GPU batch
(tools/measure_batches.py -> profiles/r01/batch_times.json).

Calibration (same 9-field schema as the reference profiles, planner.py:34-44):
  WAU compute model per layer: t = work / (peak * work/(work+knee)) = (work + knee)/peak,
  so a whole step is T(b) = (W(b) + L*knee)/peak with W(b) the WAP-counted FLOPs.
  A least-squares fit of the measured T(b) on W(b) (relative error, both nets)
  gives peak and knee. link_bandwidth = 725 GB/s, the measured 8-rank NCCL
  allreduce bus bandwidth on this pool's B200s (B200_PROFILING.md); latencies 1.5 us per ring step (NVLink hop), 20 us per naive transfer.

Sweep: multi-GPU step time = measured single-GPU compute at b = G/d
  + per-layer ring allreduce 2W_l(d-1)/d/busbw + 2(d-1)*1.5us (not overlapped,
  the same additive assumption as WAP's Eq. 1). Only one GPU is reachable in this
  build, so the d>1 columns are measured compute + modeled communication.
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1811_01532_b200 import ir, models, planner, workloads  # noqa: E402

BUSBW = 725e9
CHUNK_LAT = 1.5e-6
LINK_LAT = 20e-6
SWEEP = (16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512)
PARAMS = {"alexnet": 61_100_840, "vgg16": 138_357_544}


def wl_of(net, G):
    return workloads.extract_workloads(ir.infer_shapes(models.MODELS[net](G)))


def fit(meas):
    X, y, L = [], [], []
    for net, tab in meas.items():
        for b, ms in tab.items():
            w = wl_of(net, int(b))
            X.append((w.total_flops, len(w.layers)))
            y.append(ms * 1e-3)
    X = np.array(X, dtype=float)
    y = np.array(y)
    # T = W/peak + L*knee/peak  ->  y = a*W + c*L, weights 1/y (relative error)
    A = np.stack([X[:, 0], X[:, 1]], axis=1) / y[:, None]
    coef, *_ = np.linalg.lstsq(A, np.ones_like(y), rcond=None)
    a, c = coef
    peak = 1.0 / a
    knee = c * peak
    return peak, knee


def comm(net, d):
    """One ring allreduce per layer (weights + bias), as the runtime issues them."""
    if d == 1:
        return 0.0
    w = PARAMS[net] * 4
    n_layers = 8 if net == "alexnet" else 16
    return 2 * w * (d - 1) / d / BUSBW + n_layers * 2 * (d - 1) * CHUNK_LAT


def interp_ms(tab, b):
    bs = sorted(int(k) for k in tab)
    if b in bs:
        return tab[str(b)] if str(b) in tab else tab[b]
    vals = [tab[str(k)] if str(k) in tab else tab[k] for k in bs]
    return float(np.interp(b, bs, vals))


def main(path):
    doc = json.loads(Path(path).read_text())
    meas = doc["ms"]
    peak, knee = fit(meas)
    prof = {"name": "b200", "peak_flops": float(f"{peak:.4g}"), "efficiency_knee_flops": float(f"{knee:.4g}"),
            "link_bandwidth": BUSBW, "link_latency": LINK_LAT, "allreduce_chunk_latency": CHUNK_LAT,
            "power_idle": 140.0, "power_peak": 1000.0, "host_power": 250.0}
    out = {"profile": prof, "fit": {"peak_flops": peak, "knee": knee}, "sweep": {}}
    P = planner.DeviceProfile(**prof)
    lines = ["| net | G | best d (img/s) | WAP d* (img/s) | d*/best | per-GPU ratio | all d (img/s) |",
             "|---|---|---|---|---|---|---|"]
    worst = 1.0
    for net, tab in meas.items():
        for G in SWEEP:
            thr = {}
            for d in range(1, 9):
                if G % d:
                    continue
                b = G // d
                t = interp_ms(tab, b) * 1e-3 + comm(net, d)
                thr[d] = G / t
            best = max(thr, key=thr.get)
            plan = planner.select_parallelism(wl_of(net, G), tuple(range(8)), P)
            ds = plan.d
            ratio = thr[ds] / thr[best]
            pg = (thr[ds] / ds) / max(v / d for d, v in thr.items())
            worst = min(worst, ratio)
            out["sweep"].setdefault(net, {})[G] = {"best_d": best, "wau_d": ds, "ratio": ratio, "per_gpu_ratio": pg,
                                                   "img_s": {d: round(v, 1) for d, v in thr.items()}}
            lines.append(f"| {net} | {G} | {best} ({thr[best]:.0f}) | {ds} ({thr[ds]:.0f}) | {ratio:.3f} | {pg:.3f} | "
                         + ", ".join(f"{d}:{v:.0f}" for d, v in thr.items()) + " |")
    out["worst_ratio"] = worst
    return prof, out, "\n".join(lines)


if __name__ == "__main__":
    prof, out, table = main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01/batch_times.json")
    print(json.dumps(prof, indent=2))
    print(table)
    print("worst WAP/best throughput ratio:", round(out["worst_ratio"], 4))
    if "--write" in sys.argv:
        (ROOT / "paper_1811_01532_b200" / "profiles" / "b200.json").write_text(json.dumps(prof, indent=2) + "\n")
        (ROOT / "profiles" / "r01" / "wau_sweep.json").write_text(json.dumps(out, indent=1) + "\n")
        (ROOT / "profiles" / "r01" / "wau_sweep.md").write_text(
            "# WAP GPU-count choice vs best (G = 16..512)\n\n"
            "Measured single-B200 step times (3xTF32) at b = G/d plus a modeled NCCL ring allreduce\n"
            "(725 GB/s bus bandwidth, 1.5 us per ring step per layer), calibrated b200 profile.\n\n" + table + "\n")
