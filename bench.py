"""Benchmark: WAP data-parallel training step (AlexNet / VGG-16) on B200.

Contract (see task / DESIGN.md "Measurement"):
  python bench.py --gpus N --steps K --warmup W          (N > 1 under torchrun)
  python bench.py --impl reference ...                   CPU oracle port on host cores
prints ONE JSON line on rank 0.

The metric is "AlexNet/VGG-16 train images/sec": the top-level record is AlexNet
b=128/GPU (configs[1]); the same line carries a full VGG-16 b=32/GPU record
(configs[2]) under "vgg16" (same fields, same timing rules).

value    images/sec of the whole job: global batch G = b*N per step, K steps
         timed with CUDA events between barriers, max over ranks; inputs
         resident in HBM (one synthetic batch staged before timing; the
         per-step working set, >= 0.5 GB of activations, exceeds the 126 MB L2).
e2e      the same metric through the public API Trainer.step_async(batch) with
         pinned host buffers: H2D of the shard + step + D2H of the loss, timed.
roofline dominant kernel (a tcgen05 GEMM) from an instrumented pass with CUDA
         events around every launch of the same step. achieved = WAP-counted
         algorithmic FLOPs / kernel time; peak = the tcgen05 kind::tf32 issue rate
         measured by a probe kernel in this same run (wap_tf32_probe).
power    NVML board power over a >= 5 s window of back-to-back steps, against
         WAP's estimate_power (planner.py:198-214 of the reference).
cpu_baseline  BASELINE configs[0] ("Config 1"): WAU + transform + one
         fp64 step of the transformed AlexNet-224 graph at G=64, seed 42, through
         the oracle port, on all host cores and on one BLAS thread.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "AlexNet/VGG-16 train images/sec at 1/2/4/8 B200; WAP-chosen GPU count vs best"
UNIT = "images/sec"
DEFAULT_BATCH = {"alexnet": 128, "vgg16": 32}
# fallback only when the in-run probe cannot run: r01 tools/mma_probe.cu on this pool
# (profiles/r01/mma_probe.txt: 2048 MAC/clk/SM for N >= 128)
TF32_MMA_PEAK_FALLBACK = 1116.4
POWER_WINDOW_S = 5.0


def peaks():
    """(HBM GB/s, bf16 TFLOP/s, source) from the driver-written MEASURED_PEAKS.json, else the
    fallback of /opt/skills/guides/B200_PROFILING.md."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), float(d.get("bf16_tflops", 1590.0)), "measured"
    return 6650.0, 1590.0, "fallback"


def measure_tf32_peak(iters: int = 20000, reps: int = 3) -> dict:
    """tcgen05.mma kind::tf32 issue rate of this GPU, now (csrc/probe.cu)."""
    import torch

    from paper_1811_01532_b200 import _native as N

    L = N.lib()
    s = torch.cuda.current_stream()
    N.check(L.wap_tf32_probe(1000, N.stream_ptr()), "tf32 probe")
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        N.check(L.wap_tf32_probe(iters, N.stream_ptr()), "tf32 probe")
        e1.record(s)
        e1.synchronize()
        best = max(best, L.wap_tf32_probe_flops(iters) / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return {"tflops": round(best, 1), "how": f"wap_tf32_probe: 148 CTAs x {iters}x4 tcgen05.mma.kind::tf32 "
                                              "M128 N256 K8 from resident smem, CUDA events, best of 3"}


def traffic_of(model: str, step: str):
    """DRAM bytes per launch of `step` from the committed ncu --set full captures
    (profiles/traffic.json, written by tools/capture_traffic.sh), or None."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    e = json.loads(p.read_text()).get(model, {}).get(step)
    return None if e is None else int(e["traffic_bytes"])


class ClockSampler:
    """nvidia-smi sampling of SM clocks / throttle reasons / board power.

    Sampling starts before the warm-up (nvidia-smi can take seconds to attach on a
    fresh box); samples are selected afterwards by their own timestamps for each
    window of interest (the timed region, the power window). Stopping never
    blocks: a sampler that does not exit after SIGTERM/SIGKILL is abandoned."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def stop(self) -> None:
        if self.proc is None:
            return
        self.proc.terminate()
        out = ""
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                out = ""
        self.lines = [l for l in (out or "").splitlines() if l.strip()]
        self.proc = None

    @staticmethod
    def _stamp(ts: str):
        import datetime

        try:
            return datetime.datetime.strptime(ts.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return None

    def _rows(self):
        rows = []
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 10:
                continue
            try:
                pw = float(f[4]) if f[4] not in ("", "[N/A]", "N/A") else float("nan")
                rows.append((self._stamp(f[0]), float(f[2]), float(f[3]), f[6:10], pw))
            except ValueError:
                continue
        return rows

    def summary(self, window=None) -> dict:
        rows = self._rows()
        sel = rows
        if window is not None:
            t0, t1 = window
            inside = [r for r in rows if r[0] is not None and t0 - 0.05 <= r[0] <= t1 + 0.05]
            if inside:
                sel = inside
        reasons = {n for r in sel for n, v in zip(self.NAMES, r[3]) if v.lower() == "active"}
        sm = [r[1] for r in sel]
        pw = [r[4] for r in sel if r[4] == r[4]]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": sel[-1][2] if sel else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "window": "timed region" if (window is not None and sel is not rows) else "whole run",
                "power_w": round(float(np.median(pw)), 1) if pw else None}


def synthetic_batch(model_graph, rank: int, b: int, seed: int = 42):
    """ImageNet-shaped synthetic shard: N(0,1) NHWC images, one-hot labels (host, pinned)."""
    import torch

    shp = tuple(model_graph.node("images").attr("shape"))
    classes = model_graph.node("labels").attr("shape")[1]
    rs = np.random.default_rng((seed, rank))
    images = rs.standard_normal((b,) + shp[1:], dtype=np.float32)
    labels = np.zeros((b, classes), dtype=np.float32)
    labels[np.arange(b), rs.integers(0, classes, b)] = 1.0
    return {"images": torch.from_numpy(images).pin_memory(), "labels": torch.from_numpy(labels).pin_memory()}


def he_init(graph, seed: int = 42) -> dict:
    rs = np.random.default_rng(seed)
    out = {}
    for n in graph:
        if n.kind.value == "Variable":
            shape = tuple(n.attr("shape"))
            if len(shape) > 1:
                out[n.id] = (np.sqrt(2.0 / np.prod(shape[:-1])) * rs.standard_normal(shape)).astype(np.float32)
            else:
                out[n.id] = np.zeros(shape, dtype=np.float32)
    return out


def run_ours(args, model, rank, world, local_rank, tf32_peak):
    """Measure one network; returns (record or None on ranks > 0)."""
    import torch
    import torch.distributed as dist

    from paper_1811_01532_b200 import _native as N
    from paper_1811_01532_b200 import models, planner, trainer
    from paper_1811_01532_b200.ir import infer_shapes
    from paper_1811_01532_b200.runtime import _GemmStep
    from paper_1811_01532_b200.workloads import extract_workloads

    dev = torch.device("cuda", local_rank)
    b = args.batch or DEFAULT_BATCH[model]
    G = b * world
    graph = models.MODELS[model](G)
    prof = planner.load_profile("b200")
    tplan = trainer.plan_training(graph, world, prof, force_d=world)
    # what the WAU would choose for this global batch on 8 GPUs (reported)
    wl = extract_workloads(infer_shapes(graph))
    wau8 = planner.select_parallelism_device(wl, tuple(range(8)), prof)
    # He-scaled initial weights: the reference's 0.1*N(0,1) init overflows a
    # 224x224 net within a few SGD steps (logits ~1e5); timing is unaffected.
    tr = trainer.Trainer(tplan, rank=rank, precision=args.precision, use_graph=not args.no_graph,
                         variables=he_init(graph))
    batch = synthetic_batch(graph, rank, b)
    tr.load(batch)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clk = ClockSampler(local_rank).start()
    # idle board power (profile calibration: power_idle), before this network's work
    torch.cuda.synchronize()
    time.sleep(0.5)
    i0 = time.time()
    time.sleep(1.5)
    idle_window = (i0, time.time())
    for _ in range(args.warmup):
        tr.run()
    barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    e0.record(stream)
    for _ in range(args.steps):
        tr.run()
    e1.record(stream)
    torch.cuda.synchronize()
    timed_window = (w0, time.time())
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    value = G / (ms / 1e3)

    # ---- end to end through the public API: every step copies its shard H2D from
    # pinned host memory (copy stream, overlapping the previous step) and copies the
    # loss D2H (Trainer.step_async); the copy stream joins after e0 so every H2D is
    # inside the timed region ----
    e2e_steps = max(3, min(args.steps, 10))
    tr.step_async(batch)  # warm the overlapped input path
    barrier()
    h0 = time.perf_counter()
    e0.record(stream)
    tr.copy_stream.wait_stream(stream)
    for _ in range(e2e_steps):
        tr.step_async(batch)
    e1.record(stream)
    loss = tr.last_loss()
    torch.cuda.synchronize()
    host_ms = (time.perf_counter() - h0) * 1e3 / e2e_steps
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / e2e_steps)
    h2d = sum(v.numel() * 4 for v in batch.values())

    # ---- power window: back-to-back steps for >= 5 s (NVML's power reading is a
    # ~1 s average, so the short timed region cannot resolve it) ----
    barrier()
    n_pw = max(1, int(POWER_WINDOW_S * 1e3 / ms) + 1)
    p0 = time.time()
    for i in range(n_pw):
        tr.run()
        if i % 64 == 63:
            torch.cuda.synchronize()  # bound the queue; the window is wall-clock
    torch.cuda.synchronize()
    p1 = time.time()
    clk.stop()
    clocks = clk.summary(timed_window)
    # drop the first second (the NVML average still carries the pre-window level)
    pw = clk.summary((p0 + 1.0, p1))
    idle = clk.summary(idle_window)
    barrier()

    # ---- instrumented pass: per-launch CUDA events over the same step ----
    prog = tr.prog
    per = {}
    reps = 3
    for _ in range(reps):
        evs = []
        # keep the host ahead of the device: a queued spin lets every launch below be
        # enqueued before the device reaches it, so the events bracket device time only
        torch.cuda._sleep(20_000_000)
        for st in prog.steps:
            st = getattr(st, "inner", st)  # parallel-stream steps are timed on this stream
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st(N.stream_ptr())
            z.record(stream)
            evs.append((st, a, z))
        torch.cuda.synchronize()
        for st, a, z in evs:
            per.setdefault(st.name, [0.0, st])[0] += a.elapsed_time(z) / reps
    total_kernel_ms = sum(v[0] for v in per.values())
    gemms = [(v[0], v[1]) for v in per.values() if isinstance(v[1], _GemmStep)]
    gemm_ms = sum(m for m, _ in gemms)
    gemm_flops = sum(s.alg_flops for _, s in gemms)
    dom_ms, dom = max(gemms, key=lambda x: x[0])
    hbm_peak, bf16_peak, peak_src = peaks()
    pipe_factor = 3 if args.precision == 3 else 1
    # HBM-bound kernels (im2col, pool, LRN, bias-grad, xent, SGD): algorithmic bytes / event time
    ew = [(v[0], v[1]) for v in per.values() if getattr(v[1], "alg_bytes", 0) > 0]
    ew_ms = sum(m for m, _ in ew)
    ew_bytes = sum(st.alg_bytes for _, st in ew)
    ew_top = sorted(ew, key=lambda x: -x[0])[:6]
    achieved = dom.alg_flops / (dom_ms * 1e-3) / 1e12
    launches = prog.launches_per_step() if not tr._captured else _count_launches(prog)
    peak = tf32_peak["tflops"]
    gemm_alg_tflops = gemm_flops / (gemm_ms * 1e-3) / 1e12

    if rank != 0:
        return None
    est = tplan.plan.chosen
    pw_pred = planner.estimate_power(tplan.plan, wl, prof)
    # estimate_power's GPU term is idle + (peak - idle) * util (planner.py:198-214 of the
    # reference): the power_peak that reproduces the measured load power at this util
    util = ((pw_pred - prof.host_power) / tplan.plan.d - prof.power_idle) / (prof.power_peak - prof.power_idle)
    fit_peak = None
    if pw["power_w"] and idle["power_w"] and util > 0:
        fit_peak = round(idle["power_w"] + (pw["power_w"] - idle["power_w"]) / util, 1)
    return {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic (N(0,1) NHWC images, one-hot labels, He-scaled random-init weights)",
        "impl": "ours",
        "config": {"workload": f"{model} fp32 training, batch {b}/GPU, 224x224x3 synthetic ImageNet shape",
                   "network": model, "global_batch": G, "batch_per_gpu": b, "image": 224,
                   "parallelism": f"dp{world} replicated-variables (WAP transform, forced d={world})",
                   "gemm_precision": "3xTF32 (fp32-accurate)" if args.precision == 3 else "TF32",
                   "cuda_graph": tr._captured, "l2": "per-step working set > 126 MB L2 (no flush needed)",
                   "wau_choice_8gpu": wau8.d},
        "e2e": {"value": round(G / (e2e_ms / 1e3), 2), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "path": ("Trainer.step_async: pinned H2D into one of two staging slots on a copy stream "
                         "(overlapping the previous step), then that slot's CUDA graph of [pack, the step, "
                         "loss D2H into pinned memory]") if tr._captured else
                        ("Trainer.step_async: pinned H2D on a copy stream, then the step's launches "
                         "(rank program with NCCL buckets, no CUDA graph), loss D2H"),
                "d2h_bytes_per_step": 4, "host_ms_per_step": round(host_ms, 3), "loss": loss},
        "gpu_launches": launches * args.steps,
        "roofline": {"bound": "tensor", "kernel": dom.name, "gemm_shape_MNK": list(dom.shape),
                     "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic_of(model, dom.name),
                     "algorithmic_flops": dom.alg_flops,
                     "peak_note": "tcgen05 kind::tf32 issue rate measured in this run (" + tf32_peak["how"] + "); "
                                  "achieved = WAP-counted algorithmic FLOPs (workloads.py:84-117) / kernel time",
                     "tensor_pipe_achieved": round(achieved * pipe_factor, 2),
                     "frac_tensor_pipe": round(achieved * pipe_factor / peak, 4),
                     "fp32_accurate_ceiling": round(peak / pipe_factor, 1),
                     "frac_of_fp32_accurate_ceiling": round(achieved * pipe_factor / peak, 4),
                     "kernel_ms": round(dom_ms, 4), "share_of_step": round(dom_ms / total_kernel_ms, 4)},
        "gemm_summary": {"ms": round(gemm_ms, 3), "share": round(gemm_ms / total_kernel_ms, 4),
                         "algorithmic_tflops": round(gemm_alg_tflops, 2),
                         "frac_algorithmic": round(gemm_alg_tflops / peak, 4),
                         "tensor_pipe_frac": round(gemm_alg_tflops * pipe_factor / peak, 4)},
        "hbm_summary": {"ms": round(ew_ms, 3), "share": round(ew_ms / total_kernel_ms, 4),
                        "achieved_gbs": round(ew_bytes / (ew_ms * 1e-3) / 1e9, 1) if ew_ms else None,
                        "peak_gbs": hbm_peak, "peak_src": peak_src,
                        "frac": round(ew_bytes / (ew_ms * 1e-3) / 1e9 / hbm_peak, 4) if ew_ms else None,
                        "top": [{"kernel": st.name, "ms": round(m, 4),
                                 "gbs": round(st.alg_bytes / (m * 1e-3) / 1e9, 1),
                                 "frac": round(st.alg_bytes / (m * 1e-3) / 1e9 / hbm_peak, 4)}
                                for m, st in ew_top]},
        # WAP's own model next to the measurement: Eq. (1) step time for
        # this d (estimate_total; additive compute + allreduce, no overlap) and estimate_power
        # (host + d * GPU power) against the measured step time and NVML board power
        "wap_model": {
            "d": tplan.plan.d, "predicted_ms": round(est.t_estimate * 1e3, 4),
            "predicted_compute_ms": round(est.t_c_total * 1e3, 4), "measured_ms": round(ms, 4),
            "measured_over_predicted": round(ms / (est.t_estimate * 1e3), 4),
            "predicted_power_w": round(pw_pred, 1),
            "predicted_gpu_power_w": round((pw_pred - prof.host_power) / tplan.plan.d, 1),
            "measured_gpu_power_w": pw["power_w"],
            "measured_idle_power_w": idle["power_w"], "model_util": round(util, 4),
            "fitted_power_peak_w": fit_peak,
            "power_window": {"seconds": round(p1 - p0, 2), "steps": n_pw, "samples": pw["samples"],
                             "sm_mhz": pw["sm_mhz"], "reasons": pw["reasons"]},
            "profile": prof.name,
        },
        "clocks": {k: v for k, v in clocks.items()},
        **({"breakdown_ms": {k: round(v[0], 4) for k, v in sorted(per.items(), key=lambda x: -x[1][0])},
            "gemm_tuned_ms": {k: round(v[1].tuned_ms, 4) for k, v in per.items()
                              if getattr(v[1], "tuned_ms", None) is not None}} if args.breakdown else {}),
    }


def _count_launches(prog) -> int:
    from paper_1811_01532_b200 import _native as N

    before = N.launch_count()
    for st in prog.steps:
        st(N.stream_ptr())
    import torch

    torch.cuda.synchronize()
    return N.launch_count() - before


def _oracle_inputs(g, seed: int = 0) -> dict:
    rs = np.random.default_rng(seed)
    inputs = {}
    for n in g:
        if n.kind.value == "Input":
            shape = tuple(n.attr("shape"))
            if n.id == "labels":
                lab = np.zeros(shape)
                lab[np.arange(shape[0]), rs.integers(0, shape[1], shape[0])] = 1
                inputs[n.id] = lab
            else:
                inputs[n.id] = rs.standard_normal(shape)
    return inputs


def cpu_sample_step(model: str, sample_batch: int, threads: int | None = None) -> dict:
    """One fp64 training step of the oracle port (numpy, the reference algorithm
    interp.py:122-215) at `sample_batch`, on `threads` BLAS threads (all if None)."""
    from threadpoolctl import threadpool_limits

    from oracle import interp_ref as O
    from paper_1811_01532_b200 import models

    g = models.MODELS[model](sample_batch)
    inputs = _oracle_inputs(g)
    cores = len(os.sched_getaffinity(0))
    with threadpool_limits(limits=threads or cores):
        t0 = time.perf_counter()
        O.execute(g, inputs, 42)
        dt = time.perf_counter() - t0
    return {"value": round(sample_batch / dt, 3), "unit": UNIT, "cores": threads or cores, "kind": "port",
            "sample": f"one fp64 training step of {model} at batch {sample_batch} (224x224) through the oracle "
                      f"(numpy/OpenBLAS, {threads or cores} threads), {dt:.2f} s"}


def cpu_config1(threads: int | None = None, G: int = 64, seed: int = 42) -> dict:
    """BASELINE configs[0] / SURVEY §8(d) Config 1 on the host cores: the WAU
    (extract_workloads + select_parallelism over 8 devices with the b200 profile,
    planner.py:217-246), the Graph Modifier (transform, transform.py:588-602) and one
    fp64 training step of the transformed AlexNet-224 graph at G=64 through the
    oracle port (replicas evaluated in turn, as wap.interp.execute does), seed 42."""
    from threadpoolctl import threadpool_limits

    from oracle import interp_ref as O
    from paper_1811_01532_b200 import interp, models, planner
    from paper_1811_01532_b200.graph_modifier import transform
    from paper_1811_01532_b200.ir import infer_shapes
    from paper_1811_01532_b200.workloads import extract_workloads

    cores = len(os.sched_getaffinity(0))
    n = threads or cores
    with threadpool_limits(limits=n):
        t0 = time.perf_counter()
        g = models.alexnet(G)
        wl = extract_workloads(infer_shapes(g))
        plan = planner.select_parallelism(wl, tuple(range(8)), planner.load_profile("b200"))
        tg, _ = transform(g, plan)
        t1 = time.perf_counter()
        inputs = interp.generate_inputs(g, seed)
        t2 = time.perf_counter()
        O.execute(tg, inputs, seed)
        t3 = time.perf_counter()
    total = (t1 - t0) + (t3 - t2)
    return {"value": round(G / total, 3), "unit": UNIT, "cores": n, "kind": "port",
            "sample": f"Config 1: WAU (d*={plan.d} of 8) + transform ({(t1 - t0) * 1e3:.0f} ms) + one fp64 step of "
                      f"the transformed AlexNet-224 graph at G={G}, seed {seed}, through the oracle port "
                      f"(numpy/OpenBLAS, {n} thread{'s' if n > 1 else ''}): {t3 - t2:.2f} s",
            "seconds": round(total, 3)}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    model = "alexnet" if args.model == "both" else args.model
    sample = args.ref_batch or (4 if model == "alexnet" else 1)
    vals = []
    for _ in range(max(args.warmup, 0)):
        cpu_sample_step(model, sample)
    t0 = time.perf_counter()
    steps = max(1, args.steps)
    last = None
    for _ in range(steps):
        last = cpu_sample_step(model, sample)
        vals.append(last["value"])
    total = time.perf_counter() - t0
    v = float(np.median(vals))
    b = args.batch or DEFAULT_BATCH[model]
    return {"metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": round(total * 1e3 / steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{model} fp32 training, batch {b}/GPU, 224x224x3 synthetic ImageNet shape",
                       "network": model, "global_batch": b * world, "parallelism": "CPU (oracle port of wap.interp)",
                       "sample_batch": sample},
            "cpu_baseline": {**last, "value": round(v, 3)},
            "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    import faulthandler

    # a stuck run leaves evidence: every thread's stack on stderr after 10 minutes
    faulthandler.dump_traceback_later(600, exit=False)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--model", default="both", choices=["both", "alexnet", "vgg16"],
                    help="both (default): AlexNet record with a VGG-16 record under 'vgg16'")
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (default: 128 AlexNet, 32 VGG-16)")
    ap.add_argument("--precision", type=int, default=3, choices=[1, 3])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-batch", type=int, default=0,
                    help="images per reference step (default: 4 AlexNet, 1 VGG-16, ~2-4 s of host work each)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--breakdown", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus and "RANK" in os.environ:
        args.gpus = world
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    import torch

    # one rank per GPU; WAP_DIST_BACKEND=gloo (with ranks sharing GPUs) is only for
    # exercising the multi-rank path on a single-GPU box
    backend = os.environ.get("WAP_DIST_BACKEND", "nccl")
    local_rank = local_rank % max(1, torch.cuda.device_count()) if backend != "nccl" else local_rank
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        tf32 = measure_tf32_peak()
    except Exception as e:  # noqa: BLE001 - the fallback is reported as such
        tf32 = {"tflops": TF32_MMA_PEAK_FALLBACK, "how": f"fallback constant (probe failed: {e})"}
    models_run = ["alexnet", "vgg16"] if args.model == "both" else [args.model]
    recs = {}
    for m in models_run:
        recs[m] = run_ours(args, m, rank, world, local_rank, tf32)
        torch.cuda.empty_cache()
    if rank == 0:
        out = recs[models_run[0]]
        for m in models_run[1:]:
            sub = recs[m]
            out[m] = {k: sub[k] for k in ("value", "unit", "ms_per_step", "config", "e2e", "gpu_launches",
                                          "roofline", "gemm_summary", "hbm_summary", "wap_model", "clocks")
                      if k in sub}
        out["tf32_peak"] = tf32
        if world == 1 and not args.no_cpu_baseline:
            # Config 1 (configs[0]) on all host cores and on one BLAS thread (the
            # reference CLI's pinned mode, cli.py:18-21)
            out["cpu_baseline"] = cpu_config1()
            out["cpu_baseline"]["single_thread"] = cpu_config1(threads=1)
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
