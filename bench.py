"""Benchmark: WAP data-parallel training step (AlexNet / VGG-16) on B200.

Contract (see task / DESIGN.md "Measurement"):
  python bench.py --gpus N --steps K --warmup W          (N > 1 under torchrun)
  python bench.py --impl reference ...                   CPU oracle port on host cores
prints ONE JSON line on rank 0.

value    images/sec of the whole job: global batch G = b*N per step, K steps
         timed with CUDA events between barriers, max over ranks; inputs
         resident in HBM (one synthetic batch staged before timing; the
         per-step working set, >= 0.5 GB of activations, exceeds the 126 MB L2).
e2e      the same metric through the public API Trainer.step(batch) with
         pinned host buffers: H2D of the shard + step + D2H of the loss, timed.
roofline dominant kernel (a tcgen05 GEMM) from an instrumented pass with CUDA
         events around every launch of the same step.
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


# tcgen05.mma kind::tf32 issue rate measured on this pool's B200 by tools/mma_probe.cu
# (profiles/r01/mma_probe.txt: 2048 MAC/clk/SM for N >= 128 = 1116 TFLOP/s; nominal 1.1 PF).
# MEASURED_PEAKS.json carries only HBM and bf16 figures, so the TF32 GEMM roofline uses this.
TF32_MMA_PEAK_TFLOPS = 1116.4


def peaks():
    """(HBM GB/s, bf16 TFLOP/s, source) from the driver-written MEASURED_PEAKS.json, else the
    fallback of /opt/skills/guides/B200_PROFILING.md."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), float(d.get("bf16_tflops", 1590.0)), "measured"
    return 6650.0, 1590.0, "fallback"


def traffic_of(model: str, step: str):
    """DRAM bytes per launch of `step` from the committed ncu --set full captures
    (profiles/traffic.json, written by tools/capture_traffic.sh), or None."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    e = json.loads(p.read_text()).get(model, {}).get(step)
    return None if e is None else int(e["traffic_bytes"])


class ClockSampler:
    """nvidia-smi sampling of SM clocks / throttle reasons around the timed region.

    Sampling starts before the warm-up (nvidia-smi can take seconds to attach on a
    fresh box) and samples are kept by their own timestamps when they fall inside
    the timed region (else every sample of the run is reported). Stopping never
    blocks: a sampler that does not exit after SIGTERM/SIGKILL is abandoned."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self.window = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def mark(self, t0: float, t1: float) -> None:
        self.window = (t0, t1)

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

    @staticmethod
    def _stamp(ts: str):
        import datetime

        try:
            return datetime.datetime.strptime(ts.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return None

    def summary(self) -> dict:
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
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
        sel = rows
        if self.window is not None:
            t0, t1 = self.window
            inside = [r for r in rows if r[0] is not None and t0 - 0.05 <= r[0] <= t1 + 0.05]
            if inside:
                sel = inside
        reasons = {n for r in sel for n, v in zip(names, r[3]) if v.lower() == "active"}
        sm = [r[1] for r in sel]
        pw = [r[4] for r in sel if r[4] == r[4]]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": sel[-1][2] if sel else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "window": "timed region" if sel is not rows else "whole run",
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


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1811_01532_b200 import _native as N
    from paper_1811_01532_b200 import models, planner, trainer, wau_device
    from paper_1811_01532_b200.ir import infer_shapes
    from paper_1811_01532_b200.runtime import _GemmStep
    from paper_1811_01532_b200.workloads import extract_workloads

    dev = torch.device("cuda", local_rank)
    b = args.batch or DEFAULT_BATCH[args.model]
    G = b * world
    graph = models.MODELS[args.model](G)
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

    clk = ClockSampler(local_rank).start()
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
    clk.mark(w0, time.time())
    clk.stop()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
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
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    host_ms = (time.perf_counter() - h0) * 1e3 / e2e_steps
    t = torch.tensor([e2e_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    h2d = sum(v.numel() * 4 for v in batch.values())

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
    tf32_peak = TF32_MMA_PEAK_TFLOPS
    pipe_factor = 3 if args.precision == 3 else 1
    # HBM-bound kernels (im2col, pool, LRN, bias-grad, xent, SGD): algorithmic bytes / event time
    ew = [(v[0], v[1]) for v in per.values() if getattr(v[1], "alg_bytes", 0) > 0]
    ew_ms = sum(m for m, _ in ew)
    ew_bytes = sum(st.alg_bytes for _, st in ew)
    ew_top = sorted(ew, key=lambda x: -x[0])[:6]
    achieved = dom.alg_flops * pipe_factor / (dom_ms * 1e-3) / 1e12
    launches = prog.launches_per_step() if not tr._captured else _count_launches(prog)

    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic (N(0,1) NHWC images, one-hot labels, He-scaled random-init weights)",
            "impl": "ours",
            "config": {"workload": f"{args.model} fp32 training, batch {b}/GPU, 224x224x3 synthetic ImageNet shape",
                       "network": args.model, "global_batch": G, "batch_per_gpu": b, "image": 224,
                       "parallelism": f"dp{world} replicated-variables (WAP transform, forced d={world})",
                       "gemm_precision": "3xTF32 (fp32-accurate)" if args.precision == 3 else "TF32",
                       "cuda_graph": tr._captured, "l2": "per-step working set > 126 MB L2 (no flush needed)",
                       "wau_choice_8gpu": wau8.d},
            "e2e": {"value": round(G / (e2e_ms / 1e3), 2), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "path": "Trainer.step_async: pinned H2D into one of two staging slots on a copy stream "
                            "(overlapping the previous step), then that slot's CUDA graph of [pack, the step, "
                            "loss D2H into pinned memory]",
                    "d2h_bytes_per_step": 4, "host_ms_per_step": round(host_ms, 3), "loss": loss},
            "gpu_launches": launches * args.steps,
            "roofline": {"bound": "tensor", "kernel": dom.name, "gemm_shape_MNK": list(dom.shape),
                         "achieved": round(achieved, 2), "peak": tf32_peak, "unit": "TFLOP/s",
                         "frac": round(achieved / tf32_peak, 4), "traffic": traffic_of(args.model, dom.name),
                         "algorithmic_flops": dom.alg_flops,
                         "peak_note": "measured tcgen05 kind::tf32 issue rate (tools/mma_probe.cu, "
                                      "profiles/r01/mma_probe.txt); achieved counts tensor-pipe FLOPs "
                                      f"({pipe_factor}x algorithmic for {'3xTF32' if pipe_factor == 3 else 'TF32'}); "
                                      "traffic = ncu dram bytes per launch (profiles/traffic.json)",
                         "kernel_ms": round(dom_ms, 4), "share_of_step": round(dom_ms / total_kernel_ms, 4)},
            "gemm_summary": {"ms": round(gemm_ms, 3), "share": round(gemm_ms / total_kernel_ms, 4),
                             "algorithmic_tflops": round(gemm_flops / (gemm_ms * 1e-3) / 1e12, 2),
                             "tensor_pipe_frac": round(gemm_flops * pipe_factor / (gemm_ms * 1e-3) / 1e12
                                                       / tf32_peak, 4)},
            "hbm_summary": {"ms": round(ew_ms, 3), "share": round(ew_ms / total_kernel_ms, 4),
                            "achieved_gbs": round(ew_bytes / (ew_ms * 1e-3) / 1e9, 1) if ew_ms else None,
                            "peak_gbs": hbm_peak, "peak_src": peak_src,
                            "frac": round(ew_bytes / (ew_ms * 1e-3) / 1e9 / hbm_peak, 4) if ew_ms else None,
                            "top": [{"kernel": st.name, "ms": round(m, 4),
                                     "gbs": round(st.alg_bytes / (m * 1e-3) / 1e9, 1),
                                     "frac": round(st.alg_bytes / (m * 1e-3) / 1e9 / hbm_peak, 4)}
                                    for m, st in ew_top]},
        }
        if args.breakdown:
            out["breakdown_ms"] = {k: round(v[0], 4) for k, v in sorted(per.items(), key=lambda x: -x[1][0])}
            # isolated autotune time of each GEMM (same launch, warm L2, no neighbours)
            out["gemm_tuned_ms"] = {k: round(v[1].tuned_ms, 4) for k, v in per.items()
                                    if getattr(v[1], "tuned_ms", None) is not None}
    clocks = clk.summary()
    # WAP's own model next to the measurement: Eq. (1) step time for
    # this d (estimate_total; additive compute + allreduce, no overlap) and estimate_power
    # (host + d * GPU power) against the measured step time and NVML board power
    if out is None:  # ranks > 0 print nothing
        return out, clocks
    est = tplan.plan.chosen
    pw = planner.estimate_power(tplan.plan, wl, prof)
    out["wap_model"] = {
        "d": tplan.plan.d, "predicted_ms": round(est.t_estimate * 1e3, 4),
        "predicted_compute_ms": round(est.t_c_total * 1e3, 4), "measured_ms": round(ms, 4),
        "measured_over_predicted": round(ms / (est.t_estimate * 1e3), 4),
        "predicted_power_w": round(pw, 1),
        "predicted_gpu_power_w": round((pw - prof.host_power) / tplan.plan.d, 1),
        "measured_gpu_power_w": clocks.get("power_w"),
        "profile": prof.name,
    }
    return out, clocks


def _count_launches(prog) -> int:
    from paper_1811_01532_b200 import _native as N

    before = N.launch_count()
    for st in prog.steps:
        st(N.stream_ptr())
    import torch

    torch.cuda.synchronize()
    return N.launch_count() - before


def cpu_baseline(model: str, sample_batch: int, threads: int | None = None) -> dict:
    """Oracle port (numpy fp64, the reference algorithm) timed on the host cores."""
    from oracle import interp_ref as O
    from paper_1811_01532_b200 import models

    g = models.MODELS[model](sample_batch)
    rs = np.random.default_rng(0)
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
    t0 = time.perf_counter()
    O.execute(g, inputs, 42)
    dt = time.perf_counter() - t0
    cores = len(os.sched_getaffinity(0))
    return {"value": round(sample_batch / dt, 3), "unit": UNIT, "cores": threads or cores, "kind": "port",
            "sample": f"one fp64 training step of {model} at batch {sample_batch} (224x224) through the oracle "
                      f"(numpy/OpenBLAS, {threads or cores} threads), {dt:.2f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    sample = args.ref_batch
    vals = []
    for _ in range(max(args.warmup, 0)):
        cpu_baseline(args.model, sample)
    t0 = time.perf_counter()
    steps = max(1, args.steps)
    last = None
    for _ in range(steps):
        last = cpu_baseline(args.model, sample)
        vals.append(last["value"])
    total = time.perf_counter() - t0
    v = float(np.median(vals))
    b = args.batch or DEFAULT_BATCH[args.model]
    return {"metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": round(total * 1e3 / steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.model} fp32 training, batch {b}/GPU, 224x224x3 synthetic ImageNet shape",
                       "network": args.model, "global_batch": b * world, "parallelism": "CPU (oracle port of wap.interp)",
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
    ap.add_argument("--model", default="alexnet", choices=["alexnet", "vgg16"])
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
    args.ref_batch = args.ref_batch or (4 if args.model == "alexnet" else 1)

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
    out, clocks = run_ours(args, rank, world, local_rank)
    if rank == 0:
        out["clocks"] = clocks
        if world == 1 and not args.no_cpu_baseline:
            # a bounded sample (~10-20 s of host work): one fp64 step at a reduced batch
            out["cpu_baseline"] = cpu_baseline(args.model, 16 if args.model == "alexnet" else 4)
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
