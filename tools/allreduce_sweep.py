"""Gradient allreduce sweep (BASELINE configs[4]): fp32 SUM allreduce of AlexNet
(61,100,840) and VGG-16 (138,357,544) parameter-sized buffers, single-shot vs the
runtime's 64 MB buckets, timed with CUDA events between barriers, max over ranks.
Bus bandwidth = 2(d-1)/d * bytes / time, against 900 GB/s NVLink 5.

    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/allreduce_sweep.py
prints one JSON line per (size, mode) on rank 0. `--backend gloo --device cpu` runs
the same harness on host tensors (tests/test_distributed_cpu.py checks the sums).
"""
import argparse
import json
import os
import time

import torch
import torch.distributed as dist

SIZES = {"alexnet": 61_100_840, "vgg16": 138_357_544}


def sweep(elems: int, bucket_bytes: int, reps: int, device, backend: str) -> list[dict]:
    rank, world = dist.get_rank(), dist.get_world_size()
    buf = torch.full((elems,), float(rank + 1), dtype=torch.float32, device=device)
    expect = world * (world + 1) / 2
    out = []
    step = max(1, bucket_bytes // 4)
    for mode in ("single", "bucketed"):
        chunks = [buf] if mode == "single" else [buf[i:i + step] for i in range(0, elems, step)]

        def once():
            for c in chunks:
                dist.all_reduce(c, op=dist.ReduceOp.SUM)

        buf.fill_(float(rank + 1))
        once()  # warm-up, also the correctness check
        ok = bool((buf == expect).all().item())
        if device.type == "cuda":
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                once()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
        else:
            dist.barrier()
            t0 = time.perf_counter()
            for _ in range(reps):
                once()
            ms = (time.perf_counter() - t0) * 1e3 / reps
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        nbytes = elems * 4
        busbw = 2 * (world - 1) / world * nbytes / (ms * 1e-3) / 1e9 if world > 1 else 0.0
        out.append({"elems": elems, "bytes": nbytes, "mode": mode, "buckets": len(chunks), "d": world,
                    "ms": round(ms, 4), "busbw_gbs": round(busbw, 1), "frac_of_900": round(busbw / 900, 4),
                    "sum_ok": ok})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="nccl")
    ap.add_argument("--device", default="cuda")
    ap.add_argument("--elems", type=int, default=0, help="one custom size instead of AlexNet/VGG-16")
    ap.add_argument("--bucket-bytes", type=int, default=64 << 20)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.device == "cuda":
        torch.cuda.set_device(local)
        device = torch.device("cuda", local)
        dist.init_process_group(args.backend, device_id=device)
    else:
        device = torch.device("cpu")
        dist.init_process_group(args.backend)
    sizes = {"custom": args.elems} if args.elems else SIZES
    for name, n in sizes.items():
        for r in sweep(n, args.bucket_bytes, args.reps, device, args.backend):
            if dist.get_rank() == 0:
                print(json.dumps({"params": name, **r}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
