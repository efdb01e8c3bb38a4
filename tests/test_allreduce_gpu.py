"""Fused gradient allreduce + SGD (csrc/allreduce.cu, wap_allreduce_sgd) over
peer-mapped / multicast memory (peer_memory.py), on the one B200 available:

* world 1, both modes: the P2P path and the NVLS path (a one-device multicast
  object: multimem.ld_reduce / multimem.st through the switch) apply
  w -= lr * g exactly, per bucket, and replay inside a CUDA graph (device-side
  epochs advance the barriers on every replay);
* world 2 as two processes sharing the GPU (gloo only for the handle exchange):
  each rank maps the other's arenas (POSIX fd + pidfd_getfd), the kernel's
  barriers synchronise the two processes, the result is the reference left fold
  g0 + g1 (interp.py:115-119) then SGD (interp.py:203-204), bitwise equal on both
  ranks; and the full Trainer in allreduce="p2p" mode (one CUDA graph per step,
  fused kernel per bucket) matches a single-process execution of the WAP-transformed
  graph.
Multi-GPU NVLink bandwidth is not measurable on a one-GPU box."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _expected(var0, grad, lr, reps=1):
    w = var0.clone()
    for _ in range(reps):
        w = torch.addcmul(w, grad, torch.full_like(grad, -lr))
    return w


@pytest.mark.parametrize("mode", ["p2p", "nvls"])
def test_world1_fused_kernel_and_graph_replay(cuda, mode):
    from paper_1811_01532_b200 import _native as N
    from paper_1811_01532_b200.peer_memory import FusedAllReduce

    if mode == "nvls":
        from paper_1811_01532_b200.peer_memory import multicast_supported

        ok, why = multicast_supported(0)
        if not ok:
            pytest.skip(f"no NVLS multicast on this box ({why})")
    n = (1 << 20) + 6  # odd tail
    fr = FusedAllReduce(0, 1, 0, mode)
    var, grad = fr.allocate(n + 2)
    g = torch.Generator(device="cuda").manual_seed(0)
    var.copy_(torch.randn(n + 2, device=cuda, generator=g))
    grad.copy_(torch.randn(n + 2, device=cuda, generator=g))
    v0 = var.clone()
    lr = 0.01
    # two buckets: [0, 4096) and [4096, n)
    fr.launch(0, 4096, lr, 0, N.stream_ptr())
    fr.launch(4096, n - 4096, lr, 1, N.stream_ptr())
    torch.cuda.synchronize()
    assert fr.status() == 0
    exp = v0.clone()
    exp[:n] = v0[:n] - lr * grad[:n]
    assert (var - exp).abs().max().item() <= 1e-6 * exp.abs().max().item()
    assert torch.equal(var[n:], v0[n:])  # outside every bucket: untouched
    # CUDA graph: three replays = three SGD steps, epochs advance on the device
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        fr.launch(0, n, lr, 2, N.stream_ptr(s))
    torch.cuda.current_stream().wait_stream(s)
    start = var.clone()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert fr.status() == 0
    exp = start.clone()
    for _ in range(3):
        exp[:n] = exp[:n] - lr * grad[:n]
    assert (var - exp).abs().max().item() <= 1e-6 * exp.abs().max().item()
    assert int(fr.counters[2].item()) == 3  # epoch of slot 2 after three replays


def _kernel_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1811_01532_b200 import _native as N
    from paper_1811_01532_b200.peer_memory import FusedAllReduce

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 300_003
        fr = FusedAllReduce(rank, world, 0, "p2p")
        var, grad = fr.allocate(n + 1)
        g = torch.Generator(device="cuda").manual_seed(100 + rank)
        grad.copy_(torch.randn(n + 1, device="cuda", generator=g))
        var.copy_(torch.arange(n + 1, device="cuda", dtype=torch.float32) * 1e-6)
        torch.cuda.synchronize()
        dist.barrier()
        fr.launch(0, 65536, 0.5, 0, N.stream_ptr())
        fr.launch(65536, n - 65536, 0.5, 1, N.stream_ptr())
        torch.cuda.synchronize()
        q.put((rank, fr.status(), var.cpu().numpy().copy(), grad.cpu().numpy().copy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_processes_fused_kernel_left_fold(cuda):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_kernel_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, status, var, grad = q.get(timeout=300)
        res[r] = (status, var, grad)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 300_003
    g = res[0][2][:n] + res[1][2][:n]  # fp32 left fold, rank order
    v0 = (np.arange(n + 1, dtype=np.float32) * np.float32(1e-6))[:n]
    exp = (v0.astype(np.float64) - 0.5 * g.astype(np.float64)).astype(np.float32)
    for r in range(world):
        assert res[r][0] == 0, "barrier timed out"
        assert np.abs(res[r][1][:n] - exp).max() <= 1e-6 * np.abs(exp).max()
    assert np.array_equal(res[0][1], res[1][1])  # replicas bitwise equal


def _bindings(graph, seed=3):
    rs = np.random.default_rng(seed)
    out = {}
    for n in graph:
        shape = tuple(n.attr("shape") or ())
        if n.kind.value == "Variable":
            fan = int(np.prod(shape[:-1])) if len(shape) > 1 else 1
            out[n.id] = (np.sqrt(2.0 / fan) if len(shape) > 1 else 0.01) * rs.standard_normal(shape)
        elif n.id == "labels":
            lab = np.zeros(shape)
            lab[np.arange(shape[0]), rs.integers(0, shape[1], shape[0])] = 1
            out[n.id] = lab
        elif n.kind.value == "Input":
            out[n.id] = rs.standard_normal(shape)
    return out


def _trainer_worker(rank, world, port, net, kw, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1811_01532_b200 import models, planner, trainer

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = models.MODELS[net](**kw)
        bind = _bindings(g)
        tp = trainer.plan_training(g, world, planner.load_profile("b200"), force_d=world)
        tr = trainer.Trainer(tp, rank=rank, variables={k: v for k, v in bind.items() if k not in ("images", "labels")},
                             bucket_bytes=1 << 20, allreduce="p2p")
        b = kw["batch"] // world
        shard = {k: torch.from_numpy(np.ascontiguousarray(bind[k][rank * b:(rank + 1) * b]).astype(np.float32))
                 for k in ("images", "labels")}
        loss = tr.step(shard, fetch=True)
        torch.cuda.synchronize()
        q.put((rank, loss, tr.variables(), len(tr.prog.buckets), tr._captured, tr.prog.fused.status()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("net,kw", [("alexnet_like", {"batch": 16}), ("alexnet", {"batch": 4, "image": 99})])
def test_two_ranks_trainer_fused_p2p_matches_single_process(cuda, net, kw):
    from oracle import interp_ref as O
    from paper_1811_01532_b200 import graph_modifier as gm
    from paper_1811_01532_b200 import interp, models, planner

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_trainer_worker, args=(r, world, port, net, kw, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, loss, var, nb, captured, status = q.get(timeout=600)
        res[r] = (loss, var, nb, captured, status)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = models.MODELS[net](**kw)
    bind = _bindings(g)
    tg = gm.transform(g, planner.ParallelPlan(world, tuple(range(world)), (), 0.0))[0]
    full = dict(bind)
    for n in tg:
        if n.kind.value == "Variable" and n.id not in full:
            full[n.id] = bind[n.id.split("/dev")[0]]
    ref = interp.execute(tg, full, 0)
    for rank, (loss, var, nb, captured, status) in res.items():
        assert status == 0
        assert captured, "the fused step should be one CUDA graph"
        assert nb >= 1
        assert abs(loss - ref[f"loss/dev{rank}"][0]) <= 1e-5 * max(1.0, abs(loss))
        for vid, val in var.items():
            upd = vid.replace(f"/dev{rank}", f"_upd/dev{rank}")
            assert O.relative_deviation(val, ref[upd]) < 1e-6, vid
    for vid in res[0][1]:
        assert np.array_equal(res[0][1][vid], res[1][1][vid.replace("/dev0", "/dev1")]), vid
