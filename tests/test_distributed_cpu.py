"""Multi-rank host logic on CPU (gloo, world_size 2 and 4).

Each rank takes its `rank_view` of the WAP-transformed graph (its replicas and
its batch shard); the rank-local AllReduceSum becomes a real gloo allreduce.
The per-rank outputs must equal the single-process evaluation of the full
transformed graph (which equals the reference's). The CPU oracle stands in for
the GPU kernels here -- test infrastructure only."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import interp_ref as O
from paper_1811_01532_b200 import graph_modifier as gm
from paper_1811_01532_b200 import ir, models, planner, trainer


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, model, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = models.MODELS[model](batch)
        tg = gm.transform(g, planner.ParallelPlan(world, tuple(range(world)), (), 0.0))[0]
        view = trainer.rank_view(tg, rank, world)
        full_inputs = O.generate_inputs(g, 42)
        b = batch // world
        shard = {k: v[rank * b:(rank + 1) * b] for k, v in full_inputs.items()}

        def allreduce(node, ins):
            t = torch.from_numpy(np.ascontiguousarray(ins[0]))
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            return t.numpy()

        out = O.execute(view, shard, 42, hooks={"AllReduceSum": allreduce})
        q.put((rank, {k: v for k, v in out.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("model,batch,world", [("alexnet_like", 16, 2), ("mlp", 24, 4), ("vgg16_like", 8, 2),
                                               ("alexnet_like", 12, 3), ("mlp", 30, 5)])
def test_rank_views_with_gloo_allreduce(model, batch, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, model, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = models.MODELS[model](batch)
    tg = gm.transform(g, planner.ParallelPlan(world, tuple(range(world)), (), 0.0))[0]
    single = O.execute(tg, O.generate_inputs(g, 42), 42)
    for rank, outs in results.items():
        assert outs, rank
        for k, v in outs.items():
            assert k.endswith(f"/dev{rank}")
            # summation order differs from the in-process left fold only by rounding
            assert O.relative_deviation(v, single[k]) < 1e-12, k


def test_rank_view_structure():
    g = models.alexnet_like(16)
    tg = gm.transform(g, planner.ParallelPlan(4, (0, 1, 2, 3), (), 0.0))[0]
    v = trainer.rank_view(tg, 2, 4)
    shaped = ir.infer_shapes(v)
    assert shaped.node("images").output_shape.dims == (4, 6, 6, 3)
    assert all(n.kind is not ir.OpKind.SPLIT for n in v)
    ars = [n for n in v if n.kind is ir.OpKind.ALL_REDUCE_SUM]
    assert len(ars) == 16 and all(len(n.inputs) == 1 for n in ars)
    assert all(n.device == 2 for n in v)
    assert set(v.outputs) == {o for o in tg.outputs if o.endswith("/dev2")}
    assert trainer.rank_view(g, 0, 1) is g


def test_plan_training_pipeline():
    g = models.alexnet_like(128)
    tp = trainer.plan_training(g, 4, planner.load_profile("pcie-box"))
    assert tp.plan.d == 1  # Table-2 analog: small batch stays on one device
    tp8 = trainer.plan_training(g, 4, planner.load_profile("pcie-box"), force_d=4)
    assert tp8.plan.d == 4 and any(n.kind is ir.OpKind.ALL_REDUCE_SUM for n in tp8.graph)


def _ar_worker(rank, world, port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    import allreduce_sweep

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, allreduce_sweep.sweep(10_007, 4096, 2, torch.device("cpu"), "gloo")))
    finally:
        dist.destroy_process_group()


def test_allreduce_sweep_harness_gloo():
    """configs[4] harness (tools/allreduce_sweep.py): single-shot and bucketed SUM
    allreduce produce the exact sum on every rank; ragged last bucket included."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ar_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, rows in res:
        assert [r["mode"] for r in rows] == ["single", "bucketed"]
        assert rows[1]["buckets"] == -(-10_007 // 1024)
        assert all(r["sum_ok"] for r in rows)
