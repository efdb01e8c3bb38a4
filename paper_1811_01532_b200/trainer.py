"""Replicated-variables data-parallel training on B200 ranks (paper §2.1, §3.2).

`plan_training` is the WAP pipeline of Fig. 2: Neural-Net Parser
(extract_workloads) -> WAU (select_parallelism, optionally on the GPU) ->
Graph Modifier (transform). `rank_view` cuts the transformed graph into the
program one rank runs: its replicas, its batch shard (the Split part
k = rows [k*G/d, (k+1)*G/d), ir.py:8-12), and a rank-local AllReduceSum per
variable that the runtime turns into an NCCL allreduce over NVLink.
`Trainer` owns one rank's Program and exposes the step a user calls.
"""

from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np

from .errors import TransformError, WorkloadError
from .graph_modifier import transform
from .ir import Graph, Node, OpKind, TensorShape, infer_shapes
from .planner import DeviceProfile, ParallelPlan, plan_for_degree, select_parallelism
from .workloads import extract_workloads


@dataclass(frozen=True)
class TrainingPlan:
    plan: ParallelPlan
    graph: Graph          # transformed (data-parallel) graph
    single: Graph         # the single-device training graph it came from


def plan_training(graph: Graph, n_devices: int, profile: DeviceProfile, algo: str = "ring",
                  force_d: int | None = None, on_device: bool = False) -> TrainingPlan:
    """Parser -> WAU -> Graph Modifier for `n_devices` available GPUs."""
    shaped = infer_shapes(graph)
    wl = extract_workloads(shaped)
    devices = tuple(range(n_devices))
    if force_d is not None:
        plan = plan_for_degree(wl, devices, profile, force_d, algo)
    elif on_device:
        from .planner import select_parallelism_device

        plan = select_parallelism_device(wl, devices, profile, algo)
    else:
        plan = select_parallelism(wl, devices, profile, algo)
    tg, _ = transform(graph, plan)
    return TrainingPlan(plan, tg, graph)


def rank_view(graph: Graph, rank: int, d: int) -> Graph:
    """Single-rank program of a transformed graph (identity when d == 1).

    Keeps the nodes placed on `rank`, replaces each batch Split by a rank-local
    Input holding the shard, and keeps each AllReduceSum with its one local
    operand (the cross-rank sum happens in the collective)."""
    if d == 1:
        return graph
    if not 0 <= rank < d:
        raise TransformError(f"rank {rank} outside [0, {d})")
    g = infer_shapes(graph)
    nodes: dict[str, Node] = {}
    split_src: dict[str, str] = {}
    for n in g:
        if n.kind is OpKind.SPLIT:
            src = g.node(n.inputs[0])
            if src.kind is not OpKind.INPUT or n.attr("axis") != src.output_shape.batch_axis:
                raise TransformError(f"rank views need batch Splits of Inputs, got {n.id!r}")
            split_src[n.id] = src.id
    for n in g:
        if n.kind is OpKind.INPUT:
            shp = n.output_shape
            dims = list(shp.dims)
            if dims[shp.batch_axis] % d:
                raise WorkloadError(f"batch of {n.id!r} not divisible by {d}")
            dims[shp.batch_axis] //= d
            nodes[n.id] = Node(n.id, OpKind.INPUT, (), {**n.attrs, "shape": tuple(dims)}, rank)
        elif n.kind is OpKind.ALL_REDUCE_SUM:
            local = [i for i in n.inputs if g.node(i).device == rank]
            if len(local) != 1:
                raise TransformError(f"{n.id!r} has {len(local)} operands on rank {rank}")
            nodes[n.id] = Node(n.id, OpKind.ALL_REDUCE_SUM, tuple(local), dict(n.attrs), rank)
        elif n.kind is OpKind.SPLIT:
            continue
        elif n.device == rank:
            ins = tuple(split_src.get(i, i) for i in n.inputs)
            nodes[n.id] = Node(n.id, n.kind, ins, dict(n.attrs), rank)
    # allreduce nodes only survive if a local node consumes them
    used = {i for n in nodes.values() for i in n.inputs}
    nodes = {k: v for k, v in nodes.items() if v.kind is not OpKind.ALL_REDUCE_SUM or k in used}
    outputs = tuple(o for o in g.outputs if o in nodes)
    return Graph(f"{g.name}@rank{rank}", nodes, outputs)


class Trainer:
    """One rank of replicated-variables SGD on the current CUDA device.

    `step(images, labels)` takes this rank's shard (host or device arrays; host
    arrays are copied H2D inside the call) and returns the rank's loss (a
    device scalar unless fetch=True). With world_size > 1 the gradients are summed
    across ranks per bucket, overlapping the rest of backward, by
      allreduce="nccl": torch.distributed all_reduce (NCCL over NVLink) on a comm
                        stream, each bucket's SGD behind it;
      allreduce="p2p":  one fused wap_allreduce_sgd kernel per bucket over
                        peer-mapped memory (left fold in rank order = the
                        reference's AllReduceSum, then SGD, then all-gather);
      allreduce="nvls": the same kernel with multimem.ld_reduce / multimem.st
                        through the NVSwitch.
    (default: $WAP_ALLREDUCE, else "nccl"). The loss seed already divides by the
    global batch, so no 1/N scaling is needed (training.py:94-102). The whole
    step is one CUDA graph whenever its collectives are capturable (d == 1,
    NCCL, or the fused kernel; not gloo)."""

    def __init__(self, tplan: TrainingPlan, rank: int = 0, precision: int = 3, seed: int = 0,
                 variables: dict | None = None, process_group=None, use_graph: bool = True,
                 bucket_bytes: int = 64 << 20, allreduce: str | None = None):
        import torch

        from .interp import initial_variables
        from .runtime import Program

        self.torch = torch
        self.tplan = tplan
        self.d = tplan.plan.d
        self.rank = rank
        self.view = rank_view(tplan.graph, rank, self.d)
        self.pg = process_group
        self.allreduce = allreduce or os.environ.get("WAP_ALLREDUCE", "nccl")
        if self.allreduce not in ("nccl", "p2p", "nvls"):
            raise TransformError(f"unknown allreduce {self.allreduce!r} (nccl, p2p, nvls)")
        collective, fused, capturable = None, None, True
        if self.d > 1 and self.allreduce == "nccl":
            import torch.distributed as dist

            collective = self._allreduce
            capturable = dist.get_backend(self.pg) == "nccl"
        elif self.d > 1:
            from .peer_memory import FusedAllReduce

            fused = FusedAllReduce(rank, self.d, torch.cuda.current_device(), self.allreduce, self.pg)
        self.prog = Program(self.view, precision=precision, in_place=True, collective=collective,
                            bucket_bytes=bucket_bytes, fused=fused, collective_capturable=capturable)
        init = initial_variables(self.view, seed)
        if variables:
            for k in init:
                base = k.split("/dev")[0]
                if k in variables:
                    init[k] = variables[k]
                elif base in variables:
                    init[k] = variables[base]
        self.prog.bind(init)
        self.inputs = [n.id for n in self.view if n.kind is OpKind.INPUT]
        self.loss_id = next(o for o in self.view.outputs if self.view.node(o).kind is OpKind.SOFTMAX_XENT_LOSS)
        self.use_graph = use_graph and capturable
        self._captured = False

    def _allreduce(self, buf) -> None:
        import torch.distributed as dist

        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.pg)

    def load(self, batch: dict) -> None:
        """Stage this rank's shard into the input buffers (H2D if host memory)."""
        self.prog.bind_async(batch)

    def run(self) -> None:
        if self.use_graph and not self._captured:
            self.prog.capture()
            self._captured = True
        self.prog.run()

    def step(self, batch: dict | None = None, fetch: bool = False):
        if batch is not None:
            self.load(batch)
        self.run()
        loss = self.prog.t[self.loss_id].buf[:1]
        return float(loss.item()) if fetch else loss

    def step_async(self, batch: dict) -> None:
        """One step from pinned host buffers without host synchronisation: the H2D
        copy of `batch` runs on a copy stream (overlapping the previous step), the
        step runs on the compute stream, and the loss is copied to a pinned host
        scalar (D2H) behind it. `last_loss()` waits for and returns that value."""
        torch = self.torch
        if not hasattr(self, "copy_stream"):
            self.copy_stream = torch.cuda.Stream()
            self._loss_host = torch.empty(1, dtype=torch.float32, pin_memory=True)
            self._loss_ev = torch.cuda.Event()
            self._e2e_graphs = [None, None]
            self._slot_free = [None, None]
            self._slot = 0
        if not self.use_graph:
            self.prog.bind_overlapped(batch, self.copy_stream)
            self.run()
            self._loss_host.copy_(self.prog.t[self.loss_id].buf[:1], non_blocking=True)
            self._loss_ev.record()
            return
        # graph path: two staging slots, each with its own CUDA graph of
        # [pack staging -> inputs, the whole step, loss D2H into pinned memory]. The H2D
        # of step i+1 fills the other slot while step i runs; it only waits for the
        # step that last read that slot (i-1), so the copy overlaps compute.
        if not self._captured:
            self.prog.capture()  # warm-up (variables restored) + the plain step graph
            self._captured = True
        if self._e2e_graphs[0] is None:
            # both slots' staging and graphs up front: no capture inside a timed loop
            loss = self.prog.t[self.loss_id].buf[:1]
            post = [] if os.environ.get("WAP_E2E_D2H_OUTSIDE") else \
                [lambda sp: self._loss_host.copy_(loss, non_blocking=True)]
            for k in (0, 1):
                staged = self.prog.staging(batch, k)
                self._e2e_graphs[k] = self.prog.capture_with(
                    pre=[lambda sp, st=staged: self.prog.pack_staged(st, sp)], post=post)
        j = self._slot
        self.prog.h2d_staged(batch, self.copy_stream, j, after=self._slot_free[j])
        self._e2e_graphs[j].replay()
        if os.environ.get("WAP_E2E_D2H_OUTSIDE"):
            self._loss_host.copy_(self.prog.t[self.loss_id].buf[:1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._slot_free[j] = ev
        self._loss_ev.record()
        self._slot = 1 - j

    def last_loss(self) -> float:
        self._loss_ev.synchronize()
        return float(self._loss_host[0])

    def variables(self) -> dict[str, np.ndarray]:
        return {n.id: self.prog.fetch(n.id) for n in self.view if n.kind is OpKind.VARIABLE}
