"""Graph Modifier: single-device training graph -> data-parallel graph (paper §3.2.2-3.2.3).

The three rewrites are the reference's (transform.py:1-24, 172-641) and emit
identical graphs (same ids, wiring, devices; serialized bytes are compared in
tests/test_host_parity.py):
  step 1  replicate_primary        MatMul/Conv2D + gradient companions + variables
                                   get d replicas `<id>/dev<k>`; batch inputs arrive
                                   through a Split of the full tensor, outputs leave
                                   through a Concat; each update is fed by a
                                   per-device AddN over every producer (naive all-to-all).
  step 2  localize_auxiliary       clone auxiliary nodes per device, cancel
                                   Concat->Split pairs: fwd/bwd become device-local.
  step 3  optimize_gradient_aggregation
                                   each variable's d AddNs -> one AllReduceSum.
After step 3 the only cross-device edges are the AllReduceSums, which is what
the GPU runtime turns into the (bucketed) NCCL allreduce; the surviving Splits
are exactly the batch sharding: rank k reads rows [k*G/d, (k+1)*G/d).

Extension: MaxPool/GradMaxPool/LRN/GradLRN are batch-shard-preserving auxiliary
kinds (cloned in step 2 like ReLU).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

from .errors import TransformError
from .ir import (
    GRAD_COMPANION_KINDS,
    PRIMARY_KINDS,
    Graph,
    Node,
    OpKind,
    base_id,
    infer_shapes,
    replica_index,
    topo_order,
    validate,
)
from .planner import ParallelPlan

INFRA_KINDS = frozenset({OpKind.SPLIT, OpKind.CONCAT, OpKind.ALL_REDUCE_SUM})
SHARD_AUX_KINDS = frozenset({
    OpKind.RELU, OpKind.BIAS_ADD, OpKind.GRAD_RELU, OpKind.GRAD_SOFTMAX_XENT,
    OpKind.MAX_POOL, OpKind.GRAD_MAX_POOL, OpKind.LRN, OpKind.GRAD_LRN,
})
PARTIAL_AUX_KINDS = frozenset({OpKind.GRAD_BIAS})
LOSS_AUX_KINDS = frozenset({OpKind.SOFTMAX_XENT_LOSS})
# input slots that carry a batch shard (the others hold the per-device weight replica)
SHARD_SLOTS = {
    OpKind.MATMUL: (0,), OpKind.CONV2D: (0,), OpKind.GRAD_MATMUL_W: (0, 1),
    OpKind.GRAD_MATMUL_X: (0,), OpKind.GRAD_CONV2D_W: (0, 1), OpKind.GRAD_CONV2D_X: (0,),
}
BATCH_OUTPUT_KINDS = PRIMARY_KINDS | {OpKind.GRAD_MATMUL_X, OpKind.GRAD_CONV2D_X}


@dataclass(frozen=True)
class TransformReport:
    step: str
    nodes_replicated: int = 0
    splits_inserted: int = 0
    concats_inserted: int = 0
    split_concat_pairs_removed: int = 0
    cross_device_edges_before: int = 0
    cross_device_edges_after: int = 0
    allreduce_nodes_inserted: int = 0

    def to_json(self) -> dict:
        return {k: getattr(self, k) for k in (
            "step", "nodes_replicated", "splits_inserted", "concats_inserted",
            "split_concat_pairs_removed", "cross_device_edges_before", "cross_device_edges_after",
            "allreduce_nodes_inserted")}


def _device_of(nodes: dict[str, Node], nid: str) -> int | None:
    while nodes[nid].kind is OpKind.SPLIT:  # a Split lives where its input lives
        nid = nodes[nid].inputs[0]
    return nodes[nid].device


def cross_device_edges(graph: Graph) -> int:
    """Edges whose endpoints sit on different devices, plus every AllReduceSum edge."""
    n_cross = 0
    for n in graph:
        for i in n.inputs:
            if n.kind is OpKind.ALL_REDUCE_SUM or graph.node(i).kind is OpKind.ALL_REDUCE_SUM:
                n_cross += 1
                continue
            a, b = _device_of(graph.nodes, i), _device_of(graph.nodes, n.id)
            if a is not None and b is not None and a != b:
                n_cross += 1
    return n_cross


def _sweep(nodes: dict[str, Node], outputs) -> tuple[dict[str, Node], int, int]:
    """Keep what the outputs (and every Input) reach; count dropped Splits/Concats."""
    live: set[str] = set()
    todo = list(outputs) + [nid for nid, n in nodes.items() if n.kind is OpKind.INPUT]
    while todo:
        nid = todo.pop()
        if nid not in live:
            live.add(nid)
            todo.extend(nodes[nid].inputs)
    dropped = [n.kind for nid, n in nodes.items() if nid not in live]
    kept = {nid: n for nid, n in nodes.items() if nid in live}
    return kept, dropped.count(OpKind.SPLIT), dropped.count(OpKind.CONCAT)


def _finalize(name: str, nodes: dict[str, Node], outputs, step: str) -> Graph:
    g = Graph(name, nodes, tuple(outputs))
    rep = validate(g)
    if not rep.ok:
        raise TransformError(f"internal error: {step} produced an invalid graph:\n{rep}")
    return g


def _unchanged(step: str, graph: Graph) -> TransformReport:
    e = cross_device_edges(graph)
    return TransformReport(step=step, cross_device_edges_before=e, cross_device_edges_after=e)


# ---------------------------------------------------------------------------
# step 1
# ---------------------------------------------------------------------------


class _Replicator:
    def __init__(self, graph: Graph, plan: ParallelPlan):
        self.src = graph
        self.d = plan.d
        self.devices = plan.devices
        self.shaped = infer_shapes(graph)
        self.order = topo_order(self.shaped)
        self.out: dict[str, Node] = {}
        self.reps: dict[str, tuple[str, ...]] = {}
        self.splits: dict[str, str] = {}
        self.concats: dict[str, str] = {}

    def kind(self, nid: str) -> OpKind:
        return self.shaped.node(nid).kind

    def full_value(self, tensor: str) -> str:
        """Where a non-replicated consumer now reads the whole tensor."""
        if tensor in self.concats:
            return self.concats[tensor]
        if tensor in self.reps:  # a replicated variable: the dev0 copy stands in
            return self.reps[tensor][0]
        return tensor

    def split_of(self, tensor: str) -> str:
        if tensor in self.splits:
            return self.splits[tensor]
        if self.kind(tensor) is OpKind.VARIABLE:
            raise TransformError(f"activation input {tensor!r} is a Variable; cannot batch-split it")
        shape = self.shaped.node(tensor).output_shape
        if shape.dims[shape.batch_axis] % self.d:
            raise TransformError(f"batch {shape.dims[shape.batch_axis]} of {tensor!r} is not divisible by d={self.d}")
        sid = f"{tensor}/split"
        self.out[sid] = Node(sid, OpKind.SPLIT, (self.full_value(tensor),),
                             {"axis": shape.batch_axis, "parts": self.d})
        self.splits[tensor] = sid
        return sid

    def replicate(self, nid: str) -> None:
        n = self.shaped.node(nid)
        slots = SHARD_SLOTS[n.kind]
        reps = []
        for k in range(self.d):
            ins = []
            for slot, i in enumerate(n.inputs):
                if slot in slots:
                    ins.append(self.split_of(i))
                elif i in self.reps and self.kind(i) is OpKind.VARIABLE:
                    ins.append(self.reps[i][k])
                else:
                    raise TransformError(f"weight input {i!r} of {nid!r} is not a Variable")
            rid = f"{nid}/dev{k}"
            self.out[rid] = Node(rid, n.kind, tuple(ins), dict(n.attrs), self.devices[k])
            reps.append(rid)
        self.reps[nid] = tuple(reps)
        if n.kind in BATCH_OUTPUT_KINDS:
            cid = f"{nid}/concat"
            self.out[cid] = Node(cid, OpKind.CONCAT, tuple(reps), {"axis": n.output_shape.batch_axis},
                                 self.devices[0])
            self.concats[nid] = cid
            return
        users = [c for c in self.shaped.consumers()[nid] if self.kind(c) is not OpKind.SGD_UPDATE]
        stray = [c for c in users if self.kind(c) is not OpKind.ADD_N]
        if stray:
            raise TransformError(f"weight gradient {nid!r} is consumed outside its update: {stray}")

    def producers(self, grad: str) -> tuple[str, ...]:
        if grad in self.reps:
            return self.reps[grad]
        g = self.shaped.node(grad)
        if g.kind is OpKind.ADD_N:
            return tuple(p for part in g.inputs for p in self.producers(part))
        return (self.full_value(grad),)

    def run(self) -> tuple[Graph, TransformReport]:
        order, d = self.order, self.d
        primaries = [nid for nid in order
                     if self.kind(nid) in PRIMARY_KINDS
                     or (self.kind(nid) in GRAD_COMPANION_KINDS and self.shaped.node(nid).attr("layer") is not None)]
        variables = [nid for nid in order if self.kind(nid) is OpKind.VARIABLE]
        updates = {self.shaped.node(nid).inputs[0]: nid for nid in order if self.kind(nid) is OpKind.SGD_UPDATE}

        for v in variables:
            n = self.shaped.node(v)
            ids = []
            for k in range(d):
                rid = f"{v}/dev{k}"
                self.out[rid] = Node(rid, OpKind.VARIABLE, (), dict(n.attrs), self.devices[k])
                ids.append(rid)
            self.reps[v] = tuple(ids)

        replicable = set(primaries)
        for nid in order:
            n = self.shaped.node(nid)
            if n.kind in (OpKind.VARIABLE, OpKind.SGD_UPDATE):
                continue
            if nid in replicable:
                self.replicate(nid)
                continue
            dev = None if n.kind is OpKind.INPUT else (n.device if n.device is not None else self.devices[0])
            self.out[nid] = replace(n, inputs=tuple(self.full_value(i) for i in n.inputs), device=dev,
                                    output_shape=None)

        upd_reps: dict[str, tuple[str, ...]] = {}
        for v in variables:
            if v not in updates:
                continue
            u = self.shaped.node(updates[v])
            feeds = self.producers(u.inputs[1])
            ids = []
            for k in range(d):
                agg = f"{v}/agg/dev{k}"
                self.out[agg] = Node(agg, OpKind.ADD_N, feeds, {"aggregates": v}, self.devices[k])
                rid = f"{u.id}/dev{k}"
                self.out[rid] = Node(rid, OpKind.SGD_UPDATE, (self.reps[v][k], agg), dict(u.attrs),
                                     self.devices[k])
                ids.append(rid)
            upd_reps[u.id] = tuple(ids)

        outputs: list[str] = []
        for o in self.src.outputs:
            if o in upd_reps:
                outputs.extend(upd_reps[o])
            elif o in self.reps and self.kind(o) is OpKind.VARIABLE:
                outputs.extend(self.reps[o])
            else:
                outputs.append(self.full_value(o))
        nodes, _, _ = _sweep(self.out, outputs)
        result = _finalize(self.src.name, nodes, outputs, "step1")
        return result, TransformReport(
            step="step1", nodes_replicated=len(primaries) + len(variables) + len(updates),
            splits_inserted=len(self.splits), concats_inserted=len(self.concats),
            cross_device_edges_before=cross_device_edges(self.src),
            cross_device_edges_after=cross_device_edges(result))


def replicate_primary(graph: Graph, plan: ParallelPlan) -> tuple[Graph, TransformReport]:
    if plan.d == 1:
        return graph, _unchanged("step1", graph)
    if plan.devices != tuple(range(plan.d)):
        raise TransformError(f"replicas need device ids 0..{plan.d - 1}, got {plan.devices}")
    for n in graph:
        if n.kind in INFRA_KINDS or replica_index(n.id) is not None:
            raise TransformError(f"graph is already parallelized: node {n.id!r} is a {n.kind.value}")
    if len(graph.devices()) > 1:
        raise TransformError(f"graph is already parallelized: devices {graph.devices()}")
    rep = validate(graph)
    if not rep.ok:
        raise TransformError(f"input graph invalid:\n{rep}")
    return _Replicator(graph, plan).run()


# ---------------------------------------------------------------------------
# step 2
# ---------------------------------------------------------------------------


def _full_groups(graph: Graph, d: int) -> dict[str, tuple[str, ...]]:
    by_base: dict[str, dict[int, str]] = {}
    for n in graph:
        k = replica_index(n.id)
        if k is not None:
            by_base.setdefault(base_id(n.id), {})[k] = n.id
    return {b: tuple(g[k] for k in range(d)) for b, g in by_base.items()
            if len(g) == d and sorted(g) == list(range(d))}


class _Localizer:
    def __init__(self, graph: Graph, plan: ParallelPlan):
        self.graph = graph
        self.d = plan.d
        self.devices = plan.devices
        self.shaped = infer_shapes(graph)
        self.nodes: dict[str, Node] = dict(self.shaped.nodes)
        self.groups = _full_groups(self.shaped, self.d)
        self.removed = 0
        self.new_splits = 0
        self.cloned = 0

    def users(self, target: str) -> list[str]:
        return sorted(nid for nid, n in self.nodes.items() if target in n.inputs)

    def rewire(self, consumer: str, old: str, new: str) -> None:
        n = self.nodes[consumer]
        self.nodes[consumer] = replace(n, inputs=tuple(new if i == old else i for i in n.inputs),
                                       output_shape=None)

    def per_device(self, tensor: str) -> tuple[str, ...] | None:
        if tensor in self.groups:
            return self.groups[tensor]
        if replica_index(tensor) is not None and base_id(tensor) in self.groups:
            return self.groups[base_id(tensor)]
        n = self.nodes[tensor]
        if n.kind is OpKind.CONCAT and tuple(n.inputs) == self.groups.get(base_id(n.inputs[0]), ()):
            return tuple(n.inputs)
        return None

    def cancel_pairs(self) -> None:
        for nid in list(self.nodes):
            n = self.nodes.get(nid)
            if n is None or n.kind is not OpKind.SPLIT:
                continue
            src = self.nodes[n.inputs[0]]
            if src.kind is not OpKind.CONCAT:
                continue
            if n.attr("axis") != src.attr("axis") or n.attr("parts") != len(src.inputs):
                raise TransformError(f"malformed pair: Concat {src.id!r} feeds Split {nid!r} "
                                     f"with mismatched axis or arity")
            for c in self.users(nid):
                self.rewire(c, nid, src.inputs[self.nodes[c].device])
            del self.nodes[nid]
            self.removed += 1

    def slots_for(self, n: Node) -> list[tuple[str, ...]] | None:
        slots = []
        for i in n.inputs:
            if i not in self.nodes:
                return None
            shards = self.per_device(i)
            if shards is None and self.nodes[i].kind is OpKind.SPLIT:
                shards = (i,) * self.d
            if shards is None:
                inode = self.nodes[i]
                shape = self.shaped.node(i).output_shape if i in self.shaped.nodes else None
                if inode.kind is not OpKind.INPUT or shape is None or shape.batch % self.d:
                    return None
                sid = f"{i}/split"
                if sid not in self.nodes:
                    self.nodes[sid] = Node(sid, OpKind.SPLIT, (i,), {"axis": shape.batch_axis, "parts": self.d})
                    self.new_splits += 1
                shards = (sid,) * self.d
            slots.append(shards)
        return slots

    def clone(self, nid: str) -> None:
        n = self.nodes[nid]
        slots = self.slots_for(n)
        if slots is None:
            return  # conservative: leave the node where it is
        reps = []
        for k in range(self.d):
            rid = f"{nid}/dev{k}"
            self.nodes[rid] = Node(rid, n.kind, tuple(s[k] for s in slots), dict(n.attrs), self.devices[k])
            reps.append(rid)
        self.groups[nid] = tuple(reps)
        self.cloned += 1
        if n.kind in PARTIAL_AUX_KINDS:
            # shard-local partial sums join every aggregator that read the original
            for c in self.users(nid):
                agg = self.nodes[c]
                if agg.kind is OpKind.ADD_N and agg.attr("aggregates") is not None:
                    ins = []
                    for i in agg.inputs:
                        ins.extend(reps if i == nid else (i,))
                    self.nodes[c] = replace(agg, inputs=tuple(ins), output_shape=None)
        elif n.kind in SHARD_AUX_KINDS:
            sid = f"{nid}/split"
            if sid in self.nodes and self.nodes[sid].inputs[0] == nid:
                for c in self.users(sid):
                    self.rewire(c, sid, reps[self.nodes[c].device])
                del self.nodes[sid]
                self.removed += 1

    def run(self) -> tuple[Graph, TransformReport]:
        before = cross_device_edges(self.graph)
        self.cancel_pairs()
        clonable = SHARD_AUX_KINDS | PARTIAL_AUX_KINDS | LOSS_AUX_KINDS
        for nid in topo_order(self.shaped):
            n = self.nodes.get(nid)
            if n is not None and n.kind in clonable and replica_index(nid) is None:
                self.clone(nid)
        outputs: list[str] = []
        for o in self.graph.outputs:
            if o in self.groups and o in self.nodes and replica_index(o) is None:
                outputs.extend(self.groups[o])
            else:
                outputs.append(o)
        nodes, ds, dc = _sweep(self.nodes, outputs)
        self.removed += min(ds, dc)
        result = _finalize(self.graph.name, nodes, outputs, "step2")
        return result, TransformReport(
            step="step2", nodes_replicated=self.cloned, splits_inserted=self.new_splits,
            split_concat_pairs_removed=self.removed, cross_device_edges_before=before,
            cross_device_edges_after=cross_device_edges(result))


def localize_auxiliary(graph: Graph, plan: ParallelPlan) -> tuple[Graph, TransformReport]:
    if plan.d == 1:
        return graph, _unchanged("step2", graph)
    return _Localizer(graph, plan).run()


# ---------------------------------------------------------------------------
# step 3
# ---------------------------------------------------------------------------


def optimize_gradient_aggregation(graph: Graph, plan: ParallelPlan) -> tuple[Graph, TransformReport]:
    if plan.d == 1:
        return graph, _unchanged("step3", graph)
    before = cross_device_edges(graph)
    nodes = dict(graph.nodes)
    clusters: dict[str, list[Node]] = {}
    for n in graph:
        if n.kind is OpKind.ADD_N and n.attr("aggregates") is not None:
            clusters.setdefault(n.attr("aggregates"), []).append(n)
    targets = {base_id(n.inputs[0]) for n in graph if n.kind is OpKind.SGD_UPDATE}
    missing = sorted(targets - set(clusters))
    if missing:
        raise TransformError(f"no AddN aggregation cluster found for variables: {missing}")
    for var, cluster in sorted(clusters.items()):
        if len(cluster) != plan.d:
            raise TransformError(f"variable {var!r} has {len(cluster)} aggregators, expected {plan.d}")
        if len({c.inputs for c in cluster}) != 1:
            raise TransformError(f"aggregators of {var!r} disagree on inputs")
        ar = f"{var}/allreduce"
        nodes[ar] = Node(ar, OpKind.ALL_REDUCE_SUM, cluster[0].inputs, {"aggregates": var})
        gone = {c.id for c in cluster}
        for nid, n in list(nodes.items()):
            if any(i in gone for i in n.inputs):
                nodes[nid] = replace(n, inputs=tuple(ar if i in gone else i for i in n.inputs),
                                     output_shape=None)
        for c in gone:
            del nodes[c]
    result = _finalize(graph.name, nodes, graph.outputs, "step3")
    return result, TransformReport(step="step3", cross_device_edges_before=before,
                                   cross_device_edges_after=cross_device_edges(result),
                                   allreduce_nodes_inserted=len(clusters))


def transform(graph: Graph, plan: ParallelPlan) -> tuple[Graph, list[TransformReport]]:
    """All three rewrites; the identity (with empty reports) when d == 1."""
    if plan.d == 1:
        return graph, [_unchanged(s, graph) for s in ("step1", "step2", "step3")]
    g1, r1 = replicate_primary(graph, plan)
    g2, r2 = localize_auxiliary(g1, plan)
    g3, r3 = optimize_gradient_aggregation(g2, plan)
    problems = check_parallel_structure(g3, plan)
    if problems:
        raise TransformError("transform broke structural invariants:\n" + "\n".join(problems))
    return g3, [r1, r2, r3]


def check_parallel_structure(graph: Graph, plan: ParallelPlan) -> list[str]:
    """One AllReduceSum per variable, no AddN aggregator left, device-local edges
    except collective traffic, and a primary replica on every device."""
    problems: list[str] = []
    variables = {base_id(n.id) for n in graph if n.kind is OpKind.VARIABLE}
    n_ar = sum(1 for n in graph if n.kind is OpKind.ALL_REDUCE_SUM)
    if n_ar != len(variables):
        problems.append(f"expected {len(variables)} AllReduceSum nodes (one per variable), found {n_ar}")
    problems += [f"AddN aggregator {n.id!r} survived step 3" for n in graph
                 if n.kind is OpKind.ADD_N and n.attr("aggregates") is not None]
    for n in graph:
        if n.kind is OpKind.ALL_REDUCE_SUM:
            continue
        dst = _device_of(graph.nodes, n.id)
        for i in n.inputs:
            if graph.node(i).kind is OpKind.ALL_REDUCE_SUM:
                continue
            src = _device_of(graph.nodes, i)
            if src is not None and dst is not None and src != dst:
                problems.append(f"cross-device edge {i!r} (dev {src}) -> {n.id!r} (dev {dst})")
    owned = {k: 0 for k in range(plan.d)}
    for n in graph:
        if n.kind in PRIMARY_KINDS and n.device is not None:
            owned[n.device] = owned.get(n.device, 0) + 1
    empty = [k for k in range(plan.d) if owned.get(k, 0) == 0]
    if empty and any(n.kind in PRIMARY_KINDS for n in graph):
        problems.append(f"devices without a primary replica: {empty}")
    return problems
