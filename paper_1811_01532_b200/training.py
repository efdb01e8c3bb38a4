"""Forward graph -> full single-device training step (forward, backward, SGD).

Same construction as the reference builder (training.py:44-168), so the
emitted node ids, attributes and wiring are identical for every graph the
reference can express:
  * one explicit gradient node per (op, differentiable input);
  * the loss seed is GradSoftmaxXent(logits, labels) with
    `denominator` = the batch it was built for (training.py:94-102) -- after
    sharding every replica keeps the *global* denominator, which is why the
    gradient allreduce is a pure sum with no 1/N;
  * multiple contributions to one tensor are summed by an AddN `d_<tensor>`;
  * BiasAdd passes its upstream gradient straight through to x;
  * one SgdUpdate `<var>_upd` per trained variable, in the order given.

Extensions: MaxPool -> GradMaxPool(x, dy), LRN -> GradLRN(x, dy), and strided /
explicitly padded Conv2D carry `stride` / `padding` (and `input_hw` on the
input gradient) onto their gradient nodes.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import BuildError
from .ir import DIFFERENTIABLE_KINDS, Graph, Node, OpKind, infer_shapes, topo_order, validate


@dataclass(frozen=True)
class TrainingGraphSpec:
    forward: Graph
    loss_node: str
    learning_rate: float
    variables: tuple[str, ...]


def _check_spec(spec: TrainingGraphSpec) -> None:
    fwd = spec.forward
    rep = validate(fwd)
    if not rep.ok:
        raise BuildError(f"forward graph invalid:\n{rep}")
    if spec.learning_rate <= 0:
        raise BuildError(f"learning rate must be positive, got {spec.learning_rate}")
    for n in fwd:
        if n.kind not in DIFFERENTIABLE_KINDS:
            raise BuildError(f"non-differentiable op: node {n.id!r} has kind {n.kind.value}")
    if spec.loss_node not in fwd.nodes:
        raise BuildError(f"loss node {spec.loss_node!r} not in forward graph")
    if fwd.node(spec.loss_node).kind is not OpKind.SOFTMAX_XENT_LOSS:
        raise BuildError(
            f"loss node {spec.loss_node!r} must be a SoftmaxXentLoss, got {fwd.node(spec.loss_node).kind.value}"
        )
    for v in spec.variables:
        if v not in fwd.nodes or fwd.node(v).kind is not OpKind.VARIABLE:
            raise BuildError(f"{v!r} is not a Variable in the forward graph")


class _Backward:
    """Accumulates gradient nodes while sweeping the forward graph in reverse."""

    def __init__(self, fwd: Graph):
        self.shaped = infer_shapes(fwd)
        self.order = topo_order(self.shaped)
        self.users = self.shaped.consumers()
        self.nodes: dict[str, Node] = dict(fwd.nodes)
        self.needs: dict[str, bool] = {}
        for nid in self.order:
            n = self.shaped.node(nid)
            self.needs[nid] = n.kind is OpKind.VARIABLE or any(self.needs[i] for i in n.inputs)
        self.parts: dict[str, list[str]] = {nid: [] for nid in self.order}
        self.grad: dict[str, str] = {}

    def emit(self, kind: OpKind, nid: str, inputs: tuple[str, ...], **attrs) -> str:
        if nid in self.nodes:
            raise BuildError(f"gradient node id {nid!r} collides with an existing node")
        self.nodes[nid] = Node(nid, kind, inputs, attrs)
        return nid

    def gid(self, tensor: str, via: str) -> str:
        # A tensor feeding several consumers gets one partial gradient per consumer.
        return f"d_{tensor}" if len(self.users[tensor]) == 1 else f"d_{tensor}_via_{via}"

    def push(self, tensor: str, grad_node: str) -> None:
        self.parts[tensor].append(grad_node)

    # -- per-kind rules -----------------------------------------------------
    def matmul(self, n: Node, g: str) -> None:
        x, w = n.inputs
        flat = bool(n.attr("flatten_lhs"))
        if self.needs[w]:
            extra = {"flatten_lhs": True} if flat else {}
            self.push(w, self.emit(OpKind.GRAD_MATMUL_W, self.gid(w, n.id), (x, g), layer=n.id, **extra))
        if self.needs[x]:
            extra = {"lhs_dims": tuple(self.shaped.node(x).output_shape.dims[1:])} if flat else {}
            self.push(x, self.emit(OpKind.GRAD_MATMUL_X, self.gid(x, n.id), (g, w), layer=n.id, **extra))

    def conv(self, n: Node, g: str) -> None:
        x, w = n.inputs
        k = self.shaped.node(w).output_shape.dims[0]
        geom = {a: n.attrs[a] for a in ("stride", "padding") if a in n.attrs}
        if self.needs[w]:
            self.push(w, self.emit(OpKind.GRAD_CONV2D_W, self.gid(w, n.id), (x, g), layer=n.id,
                                   kernel_size=k, **geom))
        if self.needs[x]:
            extra = dict(geom)
            if geom:
                extra["input_hw"] = tuple(self.shaped.node(x).output_shape.dims[1:3])
            self.push(x, self.emit(OpKind.GRAD_CONV2D_X, self.gid(x, n.id), (g, w), layer=n.id, **extra))

    def bias_add(self, n: Node, g: str) -> None:
        x, b = n.inputs
        if self.needs[b]:
            self.push(b, self.emit(OpKind.GRAD_BIAS, self.gid(b, n.id), (g,)))
        if self.needs[x]:
            self.push(x, g)

    def unary(self, n: Node, g: str, kind: OpKind) -> None:
        (x,) = n.inputs
        if self.needs[x]:
            self.push(x, self.emit(kind, self.gid(x, n.id), (x, g), **dict(n.attrs)))

    def run(self, loss: Node) -> None:
        logits, labels = loss.inputs
        batch = self.shaped.node(logits).output_shape.batch
        self.push(logits, self.emit(OpKind.GRAD_SOFTMAX_XENT, f"d_{logits}", (logits, labels),
                                    denominator=batch))
        for nid in reversed(self.order):
            n = self.shaped.node(nid)
            if nid == loss.id or not self.needs[nid] or not self.parts[nid]:
                continue
            parts = self.parts[nid]
            g = parts[0] if len(parts) == 1 else self.emit(OpKind.ADD_N, f"d_{nid}", tuple(parts))
            self.grad[nid] = g
            if n.kind is OpKind.MATMUL:
                self.matmul(n, g)
            elif n.kind is OpKind.CONV2D:
                self.conv(n, g)
            elif n.kind is OpKind.BIAS_ADD:
                self.bias_add(n, g)
            elif n.kind is OpKind.RELU:
                self.unary(n, g, OpKind.GRAD_RELU)
            elif n.kind is OpKind.MAX_POOL:
                self.unary(n, g, OpKind.GRAD_MAX_POOL)
            elif n.kind is OpKind.LRN:
                self.unary(n, g, OpKind.GRAD_LRN)
            # Inputs / Variables are leaves.


def build_training_graph(spec: TrainingGraphSpec) -> Graph:
    """Append backward nodes and per-variable SgdUpdates to `spec.forward`."""
    _check_spec(spec)
    fwd = spec.forward
    bw = _Backward(fwd)
    bw.run(fwd.node(spec.loss_node))
    updates = []
    for v in spec.variables:
        if v not in bw.grad:
            raise BuildError(f"variable {v!r} is not reachable from the loss")
        updates.append(bw.emit(OpKind.SGD_UPDATE, f"{v}_upd", (v, bw.grad[v]),
                               learning_rate=spec.learning_rate))
    graph = Graph(f"{fwd.name}_train", bw.nodes, (spec.loss_node, *updates))
    rep = validate(graph)
    if not rep.ok:
        raise BuildError(f"internal error, built graph invalid:\n{rep}")
    return graph
