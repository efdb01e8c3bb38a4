"""CPU ORACLE (test infrastructure only) -- numpy float64 restatement of the
reference interpreter `wap.interp` (/root/reference/pkg/src/wap/interp.py).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker or the timed CPU
baseline -- never as a product path. The GPU runtime fails loudly without its
CUDA extension; it never routes through here.

Parity pinning:
  * every rule the reference has is restated with the same numpy operations in
    the same order (conv as K*K shifted matmuls, tensordot wgrad, scatter dgrad,
    left-fold AddN/AllReduceSum, pairwise batch means), and is checked against
    the live reference (tests/test_oracle.py) and against committed golden
    outputs of the reference (tests/golden/*.npz, made by tests/golden/make_golden.py);
  * the extension rules (strided/padded Conv2D, MaxPool, LRN and their
    gradients) have no reference counterpart ("parity unpinned" by the
    reference); they reduce exactly to the reference rules at stride 1 /
    'same' padding and are cross-checked against torch.nn.functional in fp64.
"""

from __future__ import annotations

import zlib

import numpy as np

INIT_SCALE = 0.1  # interp.py:36


# ---------------------------------------------------------------------------
# deterministic bindings (interp.py:39-66)
# ---------------------------------------------------------------------------
def rng(seed: int, namespace: str, name: str) -> np.random.Generator:
    """interp.py:39-41: PCG64 keyed by (seed & 0xFFFFFFFF, crc32(f'{ns}:{name}'))."""
    return np.random.default_rng((int(seed) & 0xFFFFFFFF, zlib.crc32(f"{namespace}:{name}".encode("utf-8"))))


def _base(nid: str) -> str:
    import re

    m = re.match(r"^(?P<base>.+)/dev(?P<idx>\d+)$", nid)
    return m.group("base") if m else nid


def initial_variables(graph, seed: int) -> dict[str, np.ndarray]:
    """interp.py:44-56."""
    return {n.id: INIT_SCALE * rng(seed, "var", _base(n.id)).standard_normal(tuple(n.attr("shape")))
            for n in graph if n.kind.value == "Variable"}


def generate_inputs(graph, seed: int) -> dict[str, np.ndarray]:
    """interp.py:59-66."""
    return {n.id: rng(seed, "in", _base(n.id)).standard_normal(tuple(n.attr("shape")))
            for n in graph if n.kind.value == "Input"}


# ---------------------------------------------------------------------------
# per-op rules
# ---------------------------------------------------------------------------
def _geom(attrs: dict, k: int) -> tuple[int, int]:
    return int(attrs.get("stride", 1)), int(attrs.get("padding", k // 2))


def _pad(x: np.ndarray, p: int) -> np.ndarray:
    b, h, w, c = x.shape
    xp = np.zeros((b, h + 2 * p, w + 2 * p, c), dtype=x.dtype)
    xp[:, p:p + h, p:p + w, :] = x
    return xp


def _win(xp: np.ndarray, u: int, v: int, s: int, ho: int, wo: int) -> np.ndarray:
    return xp[:, u:u + s * (ho - 1) + 1:s, v:v + s * (wo - 1) + 1:s, :]


def conv2d(x: np.ndarray, w: np.ndarray, stride: int = 1, padding: int | None = None) -> np.ndarray:
    """interp.py:69-79 (K*K shifted matmuls), generalised to stride/padding."""
    k = w.shape[0]
    p = k // 2 if padding is None else padding
    b, h, wd, _ = x.shape
    ho, wo = (h + 2 * p - k) // stride + 1, (wd + 2 * p - k) // stride + 1
    xp = _pad(x, p)
    out = np.zeros((b, ho, wo, w.shape[3]), dtype=x.dtype)
    for u in range(k):
        for v in range(k):
            out += _win(xp, u, v, stride, ho, wo) @ w[u, v]
    return out


def conv2d_grad_w(x: np.ndarray, dy: np.ndarray, k: int, stride: int = 1, padding: int | None = None) -> np.ndarray:
    """interp.py:82-91 (per-tap tensordot over B,H,W), generalised."""
    p = k // 2 if padding is None else padding
    _, ho, wo, co = dy.shape
    xp = _pad(x, p)
    dw = np.zeros((k, k, x.shape[3], co), dtype=x.dtype)
    for u in range(k):
        for v in range(k):
            dw[u, v] = np.tensordot(_win(xp, u, v, stride, ho, wo), dy, axes=([0, 1, 2], [0, 1, 2]))
    return dw


def conv2d_grad_x(dy: np.ndarray, w: np.ndarray, stride: int = 1, padding: int | None = None,
                  input_hw: tuple[int, int] | None = None) -> np.ndarray:
    """interp.py:94-102 (scatter dy @ W[u,v]^T into the padded input, crop)."""
    k = w.shape[0]
    p = k // 2 if padding is None else padding
    b, ho, wo, _ = dy.shape
    h, wd = (ho, wo) if input_hw is None else input_hw
    # padded extent must hold every tap window
    hp = max(h + 2 * p, stride * (ho - 1) + k)
    wp = max(wd + 2 * p, stride * (wo - 1) + k)
    dxp = np.zeros((b, hp, wp, w.shape[2]), dtype=dy.dtype)
    for u in range(k):
        for v in range(k):
            dxp[:, u:u + stride * (ho - 1) + 1:stride, v:v + stride * (wo - 1) + 1:stride, :] += dy @ w[u, v].T
    return dxp[:, p:p + h, p:p + wd, :]


def softmax(z: np.ndarray) -> np.ndarray:
    """interp.py:109-112."""
    e = np.exp(z - z.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


def left_fold(xs: list[np.ndarray]) -> np.ndarray:
    """interp.py:115-119."""
    acc = xs[0].copy()
    for a in xs[1:]:
        acc = acc + a
    return acc


def xent_loss(logits: np.ndarray, labels: np.ndarray) -> np.ndarray:
    """interp.py:170-175: shard-mean cross entropy, literal formula."""
    z = logits - logits.max(axis=1, keepdims=True)
    logp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
    return np.array([(-(labels * logp).sum(axis=1)).sum() / logits.shape[0]])


def maxpool(x: np.ndarray, window: int, stride: int) -> tuple[np.ndarray, np.ndarray]:
    """Extension. VALID max pooling; argmax = first maximum in row-major window order."""
    b, h, w, c = x.shape
    ho, wo = (h - window) // stride + 1, (w - window) // stride + 1
    stack = np.stack([_win(x, i, j, stride, ho, wo) for i in range(window) for j in range(window)], axis=0)
    arg = stack.argmax(axis=0)  # numpy argmax returns the first maximum
    return np.take_along_axis(stack, arg[None], axis=0)[0], arg


def maxpool_grad(x: np.ndarray, dy: np.ndarray, window: int, stride: int) -> np.ndarray:
    """Extension. Route dy to the first-maximum position of each window."""
    _, ho, wo, _ = dy.shape
    _, arg = maxpool(x, window, stride)
    dx = np.zeros_like(x)
    for i in range(window):
        for j in range(window):
            sel = (arg == i * window + j)
            dx[:, i:i + stride * (ho - 1) + 1:stride, j:j + stride * (wo - 1) + 1:stride, :] += np.where(sel, dy, 0.0)
    return dx


def _lrn_scale(x: np.ndarray, size: int, alpha: float, k: float) -> np.ndarray:
    c = x.shape[-1]
    half = size // 2
    sq = np.concatenate([np.zeros(x.shape[:-1] + (half,)), x * x, np.zeros(x.shape[:-1] + (half,))], axis=-1)
    acc = np.zeros_like(x)
    for j in range(size):
        acc += sq[..., j:j + c]
    return k + alpha * acc


def lrn(x: np.ndarray, size: int, alpha: float, beta: float, bias: float) -> np.ndarray:
    """Extension. Krizhevsky across-channel LRN: x / (bias + alpha*sum x^2)^beta."""
    return x * _lrn_scale(x, size, alpha, bias) ** (-beta)


def lrn_grad(x: np.ndarray, dy: np.ndarray, size: int, alpha: float, beta: float, bias: float) -> np.ndarray:
    """Extension. d/dx of lrn(): dy*s^-b - 2ab x sum_{j~c} dy_j x_j s_j^(-b-1)."""
    s = _lrn_scale(x, size, alpha, bias)
    t = dy * x * s ** (-beta - 1.0)
    c = x.shape[-1]
    half = size // 2
    tp = np.concatenate([np.zeros(x.shape[:-1] + (half,)), t, np.zeros(x.shape[:-1] + (half,))], axis=-1)
    acc = np.zeros_like(x)
    for j in range(size):
        acc += tp[..., j:j + c]
    return dy * s ** (-beta) - 2.0 * alpha * beta * x * acc


# ---------------------------------------------------------------------------
# graph evaluation (interp.py:122-215)
# ---------------------------------------------------------------------------
def _topo(graph) -> list[str]:
    import heapq

    indeg = {n.id: len(n.inputs) for n in graph}
    users: dict[str, list[str]] = {n.id: [] for n in graph}
    for n in graph:
        for i in n.inputs:
            users[i].append(n.id)
    ready = [nid for nid, k in indeg.items() if k == 0]
    heapq.heapify(ready)
    order = []
    while ready:
        nid = heapq.heappop(ready)
        order.append(nid)
        for u in users[nid]:
            indeg[u] -= 1
            if indeg[u] == 0:
                heapq.heappush(ready, u)
    return order


def execute(graph, inputs: dict[str, np.ndarray], seed: int = 0, keep: set[str] | None = None,
            hooks: dict | None = None) -> dict[str, np.ndarray]:
    """Evaluate every node in topological order (ties by id); returns the graph
    outputs (plus any ids in `keep`). Works on the reference's Graph objects or
    this package's (duck-typed: id, kind.value, inputs, attrs, device).
    `hooks` maps a kind name to fn(node, input_values) overriding its rule
    (tests use it to put a real gloo allreduce behind a rank-local AllReduceSum)."""
    vals: dict[str, object] = {}
    nodes = {n.id: n for n in graph}

    def fetch(consumer, pid):
        v = vals[pid]
        if isinstance(v, tuple):  # Split parts are picked by the consumer's device
            if consumer.device is None or not 0 <= consumer.device < len(v):
                raise ValueError(f"node {consumer.id!r} consumes split {pid!r} but has no part device")
            return v[consumer.device]
        return v

    for nid in _topo(graph):
        n = nodes[nid]
        kind = n.kind.value
        a = n.attrs
        if kind == "Input":
            vals[nid] = np.asarray(inputs[nid], dtype=np.float64)
            continue
        if kind == "Variable":
            if nid in inputs:
                vals[nid] = np.asarray(inputs[nid], dtype=np.float64)
            else:
                vals[nid] = INIT_SCALE * rng(seed, "var", _base(nid)).standard_normal(tuple(a["shape"]))
            continue
        ins = [fetch(n, i) for i in n.inputs]
        if hooks and kind in hooks:
            vals[nid] = hooks[kind](n, ins)
            continue
        if kind == "MatMul":
            x = ins[0].reshape(ins[0].shape[0], -1) if a.get("flatten_lhs") else ins[0]
            out = x @ ins[1]
        elif kind == "Conv2D":
            s, p = _geom(a, ins[1].shape[0])
            out = conv2d(ins[0], ins[1], s, p)
        elif kind == "BiasAdd":
            out = ins[0] + ins[1]
        elif kind == "ReLU":
            out = np.maximum(ins[0], 0.0)
        elif kind == "SoftmaxXentLoss":
            out = xent_loss(ins[0], ins[1])
        elif kind == "Split":
            out = tuple(np.split(ins[0], a["parts"], axis=a["axis"]))
        elif kind == "Concat":
            out = np.concatenate(ins, axis=a["axis"])
        elif kind in ("AddN", "AllReduceSum"):
            out = left_fold(ins)
        elif kind == "GradMatMulW":
            x = ins[0].reshape(ins[0].shape[0], -1) if a.get("flatten_lhs") else ins[0]
            out = x.T @ ins[1]
        elif kind == "GradMatMulX":
            out = ins[0] @ ins[1].T
            if a.get("lhs_dims") is not None:
                out = out.reshape((out.shape[0], *a["lhs_dims"]))
        elif kind == "GradConv2DW":
            k = a["kernel_size"]
            s, p = _geom(a, k)
            out = conv2d_grad_w(ins[0], ins[1], k, s, p)
        elif kind == "GradConv2DX":
            s, p = _geom(a, ins[1].shape[0])
            hw = a.get("input_hw")
            out = conv2d_grad_x(ins[0], ins[1], s, p, tuple(hw) if hw is not None else None)
        elif kind == "GradBias":
            out = ins[0].sum(axis=tuple(range(ins[0].ndim - 1)))
        elif kind == "GradReLU":
            out = ins[1] * (ins[0] > 0)
        elif kind == "GradSoftmaxXent":
            out = (softmax(ins[0]) - ins[1]) / a.get("denominator", ins[0].shape[0])
        elif kind == "SgdUpdate":
            out = ins[0] - a["learning_rate"] * ins[1]
        elif kind == "MaxPool":
            out = maxpool(ins[0], a["window"], a["stride"])[0]
        elif kind == "GradMaxPool":
            out = maxpool_grad(ins[0], ins[1], a["window"], a["stride"])
        elif kind == "LRN":
            out = lrn(ins[0], a["size"], a["alpha"], a["beta"], a["bias"])
        elif kind == "GradLRN":
            out = lrn_grad(ins[0], ins[1], a["size"], a["alpha"], a["beta"], a["bias"])
        else:
            raise ValueError(f"no oracle rule for kind {kind}")
        vals[nid] = out
    want = list(graph.outputs) + sorted(keep or ())
    return {o: vals[o] for o in want}


def relative_deviation(a: np.ndarray, b: np.ndarray) -> float:
    """interp.py:242-246: max|a-b| / max(max|a|, max|b|, 1e-30)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"output shapes differ: {a.shape} vs {b.shape}")
    scale = max(float(np.abs(a).max(initial=0.0)), float(np.abs(b).max(initial=0.0)), 1e-30)
    return float(np.abs(a - b).max(initial=0.0)) / scale
