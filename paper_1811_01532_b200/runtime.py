"""GPU runtime: lower a (per-device) WAP training graph to a static sequence of
sm_100a kernel launches over preallocated HBM buffers.

This is the B200 replacement of the reference's per-OpKind interpreter loop
(interp.py:145-210). Instead of evaluating nodes one by one in fp64 numpy, a
`Program`:

1. chooses a strategy per Conv2D: `shifted` (stride-1 same conv with Ci % 32
   == 0: a tcgen05 shifted GEMM over the padded-flat NHWC grid, no im2col
   traffic) or `im2col` (first layers / strided / odd channel counts: one im2col
   pass, then the same tcgen05 GEMM; the column buffer is reused by the weight
   gradient);
2. fuses what the reference keeps as separate nodes: Conv2D/MatMul + BiasAdd +
   ReLU in the GEMM epilogue, GradReLU into the producer of its upstream
   gradient (dgrad / FC-dX epilogue, MaxPool/LRN backward, col2im),
   SoftmaxXentLoss + GradSoftmaxXent in one kernel;
3. assigns every tensor a layout (NHWC with `pad` trailing zero columns per
   image row and zero rows per image, and a channel stride `ld` rounded to 4) by solving "same grid" constraints with a
   union-find, so a conv's input, output, gradients and weight-gradient
   operands share one padded-flat grid;
4. allocates all buffers once (variables and their gradients in two flat
   arenas with identical offsets, so SGD and the gradient allreduce are
   contiguous bucket operations), pre-encodes every TMA descriptor, and records
   the launch list; `run()` replays it on the current stream and `capture()`
   turns it into a CUDA graph.

Graph outputs keep the reference semantics exactly (loss = shard mean,
updated variables), so `execute()` in interp.py is a drop-in for
`wap.interp.execute`. There is no host fallback: without the native library
every constructor raises.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import EvalError
from .ir import Graph, Node, OpKind, conv_geometry, infer_shapes, topo_order

SHIFTED_MAX_TAPS = N.MAX_TAPS


def _ceil4(x: int) -> int:
    return (x + 3) // 4 * 4


class _UF:
    def __init__(self):
        self.p: dict[str, str] = {}

    def find(self, a: str) -> str:
        self.p.setdefault(a, a)
        while self.p[a] != a:
            self.p[a] = self.p[self.p[a]]
            a = self.p[a]
        return a

    def union(self, a: str, b: str) -> None:
        ra, rb = self.find(a), self.find(b)
        if ra != rb:
            self.p[rb] = ra


@dataclass
class Tensor:
    """A device buffer plus its layout. `dims` are the logical dims."""

    dims: tuple[int, ...]
    pad: int
    ld: int
    buf: object  # torch.Tensor (storage view)
    kind: str    # 'nhwc' | 'mat' | 'vec' | 'kkio'

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    def layout(self) -> N.wap_layout_t:
        l = N.wap_layout_t()
        if self.kind == "nhwc":
            b, h, w, c = self.dims
            l.B, l.H, l.W, l.C, l.pad = b, h, w, c, self.pad
        elif self.kind == "mat":
            l.B, l.H, l.W, l.C, l.pad = self.dims[0], 1, 1, self.dims[1], 0
        elif self.kind == "kkio":
            k, _, ci, co = self.dims
            l.B, l.H, l.W, l.C, l.pad = k * k * ci, 1, 1, co, 0
        else:  # vec
            l.B, l.H, l.W, l.C, l.pad = 1, 1, 1, self.dims[0], 0
        l.ld = self.ld
        return l

    @property
    def rows(self) -> int:
        """Rows of the 2D [rows, ld] view (padded grid rows for NHWC)."""
        if self.kind == "nhwc":
            b, h, w, _ = self.dims
            return b * (h + self.pad) * (w + self.pad)
        if self.kind == "mat":
            return self.dims[0]
        if self.kind == "kkio":
            k, _, ci, _ = self.dims
            return k * k * ci
        return 1

    def numel_storage(self) -> int:
        return self.rows * self.ld


def storage_kind(dims: tuple[int, ...], is_conv_weight: bool = False) -> str:
    if is_conv_weight:
        return "kkio"
    return {4: "nhwc", 2: "mat", 1: "vec"}.get(len(dims), "bad")


@dataclass
class Step:
    name: str
    fn: object
    args: tuple
    what: str = ""
    keep: list = field(default_factory=list)  # objects that must outlive the step (plans, ctypes arrays)
    alg_bytes: int = 0  # algorithmic HBM bytes per launch (each logical element read/written once)

    def __call__(self, stream: int) -> None:
        rc = self.fn(*self.args, stream) if self.fn is not None else 0
        if rc:
            N.check(rc, f"{self.what or self.name}")


class _GemmStep:
    def __init__(self, name, call):
        self.name = name
        self.call = call

    def __call__(self, stream: int) -> None:
        N.check(N.lib().wap_gemm_plan_run(self.call._plan, stream), f"gemm {self.name}")


class Program:
    """A lowered training step for one device.

    graph:        a training graph (single-device, a transformed multi-device
                  graph evaluated in this one process, or a rank view whose
                  AllReduceSum nodes have a single local input).
    precision:    3 = 3xTF32 (fp32-accurate, default), 1 = TF32.
    in_place:     SgdUpdate overwrites the variable buffers (training loop);
                  otherwise updates go to fresh output buffers (execute()).
    collective:   callable(arena slice) performing the cross-rank SUM of a
                  gradient bucket in place (NCCL / gloo; None: single process).
    fused:        a peer_memory.FusedAllReduce: the variable / gradient arenas
                  live in peer-mapped memory and every bucket's allreduce + SGD
                  is ONE wap_allreduce_sgd launch (replaces `collective`).
    """

    def __init__(self, graph: Graph, precision: int = 3, device=None, in_place: bool = False,
                 collective=None, bucket_bytes: int = 64 << 20, autotune: bool | None = None, fused=None,
                 collective_capturable: bool = False):
        import torch

        import os

        self._collectives: list = []
        self.bucket_bytes = bucket_bytes
        self.autotune = autotune if autotune is not None else os.environ.get("WAP_AUTOTUNE", "1") != "0"
        self.buckets: list = []

        self.torch = torch
        self.L = N.lib()
        if not torch.cuda.is_available():
            raise N.NativeUnavailable("CUDA device required: the WAP runtime has no host fallback")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.g = infer_shapes(graph)
        self.order = topo_order(self.g)
        self.users = self.g.consumers()
        self.precision = precision
        self.in_place = in_place
        self.collective = collective
        self.collective_capturable = collective_capturable  # NCCL: recordable into the step's CUDA graph
        self.fused = fused
        if fused is not None and (collective is not None or not in_place):
            raise EvalError("the fused allreduce + SGD needs an in-place training program and no other collective")
        self.t: dict[str, Tensor] = {}
        self.steps: list = []
        self.update_steps: list = []
        self.graph_exec = None
        with torch.cuda.device(self.device):
            self._analyze()
            self._layouts()
            self._allocate()
            self._lower()

    # ------------------------------------------------------------------ utils
    def node(self, nid: str) -> Node:
        return self.g.node(nid)

    def dims(self, nid: str) -> tuple[int, ...]:
        return self.g.node(nid).output_shape.dims

    def kind(self, nid: str) -> OpKind:
        return self.g.node(nid).kind

    # --------------------------------------------------------------- analysis
    def _conv_of_weight(self, w: str) -> str:
        convs = [u for u in self.users[w] if self.kind(u) is OpKind.CONV2D and self.node(u).inputs[1] == w]
        if len(convs) != 1:
            raise EvalError(f"cannot associate weight {w!r} with a unique Conv2D")
        return convs[0]

    def _conv_of_wgrad(self, n: Node) -> str:
        x, g = n.inputs
        k = n.attr("kernel_size")
        cands = [u for u in self.users[x] if self.kind(u) is OpKind.CONV2D and self.node(u).inputs[0] == x
                 and self.node(u).device == n.device
                 and self.dims(self.node(u).inputs[1])[0] == k and self.dims(u) == self.dims(g)
                 and conv_geometry(self.node(u), k) == conv_geometry(n, k)]
        if len(cands) != 1:
            raise EvalError(f"cannot associate {n.id!r} with a unique Conv2D")
        return cands[0]

    def _analyze(self) -> None:
        g = self.g
        outputs = set(g.outputs)
        self.strategy: dict[str, str] = {}
        for nid in self.order:
            n = self.node(nid)
            if n.kind is OpKind.CONV2D:
                k = self.dims(n.inputs[1])[0]
                s, p = conv_geometry(n, k)
                ci = self.dims(n.inputs[0])[3]
                ok = s == 1 and p == k // 2 and k % 2 == 1 and ci % 32 == 0 and k * k <= SHIFTED_MAX_TAPS
                if ok:
                    self.strategy[nid] = "shifted"
                elif self._s2d_geometry(n):
                    self.strategy[nid] = "s2d"
                elif self._direct_ok(n):
                    self.strategy[nid] = "direct"
                else:
                    self.strategy[nid] = "im2col"
        # forward epilogue fusion: producer -> (bias node | None, relu node | None)
        self.fwd_fuse: dict[str, tuple[str | None, str | None]] = {}
        self.virtual: set[str] = set()
        self.mask_alias: dict[str, str] = {}
        for nid in self.order:
            n = self.node(nid)
            if n.kind not in (OpKind.CONV2D, OpKind.MATMUL) or nid in outputs:
                continue
            us = self.users[nid]
            if len(us) != 1 or self.kind(us[0]) is not OpKind.BIAS_ADD or self.node(us[0]).inputs[0] != nid:
                continue
            zb = us[0]
            if self.kind(self.node(zb).inputs[1]) is not OpKind.VARIABLE:
                continue
            zu = self.users[zb]
            relus = [u for u in zu if self.kind(u) is OpKind.RELU]
            others = [u for u in zu if u not in relus]
            if len(relus) == 1 and zb not in outputs and \
                    all(self.kind(u) is OpKind.GRAD_RELU and self.node(u).inputs[0] == zb for u in others):
                r = relus[0]
                self.fwd_fuse[nid] = (zb, r)
                self.virtual |= {nid, zb}
                self.mask_alias[zb] = r
            else:
                self.fwd_fuse[nid] = (zb, None)
                self.virtual.add(nid)
        # a shifted conv's output lives on its input's padded grid; a conv that
        # feeds a flattening MatMul needs compact rows instead -> im2col
        flat_inputs = {self.node(u).inputs[0] for u in self.order
                       if self.kind(u) in (OpKind.MATMUL, OpKind.GRAD_MATMUL_W) and self.node(u).attr("flatten_lhs")}
        for nid, strat in self.strategy.items():
            if strat == "shifted" and self.fused_out(nid) in flat_inputs:
                self.strategy[nid] = "im2col"
        # backward: GradReLU fused into the producer of its upstream gradient
        self.bwd_mask: dict[str, str] = {}  # producer -> GradReLU node it writes for
        fusable = (OpKind.GRAD_MATMUL_X, OpKind.GRAD_CONV2D_X, OpKind.GRAD_MAX_POOL, OpKind.GRAD_LRN)
        for nid in self.order:
            n = self.node(nid)
            if n.kind is not OpKind.GRAD_RELU:
                continue
            prod = n.inputs[1]
            if self.kind(prod) in fusable and self.users[prod] == [nid] and prod not in outputs:
                self.bwd_mask[prod] = nid
                self.virtual.add(prod)
        # softmax cross-entropy pairs
        self.xent: dict[tuple[str, str], dict[str, str]] = {}
        for nid in self.order:
            n = self.node(nid)
            if n.kind in (OpKind.SOFTMAX_XENT_LOSS, OpKind.GRAD_SOFTMAX_XENT):
                key = tuple(n.inputs)
                self.xent.setdefault(key, {})["loss" if n.kind is OpKind.SOFTMAX_XENT_LOSS else "grad"] = nid
        # MaxPool argmax owners: (input, window, stride) -> MaxPool node
        self.pool_of: dict[tuple, str] = {}
        self._pool_lrn: dict[str, tuple] = {}  # GradLRN id -> its fused GradMaxPool operands
        self._lrn_pool: dict[str, Node] = {}  # MaxPool id -> the LRN fused into its forward
        for nid in self.order:
            n = self.node(nid)
            if n.kind is OpKind.MAX_POOL:
                self.pool_of[(n.inputs[0], n.attr("window"), n.attr("stride"))] = nid
        # ReLU outputs of forward conv GEMMs used as the GradReLU mask of a shifted conv
        # dgrad GEMM: the forward epilogue also writes them as bits (1 bit per element),
        # and the dgrad epilogue reads 4 bytes per 32 columns instead of 128
        self.bits_src: set[str] = set()
        if os.environ.get("WAP_NO_MASK_BITS") is None:
            relu_out = {self.fused_out(c): c for c in self.order
                        if self.kind(c) is OpKind.CONV2D and self.fwd_fuse.get(c, (None, None))[1] is not None}
            for prod, gr in self.bwd_mask.items():
                if self.kind(prod) is not OpKind.GRAD_CONV2D_X:
                    continue
                conv = self._conv_of_weight(self.node(prod).inputs[1])
                src = self.mask_src(self.node(gr).inputs[0])
                if self.strategy.get(conv) == "shifted" and src in relu_out:
                    self.bits_src.add(src)
        self.mask_bits: dict[str, object] = {}
        # pools whose every backward is fused with the GradReLU of the ReLU feeding them:
        # the argmax can carry that mask (WAP_POOL_RELU_FUSED)
        self.pool_relu_fused: set[str] = set()
        for key, pool in self.pool_of.items():
            x_id = key[0]
            grads = [u for u in self.order if self.kind(u) is OpKind.GRAD_MAX_POOL
                     and (self.node(u).inputs[0], self.node(u).attr("window"), self.node(u).attr("stride")) == key]
            if grads and all(g in self.bwd_mask and
                             self.mask_src(self.node(self.bwd_mask[g]).inputs[0]) == self.mask_src(x_id)
                             for g in grads):
                self.pool_relu_fused.add(pool)

    def _direct_ok(self, n: Node) -> bool:
        """First-layer stride-1 conv over a <=4-channel graph input (one float4 per
        pixel): computed directly on CUDA cores (wap_conv_direct), no im2col GEMM."""
        if self.kind(n.inputs[0]) is not OpKind.INPUT or os.environ.get("WAP_NO_DIRECT"):
            return False
        k = self.dims(n.inputs[1])[0]
        s, p = conv_geometry(n, k)
        ci = self.dims(n.inputs[0])[3]
        co = self.dims(n.id)[3]
        return s == 1 and ci <= 4 and co % 32 == 0 and k * k * ci * 32 * 4 <= 48 * 1024

    def _s2d_geometry(self, n: Node):
        """Space-to-depth plan of a strided conv over a graph input (first layer, no
        dgrad): (s, p, ks, Hs, Ws, ldc, halo) when the stride-s conv equals a
        ks x ks VALID stride-1 conv over the s2d grid, else None."""
        if self.kind(n.inputs[0]) is not OpKind.INPUT or os.environ.get("WAP_NO_S2D"):
            return None
        k = self.dims(n.inputs[1])[0]
        s, p = conv_geometry(n, k)
        b, h, w, c = self.dims(n.inputs[0])
        _, ho, wo, _ = self.dims(n.id)
        if s < 2 or (h + 2 * p) % s or (w + 2 * p) % s:
            return None
        ks = -(-k // s)
        hs, ws = (h + 2 * p) // s, (w + 2 * p) // s
        if hs - ks + 1 != ho or ws - ks + 1 != wo or hs - ho != ws - wo or ks * ks > SHIFTED_MAX_TAPS:
            return None
        ldc = -(-(s * s * c) // 32) * 32
        return s, p, ks, hs, ws, ldc, hs - ho

    def _bits_out(self, out_id: str):
        """(see _gemm: dropped again if the producing GEMM would split K)"""
        return self._bits_alloc(out_id)

    def _bits_alloc(self, out_id: str):
        """Bit-packed ReLU mask buffer for a forward conv output (None if not needed)."""
        if out_id not in self.bits_src:
            return None
        t = self.t[out_id]
        ldw = -(-t.dims[-1] // 32)
        buf = self.torch.zeros(t.rows * ldw, dtype=self.torch.int32, device=self.device)
        buf.ld_words = ldw
        self.mask_bits[out_id] = buf
        return buf

    def mask_src(self, nid: str) -> str:
        return self.mask_alias.get(nid, nid)

    def fused_out(self, nid: str) -> str:
        """The tensor a (possibly fused) Conv2D/MatMul actually writes."""
        if nid in self.fwd_fuse:
            zb, r = self.fwd_fuse[nid]
            return r if r is not None else zb
        return nid

    # ---------------------------------------------------------------- layouts
    def _layouts(self) -> None:
        uf = _UF()
        lb: dict[str, int] = {}
        for nid in self.order:
            uf.find(nid)

        def need(t, p):
            lb[t] = max(lb.get(t, 0), p)

        for nid, (zb, r) in self.fwd_fuse.items():
            uf.union(nid, zb)
            if r is not None:
                uf.union(nid, r)
        for prod, gr in self.bwd_mask.items():
            uf.union(prod, gr)
        for nid in self.order:
            n = self.node(nid)
            if n.kind is OpKind.CONV2D:
                out = self.fused_out(nid)
                if self.strategy[nid] == "shifted":
                    k = self.dims(n.inputs[1])[0]
                    uf.union(n.inputs[0], out)
                    need(n.inputs[0], k // 2)
                elif self.strategy[nid] == "s2d":
                    need(out, self._s2d_geometry(n)[6])  # output grid = the s2d grid
            elif n.kind is OpKind.GRAD_CONV2D_X:
                conv = self._conv_of_weight(n.inputs[1])
                uf.union(n.inputs[0], self.fused_out(conv))
                if self.strategy[conv] == "shifted":
                    uf.union(nid, self.node(conv).inputs[0])
                    if nid in self.bwd_mask:
                        uf.union(nid, self.mask_src(self.node(self.bwd_mask[nid]).inputs[0]))
            elif n.kind is OpKind.GRAD_CONV2D_W:
                conv = self._conv_of_wgrad(n)
                uf.union(n.inputs[1], self.fused_out(conv))
                if self.strategy[conv] == "shifted":
                    uf.union(n.inputs[0], self.fused_out(conv))
            elif n.kind is OpKind.GRAD_MATMUL_X and nid in self.bwd_mask:
                uf.union(nid, self.mask_src(self.node(self.bwd_mask[nid]).inputs[0]))
            elif n.kind is OpKind.SPLIT:
                uf.union(nid, n.inputs[0])
            elif n.kind in (OpKind.ADD_N, OpKind.ALL_REDUCE_SUM):
                for i in n.inputs:
                    uf.union(nid, i)
            elif n.kind is OpKind.GRAD_RELU and nid not in self.bwd_mask.values():
                pass  # elementwise kernel handles any pair of layouts
        pad_of_class: dict[str, int] = {}
        for t, p in lb.items():
            r = uf.find(t)
            pad_of_class[r] = max(pad_of_class.get(r, 0), p)
        self.pad = {nid: (pad_of_class.get(uf.find(nid), 0) if len(self.dims(nid)) == 4 else 0)
                    for nid in self.order}
        # flatten MatMul inputs must be compact rows
        for nid in self.order:
            n = self.node(nid)
            if n.kind in (OpKind.MATMUL, OpKind.GRAD_MATMUL_W) and n.attr("flatten_lhs"):
                x = n.inputs[0]
                d = self.dims(x)
                if self.pad[x] or d[-1] % 4:
                    raise EvalError(f"flatten of {x!r} needs an unpadded layout with C % 4 == 0, got pad "
                                    f"{self.pad[x]} C {d[-1]}")

    # ------------------------------------------------------------- allocation
    def _new(self, dims, pad=0, kind=None, zero=True, arena=None) -> Tensor:
        torch = self.torch
        kind = kind or storage_kind(dims)
        ld = _ceil4(dims[-1])
        t = Tensor(tuple(dims), pad, ld, None, kind)
        n = t.numel_storage()
        if arena is not None:
            t.buf = arena(n)
        else:
            alloc = torch.zeros if zero else torch.empty
            t.buf = alloc(n, dtype=torch.float32, device=self.device)
        return t

    def _allocate(self) -> None:
        torch = self.torch
        g = self.g
        # variables and their update gradients live in two arenas with equal offsets
        self.var_ids = [nid for nid in self.order if self.kind(nid) is OpKind.VARIABLE]
        conv_w = {self.node(u).inputs[1] for u in self.order if self.kind(u) is OpKind.CONV2D}
        sizes = {}
        for v in self.var_ids:
            d = self.dims(v)
            t = Tensor(d, 0, _ceil4(d[-1]), None, storage_kind(d, v in conv_w))
            sizes[v] = _ceil4(t.numel_storage())
        # gradient arena ordered by reverse topological position of the update
        # (= the order backward produces gradients) so buckets are contiguous
        self.updates = [nid for nid in self.order if self.kind(nid) is OpKind.SGD_UPDATE]
        order_pos = {nid: i for i, nid in enumerate(self.order)}

        def grad_ready(u):
            return order_pos[self.node(u).inputs[1]]

        upd_sorted = sorted(self.updates, key=grad_ready, reverse=True)
        arena_vars = [self.node(u).inputs[0] for u in upd_sorted]
        arena_vars += [v for v in self.var_ids if v not in arena_vars]
        self.arena_off: dict[str, int] = {}
        off = 0
        for v in arena_vars:
            self.arena_off[v] = off
            off += sizes[v]
        self.arena_numel = max(off, 4)
        if self.fused is not None:
            # peer-mapped (and multicast) arenas: every rank's fused allreduce + SGD
            # reads our gradients and writes our variables directly
            self.var_arena, self.grad_arena = self.fused.allocate(self.arena_numel)
        else:
            self.var_arena = torch.zeros(self.arena_numel, dtype=torch.float32, device=self.device)
            self.grad_arena = torch.zeros(self.arena_numel, dtype=torch.float32, device=self.device)
        for v in self.var_ids:
            d = self.dims(v)
            o = self.arena_off[v]
            self.t[v] = Tensor(d, 0, _ceil4(d[-1]), self.var_arena[o:o + sizes[v]], storage_kind(d, v in conv_w))
        # the gradient each update consumes is written straight into the grad arena
        self.grad_slot: dict[str, str] = {}
        for u in self.updates:
            v, gsrc = self.node(u).inputs
            o = self.arena_off[v]
            d = self.dims(v)
            if gsrc in self.t or self.kind(gsrc) in (OpKind.VARIABLE, OpKind.INPUT):
                continue
            target = gsrc
            gn = self.node(gsrc)
            if gn.kind is OpKind.ALL_REDUCE_SUM and len(gn.inputs) == 1:
                target = gn.inputs[0]  # rank view: the local gradient IS the allreduce buffer
            slot = Tensor(d, 0, _ceil4(d[-1]), self.grad_arena[o:o + sizes[v]], storage_kind(d, v in conv_w))
            self.t[target] = slot
            self.t[gsrc] = slot
            self.grad_slot[target] = v
        # activations / gradients
        for nid in self.order:
            n = self.node(nid)
            if nid in self.t or nid in self.virtual:
                continue
            if n.kind is OpKind.SPLIT:
                continue  # views, created during lowering
            if n.kind is OpKind.SGD_UPDATE:
                v = n.inputs[0]
                if self.in_place:
                    self.t[nid] = self.t[v]
                else:
                    d = self.dims(nid)
                    self.t[nid] = self._new(d, 0, kind=self.t[v].kind)
                continue
            d = self.dims(nid)
            if n.kind in (OpKind.GRAD_CONV2D_W,):
                self.t[nid] = self._new(d, 0, kind="kkio")
                continue
            if n.kind is OpKind.ALL_REDUCE_SUM and len(n.inputs) == 1:
                raise EvalError(f"rank-local AllReduceSum {nid!r} must feed an SgdUpdate")
            self.t[nid] = self._new(d, self.pad.get(nid, 0))
        # aliases for fused/virtual producers
        for nid, (zb, r) in self.fwd_fuse.items():
            if r is not None:
                self.t[zb] = self.t[r]  # mask source: relu(x) > 0  <=>  x > 0

    # ---------------------------------------------------------------- lowering
    def _emit(self, name, fn, args, what="", keep=None, alg_bytes=0):
        self.steps.append(Step(name, fn, tuple(args), what, keep or [], int(alg_bytes)))

    @staticmethod
    def _nbytes(*tensors) -> int:
        """fp32 bytes of the logical elements of `tensors` (halo and lane padding excluded)."""
        return sum(4 * int(np.prod(t.dims)) for t in tensors if t is not None)

    def _gemm(self, name, M, Nn, K, a, b, out: Tensor, bias=None, relu=False, mask: Tensor | None = None,
              halo=(0, 0, 0), splits=0, to_updates=False, mbits_out=None, mbits_in=None, mask_fallback=None):
        from .kernels import GemmCall

        d = N.wap_gemm_desc_t()
        d.M, d.N, d.K = M, Nn, K
        d.a, d.b = a, b
        d.c = out.ptr
        d.ldc = out.ld
        d.bias = bias.ptr if bias is not None else None
        d.relu = 1 if relu else 0
        d.mask = mask.ptr if mask is not None else None
        d.ldm = mask.ld if mask is not None else 0
        d.halo_pad, d.halo_h, d.halo_w = halo
        d.precision = self.precision
        d.splits = splits
        # mask bits need the non-split epilogue: GEMMs whose automatic plan would
        # split K (small M, long K; splitting also keeps their fp32 sums short) keep
        # the float mask, and a producer that would split publishes no bits
        if (mbits_out is not None or mbits_in is not None) and self.L.wap_gemm_workspace_bytes(C.byref(d)) > 0:
            if mbits_out is not None:
                self.mask_bits.pop(name_out_of(self, mbits_out), None)
            mbits_out = None
            if mbits_in is not None:
                d.mask = mask_fallback.ptr if mask_fallback is not None else None
                d.ldm = mask_fallback.ld if mask_fallback is not None else 0
            mbits_in = None
        if mbits_out is not None:
            d.mbits_out, d.mbits_out_ld = mbits_out.data_ptr(), mbits_out.ld_words
        if mbits_in is not None:
            d.mbits_in, d.mbits_in_ld = mbits_in.data_ptr(), mbits_in.ld_words
        call = GemmCall(d, device=self.device)
        step = _GemmStep(name, call)
        step.desc = d
        from .workloads import node_flops

        nid = name[:-5] if name.endswith("/dcol") else name
        # algorithmic FLOPs by WAP's counting rule (workloads.py:84-117): no halo rows, no padding lanes
        step.alg_flops = node_flops(self.g, nid) if nid in self.g.nodes else 2 * M * Nn * K
        step.shape = (M, Nn, K)
        (self.update_steps if to_updates else self.steps).append(step)
        return call

    def _operand(self, t: Tensor, mn_major: bool, inner: int | None = None, tap_period=0, offsets=(0,)):
        return N.operand(t.ptr, inner=inner if inner is not None else t.dims[-1], outer=t.rows, ld=t.ld,
                         mn_major=mn_major, tap_period=tap_period, offsets=offsets)

    def _lower(self) -> None:
        L = self.L
        self.step_end: dict[str, int] = {}  # node id -> number of steps emitted once it is lowered
        for nid in self.order:
            self._lower_node(nid)
            self.step_end[nid] = len(self.steps)
        if self.autotune:
            self._autotune_gemms()
        self._parallelize_weight_grads()
        self._schedule_collectives()
        self._fuse_updates()
        self.steps.extend(self.update_steps)
        self.update_steps = []

    def _parallelize_weight_grads(self) -> None:
        """Training (in-place) programs: weight and bias gradients (GradConv2DW,
        GradMatMulW, GradBias) depend only on forward activations and the layer's
        upstream gradient, and feed only the update / allreduce. Issue them on a
        second stream forked at their position, so they overlap the data-gradient
        chain (dgrad of the same layer and everything below it); a join before the
        updates restores the order. Captured CUDA graphs keep the two branches."""
        self.par_stream = None
        if not self.in_place:
            return
        kinds = (OpKind.GRAD_CONV2D_W, OpKind.GRAD_MATMUL_W, OpKind.GRAD_BIAS)
        side = None
        for i, st in enumerate(self.steps):
            base = st.name.split("/")[0]  # a wgrad's companion steps (s2d fold) follow it
            if base in self.g.nodes and self.kind(base) in kinds:
                if side is None:
                    side = self.torch.cuda.Stream(device=self.device)
                self.steps[i] = _ParallelStep(st, side, self.torch)
        if side is not None:
            self.par_stream = side
            self.steps.append(_JoinParallel(side, self.torch))

    def _lower_node(self, nid: str) -> None:
        """Lower one graph node to its launch step(s)."""
        L = self.L
        n = self.node(nid)
        k = n.kind
        if k in (OpKind.INPUT, OpKind.VARIABLE):
            return
        if k is OpKind.CONV2D:
            self._lower_conv(n)
        elif k is OpKind.MATMUL:
            self._lower_matmul(n)
        elif k is OpKind.BIAS_ADD:
            if self.node(n.inputs[0]).id in self.fwd_fuse:
                return  # fused into the GEMM epilogue
            self._elementwise(0, n.inputs[0], None, n.inputs[1], nid)
        elif k is OpKind.RELU:
            if n.inputs[0] in self.mask_alias and self.mask_alias[n.inputs[0]] == nid:
                return  # fused
            self._elementwise(1, n.inputs[0], None, None, nid)
        elif k is OpKind.GRAD_RELU:
            if nid in self.bwd_mask.values():
                return  # written by the fused producer
            self._elementwise(3, n.inputs[1], self.mask_src(n.inputs[0]), None, nid)
        elif k in (OpKind.SOFTMAX_XENT_LOSS, OpKind.GRAD_SOFTMAX_XENT):
            self._lower_xent(n)
        elif k is OpKind.GRAD_BIAS:
            self._lower_bias_grad(n)
        elif k is OpKind.GRAD_MATMUL_W:
            self._lower_matmul_w(n)
        elif k is OpKind.GRAD_MATMUL_X:
            self._lower_matmul_x(n)
        elif k is OpKind.GRAD_CONV2D_W:
            self._lower_conv_w(n)
        elif k is OpKind.GRAD_CONV2D_X:
            self._lower_conv_x(n)
        elif k is OpKind.MAX_POOL:
            self._lower_pool(n)
        elif k is OpKind.GRAD_MAX_POOL:
            self._lower_pool_grad(n)
        elif k is OpKind.LRN:
            self._lower_lrn(n)
        elif k is OpKind.GRAD_LRN:
            self._lower_lrn_grad(n)
        elif k in (OpKind.ADD_N,):
            self._lower_add_n(n)
        elif k is OpKind.ALL_REDUCE_SUM:
            self._lower_allreduce(n)
        elif k is OpKind.SPLIT:
            pass  # resolved by consumers (see _in)
        elif k is OpKind.CONCAT:
            self._lower_concat(n)
        elif k is OpKind.SGD_UPDATE:
            self._lower_sgd(n)
        else:
            raise EvalError(f"no GPU rule for kind {k.value}")

    def _autotune_gemms(self, reps: int = 3) -> None:
        """Per-GEMM launch configuration: one CTA vs a CTA pair (cta_group::2), halo
        window on/off, BN = 128 vs wide tiles, explicit K splits for FC GEMMs.

        Results never depend on the run (plan_cache.py): a GEMM whose descriptor is
        in the committed plan file takes that configuration without timing; otherwise
        only candidates with the automatic plan's numerics signature (same K split
        and MMA pairing, hence the same accumulation order per element) are timed.
        WAP_AUTOTUNE_FREE=1 lifts the restriction (tools/tune_plans.py uses it to
        write the plan file). Buffers are already allocated; timings are
        data-independent."""
        from . import plan_cache
        from .kernels import GemmCall

        torch = self.torch
        stream = torch.cuda.current_stream(self.device)
        s = N.stream_ptr()
        free = os.environ.get("WAP_AUTOTUNE_FREE") == "1"
        reps = int(os.environ.get("WAP_AUTOTUNE_REPS", reps))  # tools/tune_plans.py times longer
        self.tuned_plans: dict[str, dict] = {}
        for st in self.steps + self.update_steps:
            if not isinstance(st, _GemmStep):
                continue
            key = plan_cache.key(st.desc)
            pinned = None if free else plan_cache.lookup(st.desc)
            if pinned is not None:
                d = type(st.desc).from_buffer_copy(st.desc)
                d.cluster, d.window, d.block_n = pinned["cluster"], pinned["window"], pinned["block_n"]
                d.splits = pinned["splits"]
                d.workspace, d.workspace_bytes = None, 0
                st.call = GemmCall(d, device=self.device)
                st.tuned_ms, st.plan_src = None, "plan file"
                self.tuned_plans[key] = dict(pinned)
                continue
            small_m = st.desc.M <= 128
            if small_m and os.environ.get("WAP_AUTOTUNE_FC", "1") == "0":
                continue
            sig = st.call.numerics()
            best, best_ms, best_choice = st.call, None, None
            a = st.desc.a
            windows = (0, -1) if (self.precision == 3 and not a.mn_major and a.ntaps > 1) else (0,)
            # BN = 128 keeps two TMEM accumulators in 3xTF32 (epilogue overlaps the next tile),
            # wider tiles halve B traffic: measure both where N allows
            bns = (0, 128) if (self.precision == 3 and st.desc.N >= 192) else (0,)
            # explicit split-K against wave quantization (WAP_AUTOTUNE_SPLITK=1): a GEMM of
            # only a few waves of output tiles (e.g. 13x13 convs: 98 CTA-pair tiles on 74
            # pairs) also tries 2-4 K slabs. Off by default: measured on B200 (r01), no
            # AlexNet / VGG-16 GEMM got faster (slab traffic + reduce > the tail wave)
            few_waves = (-(-st.desc.M // 128)) * (-(-st.desc.N // 256)) < 4 * 148
            auto_split = self.L.wap_gemm_workspace_bytes(C.byref(st.desc)) > 0
            k_chunks = -(-st.desc.K // 32)
            splits_opts = (0,) + tuple(x for x in (2, 3, 4) if few_waves and not auto_split
                                       and st.desc.splits == 0 and k_chunks >= 16 * x
                                       and os.environ.get("WAP_AUTOTUNE_SPLITK", "0") == "1")
            if small_m:
                # FC layers (M = batch <= 128): a handful of output tiles, so the K split
                # sets the grid; the automatic plan (<= one wave) vs ~2-4 waves of slabs
                # (M x N slabs are small: e.g. 19 MB at fc6 x 9). Measured r01: BN = 128
                # wins on every AlexNet FC GEMM (fc8 0.031 -> 0.024 ms), 9 slabs on fc6/fc7
                splits_opts = (0,) + tuple(x for x in (9, 18) if k_chunks >= 8 * x)
            for cluster, window, bn, sp in [(c, w, b, x) for c in ((1,) if small_m else (1, 2))
                                            for w in windows for b in bns for x in splits_opts]:
                d = type(st.desc).from_buffer_copy(st.desc)
                d.cluster = cluster
                d.window = window
                d.block_n = bn
                d.splits = sp if sp else st.desc.splits
                d.workspace, d.workspace_bytes = None, 0
                try:
                    call = GemmCall(d, device=self.device)
                except Exception:
                    continue
                if not free and call.numerics() != sig:
                    continue
                N.check(self.L.wap_gemm_plan_run(call._plan, s), "autotune warm-up")
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(reps):
                    N.check(self.L.wap_gemm_plan_run(call._plan, s), "autotune")
                e1.record(stream)
                e1.synchronize()
                ms = e0.elapsed_time(e1) / reps
                if os.environ.get("WAP_AUTOTUNE_LOG"):
                    print(f"autotune {st.name} M={d.M} N={d.N} K={d.K} cluster={cluster} window={window} bn={bn} "
                          f"splits={sp} sig={call.numerics()} {ms:.4f} ms", flush=True)
                if best_ms is None or ms < best_ms:
                    best, best_ms = call, ms
                    best_choice = {"cluster": cluster, "window": window, "block_n": bn, "splits": d.splits}
            st.call = best
            st.tuned_ms = best_ms
            st.plan_src = "autotune (free)" if free else "autotune (numerics-preserving)"
            if best_choice is not None:
                self.tuned_plans[key] = best_choice

    def _schedule_collectives(self) -> None:
        """Bucket the rank-local gradient allreduces and overlap them with backward.

        Gradients live in one arena in readiness order, so a bucket is a
        contiguous slice. Each bucket's allreduce is issued on a side stream as
        soon as its last gradient is produced (event on the compute stream), while
        the remaining backward kernels keep running; a join step makes the
        compute stream wait for the side stream before the SGD update."""
        if not self._collectives:
            return
        items = sorted(self._collectives, key=lambda x: x[0])
        base = self.grad_arena.data_ptr()
        buckets: list[list] = []
        for ready, nid, t in items:
            lo = (t.ptr - base) // 4
            hi = lo + t.numel_storage()
            if buckets:
                b = buckets[-1]
                adjacent = lo == b[2] or hi == b[1]
                if adjacent and (max(hi, b[2]) - min(lo, b[1])) * 4 <= self.bucket_bytes:
                    b[0] = max(b[0], ready)
                    b[1], b[2] = min(lo, b[1]), max(hi, b[2])
                    b[3].append(nid)
                    continue
            buckets.append([ready, lo, hi, [nid]])
        side = self.torch.cuda.Stream(device=self.device)
        self.comm_stream = side
        inserts: dict[int, list] = {}
        if self.fused is not None:
            self._schedule_fused(buckets, side, inserts)
            return
        # SGD of a bucket also runs on the comm stream, right behind its allreduce,
        # once the last backward kernel reading those weights (GradMatMulX /
        # GradConv2DX) has been issued: the update overlaps the rest of backward.
        lr = self._uniform_lr()
        self.bucket_sgd = self.in_place and lr is not None
        var_of_slot = {self.arena_off[v]: v for v in self.arena_off}
        for ready, lo, hi, ids in buckets:
            buf = self.grad_arena[lo:hi]
            inserts.setdefault(ready, []).append(
                _BucketStep("+".join(ids), self.collective, buf, side, self.torch, self.par_stream,
                            self.collective_capturable))
            if self.bucket_sgd:
                vars_in = [v for o, v in var_of_slot.items() if lo <= o < hi]
                readers = [self.step_end[u] for v in vars_in for u in self.users[v]
                           if self.kind(u) is not OpKind.SGD_UPDATE]
                at = max([ready] + readers)
                sgd = Step(f"sgd[{lo}:{hi}]", self.L.wap_sgd,
                           (self.var_arena[lo:hi].data_ptr(), buf.data_ptr(), C.c_float(lr),
                            self.var_arena[lo:hi].data_ptr(), hi - lo), "SgdUpdate (bucket)",
                           alg_bytes=12 * (hi - lo))
                inserts.setdefault(at, []).append(_SideStep(sgd, side, self.torch))
        new_steps = []
        for i, st in enumerate(self.steps):
            new_steps.extend(inserts.get(i, []))
            new_steps.append(st)
        new_steps.extend(inserts.get(len(self.steps), []))
        new_steps.append(_JoinStep(side, self.torch))
        self.steps = new_steps
        self.buckets = [(lo * 4, hi * 4, ids) for _, lo, hi, ids in buckets]

    def _schedule_fused(self, buckets, side, inserts) -> None:
        """One wap_allreduce_sgd per bucket on the comm stream: reduce-scatter +
        SGD + all-gather over peer memory (csrc/allreduce.cu). It writes every
        rank's copy of the bucket's variables, so it goes where the bucket SGD
        would: behind the bucket's last gradient AND the last backward kernel
        reading those weights; the kernel's entry barrier extends that to all ranks."""
        from . import _native as N

        lr = self._uniform_lr()
        if lr is None:
            raise EvalError("the fused allreduce + SGD needs one learning rate for every variable")
        if len(buckets) > N.AR_SLOTS:
            raise EvalError(f"{len(buckets)} buckets exceed the {N.AR_SLOTS} barrier slots; raise bucket_bytes")
        var_of_slot = {self.arena_off[v]: v for v in self.arena_off}
        for slot, (ready, lo, hi, ids) in enumerate(buckets):
            vars_in = [v for o, v in var_of_slot.items() if lo <= o < hi]
            readers = [self.step_end[u] for v in vars_in for u in self.users[v]
                       if self.kind(u) is not OpKind.SGD_UPDATE]
            at = max([ready] + readers)
            inserts.setdefault(at, []).append(
                _FusedBucketStep("+".join(ids), self.fused, lo, hi - lo, lr, slot, side, self.torch, self.par_stream))
        new_steps = []
        for i, st in enumerate(self.steps):
            new_steps.extend(inserts.get(i, []))
            new_steps.append(st)
        new_steps.extend(inserts.get(len(self.steps), []))
        new_steps.append(_JoinFused(side, self.torch))
        self.steps = new_steps
        self.bucket_sgd = True
        self.buckets = [(lo * 4, hi * 4, ids) for _, lo, hi, ids in buckets]

    def _uniform_lr(self):
        lrs = {float(self.node(u).attr("learning_rate")) for u in self.updates}
        return lrs.pop() if len(lrs) == 1 else None

    def _fuse_updates(self) -> None:
        """In-place training: one SGD launch over the whole variable arena when all
        updates share a learning rate (variables without an update have a zero
        gradient slot, so w - lr*0 leaves them unchanged). With cross-rank
        buckets the updates already ran per bucket on the comm stream."""
        if not self.in_place or not self.update_steps:
            return
        if getattr(self, "bucket_sgd", False) and self.buckets:
            covered = sum(hi - lo for lo, hi, _ in self.buckets) // 4
            upd_vars = {self.node(u).inputs[0] for u in self.updates}
            if covered and all(any(lo // 4 <= self.arena_off[v] < hi // 4 for lo, hi, _ in self.buckets)
                               for v in upd_vars):
                self.update_steps = []
                return
        lr = self._uniform_lr()
        if lr is None or any(not isinstance(s, Step) for s in self.update_steps):
            return
        self.update_steps = [Step("sgd(arena)", self.L.wap_sgd,
                                  (self.var_arena.data_ptr(), self.grad_arena.data_ptr(), C.c_float(lr),
                                   self.var_arena.data_ptr(), self.arena_numel), "SgdUpdate (fused arena)",
                                  alg_bytes=12 * self.arena_numel)]

    # -- tensor access ---------------------------------------------------------
    def _in(self, consumer: Node, nid: str) -> Tensor:
        """Materialized input tensor; Split parts become row views."""
        n = self.node(nid)
        if n.kind is OpKind.SPLIT:
            src = self._in(n, n.inputs[0])
            parts = n.attr("parts")
            if n.attr("axis") != 0:
                raise EvalError("Split is supported along the batch axis (0) only")
            dev = consumer.device
            if dev is None or not 0 <= dev < parts:
                raise EvalError(f"node {consumer.id!r} consumes split {nid!r} but has no part device")
            per = src.numel_storage() // parts
            dims = (src.dims[0] // parts,) + tuple(src.dims[1:])
            kind = src.kind
            return Tensor(dims, src.pad, src.ld, src.buf[dev * per:(dev + 1) * per], kind)
        if nid not in self.t:
            raise EvalError(f"tensor {nid!r} was not materialized")
        return self.t[nid]

    def _out(self, nid: str) -> Tensor:
        return self.t[nid]

    # -- forward -------------------------------------------------------------
    def _lower_conv(self, n: Node) -> None:
        x = self._in(n, n.inputs[0])
        w = self._in(n, n.inputs[1])
        kk, _, ci, co = w.dims
        s, p = conv_geometry(n, kk)
        zb, r = self.fwd_fuse.get(n.id, (None, None))
        out_id = self.fused_out(n.id)
        y = self._out(out_id)
        bias = self._in(self.node(zb), self.node(zb).inputs[1]) if zb is not None else None
        relu = r is not None
        b, ho, wo, _ = self.dims(n.id)
        if self.strategy[n.id] == "direct":
            if x.ld != 4:
                raise EvalError(f"{n.id!r}: direct conv needs the input packed as one float4 per pixel")
            bits = self._bits_alloc(out_id) if out_id in self.bits_src else None
            self._emit(n.id, self.L.wap_conv_direct,
                       (x.ptr, x.layout(), w.ptr, kk, p, w.ld, bias.ptr if bias is not None else None,
                        1 if relu else 0, y.ptr, y.layout(), bits.data_ptr() if bits is not None else None,
                        bits.ld_words if bits is not None else 0), "Conv2D (direct, CUDA cores)",
                       alg_bytes=self._nbytes(x, y), keep=[bits] if bits is not None else None)
            return
        if self.strategy[n.id] == "s2d":
            s_, p_, ks, hs, ws, ldc, halo = self._s2d_geometry(n)
            if y.pad != halo:
                raise EvalError(f"{n.id!r}: s2d output needs a trailing halo of {halo}, layout has {y.pad}")
            torch = self.torch
            rows = b * hs * ws
            xs = torch.zeros(rows * ldc, dtype=torch.float32, device=self.device)
            wsb = torch.zeros(ks * ks * ldc * w.ld, dtype=torch.float32, device=self.device)
            self.t[f"{n.id}::s2d"] = Tensor((rows, ldc), 0, ldc, xs, "mat")
            self._emit(n.id + "/s2d", self.L.wap_s2d_input, (x.ptr, x.layout(), s_, p_, hs, ws, xs.data_ptr(), ldc),
                       "space-to-depth", keep=[xs], alg_bytes=self._nbytes(x) + 4 * rows * ldc)
            self._emit(n.id + "/s2d_w", self.L.wap_s2d_weight,
                       (w.ptr, wsb.data_ptr(), kk, ci, co, w.ld, s_, ldc, w.ld, 0), "space-to-depth weights",
                       keep=[wsb], alg_bytes=4 * (kk * kk * ci + ks * ks * ldc) * co)
            a = N.operand(xs.data_ptr(), inner=ldc, outer=rows, ld=ldc, mn_major=False, tap_period=ldc,
                          offsets=tuple(u * ws + v for u in range(ks) for v in range(ks)))
            bo = N.operand(wsb.data_ptr(), inner=co, outer=ks * ks * ldc, ld=w.ld, mn_major=True)
            self._gemm(n.id, rows, co, ks * ks * ldc, a, bo, y, bias=bias, relu=relu, halo=(halo, ho, wo),
                       mbits_out=self._bits_out(out_id))
            return
        if self.strategy[n.id] == "shifted":
            P = x.pad
            assert y.pad == P, (n.id, y.pad, P)
            wp = x.dims[2] + P
            shifts = [(u - p) * wp + (v - p) for u in range(kk) for v in range(kk)]
            a = self._operand(x, False, inner=ci, tap_period=ci, offsets=tuple(shifts))
            bo = N.operand(w.ptr, inner=co, outer=kk * kk * ci, ld=w.ld, mn_major=True)
            self._gemm(n.id, x.rows, co, kk * kk * ci, a, bo, y, bias=bias, relu=relu, halo=(P, ho, wo),
                       mbits_out=self._bits_out(out_id))
        else:
            P = y.pad
            K = kk * kk * ci
            ldcol = _ceil4(K)
            rows = b * (ho + P) * (wo + P)
            col = self.torch.empty(rows * ldcol, dtype=self.torch.float32, device=self.device)
            self.t[f"{n.id}::col"] = Tensor((rows, K), 0, ldcol, col, "mat")
            self._emit(n.id + "/im2col", self.L.wap_im2col,
                       (x.ptr, x.layout(), kk, s, p, ho, wo, P, col.data_ptr(), ldcol), "im2col",
                       alg_bytes=self._nbytes(x) + 4 * b * ho * wo * K)
            ct = self.t[f"{n.id}::col"]
            a = self._operand(ct, False, inner=K)
            bo = N.operand(w.ptr, inner=co, outer=K, ld=w.ld, mn_major=True)
            self._gemm(n.id, rows, co, K, a, bo, y, bias=bias, relu=relu, halo=(P, ho, wo) if P else (0, 0, 0),
                       mbits_out=self._bits_out(out_id))

    def _lower_matmul(self, n: Node) -> None:
        x = self._in(n, n.inputs[0])
        w = self._in(n, n.inputs[1])
        i, o = w.dims
        zb, r = self.fwd_fuse.get(n.id, (None, None))
        y = self._out(self.fused_out(n.id))
        bias = self._in(self.node(zb), self.node(zb).inputs[1]) if zb is not None else None
        rows = x.dims[0]
        ld = x.ld if x.kind == "mat" else int(np.prod(x.dims[1:]))
        a = N.operand(x.ptr, inner=i, outer=rows, ld=ld, mn_major=False)
        bo = N.operand(w.ptr, inner=o, outer=i, ld=w.ld, mn_major=True)
        self._gemm(n.id, rows, o, i, a, bo, y, bias=bias, relu=r is not None)

    def _elementwise(self, op, x_id, aux_id, bias_id, out_id) -> None:
        node = self.node(out_id)
        x = self._in(node, x_id)
        aux = self._in(node, aux_id) if aux_id is not None else None
        bias = self._in(node, bias_id) if bias_id is not None else None
        y = self._out(out_id)
        xl, yl = self._as_compat(x, y)
        al = self._as_compat(aux, y)[0] if aux is not None else N.wap_layout_t()
        self._emit(out_id, self.L.wap_elementwise,
                   (op, x.ptr, xl, aux.ptr if aux is not None else None, al,
                    bias.ptr if bias is not None else None, y.ptr, yl), f"elementwise[{op}] {out_id}",
                   alg_bytes=self._nbytes(x, aux, bias, y))

    @staticmethod
    def _as_compat(a: Tensor, b: Tensor):
        """Layouts of a and b viewed with the same logical dims (flatten-aware)."""
        la, lb = a.layout(), b.layout()
        if (la.B, la.H, la.W, la.C) != (lb.B, lb.H, lb.W, lb.C):
            if a.kind == "mat" and b.kind == "nhwc" and b.pad == 0 and b.ld == b.dims[-1]:
                lb2 = N.wap_layout_t(la.B, la.H, la.W, la.C, 0, la.ld)
                lb2.ld = int(np.prod(b.dims[1:]))
                return la, lb2
            if b.kind == "mat" and a.kind == "nhwc" and a.pad == 0 and a.ld == a.dims[-1]:
                la2 = N.wap_layout_t(lb.B, lb.H, lb.W, lb.C, 0, int(np.prod(a.dims[1:])))
                return la2, lb
            raise EvalError(f"incompatible layouts {a.dims} vs {b.dims}")
        return la, lb

    def _lower_xent(self, n: Node) -> None:
        key = tuple(n.inputs)
        pair = self.xent[key]
        first = pair.get("loss") or pair.get("grad")
        if pair.get("loss") and pair.get("grad"):
            # emit once, at the first of the two in topological order
            pos = {x: i for i, x in enumerate(self.order)}
            first = min(pair.values(), key=lambda x: pos[x])
        if n.id != first:
            return
        z = self._in(n, n.inputs[0])
        y = self._in(n, n.inputs[1])
        rows, cols = z.dims
        loss = self.t[pair["loss"]] if "loss" in pair else self._new((1,))
        if "grad" in pair:
            dz = self.t[pair["grad"]]
            denom = self.node(pair["grad"]).attr("denominator", rows)
        else:
            dz = self._new((rows, cols))
            denom = rows
        work = self.torch.empty(rows, dtype=self.torch.float32, device=self.device)
        self._emit(n.id + "/xent", self.L.wap_xent_fwd_bwd,
                   (z.ptr, z.ld, y.ptr, y.ld, rows, cols, C.c_float(float(denom)), loss.ptr, dz.ptr, dz.ld,
                    work.data_ptr()), "softmax-xent", keep=[work, loss, dz], alg_bytes=12 * rows * cols)

    def _lower_bias_grad(self, n: Node) -> None:
        dy = self._in(n, n.inputs[0])
        db = self._out(n.id)
        lay = dy.layout()
        wf = self.L.wap_bias_grad_work_floats(lay)
        work = self.torch.empty(max(wf, 1), dtype=self.torch.float32, device=self.device)
        self._emit(n.id, self.L.wap_bias_grad, (dy.ptr, lay, db.ptr, work.data_ptr()), "GradBias", keep=[work],
                   alg_bytes=self._nbytes(dy, db))

    # -- backward GEMMs ------------------------------------------------------
    def _lower_matmul_w(self, n: Node) -> None:
        x = self._in(n, n.inputs[0])
        dy = self._in(n, n.inputs[1])
        dw = self._out(n.id)
        i, o = self.dims(n.id)
        rows = x.dims[0]
        ldx = x.ld if x.kind == "mat" else int(np.prod(x.dims[1:]))
        a = N.operand(x.ptr, inner=i, outer=rows, ld=ldx, mn_major=True)
        bo = N.operand(dy.ptr, inner=o, outer=rows, ld=dy.ld, mn_major=True)
        self._gemm(n.id, i, o, rows, a, bo, dw)

    def _lower_matmul_x(self, n: Node) -> None:
        dy = self._in(n, n.inputs[0])
        w = self._in(n, n.inputs[1])
        i, o = w.dims
        gr = self.bwd_mask.get(n.id)
        out = self._out(gr if gr else n.id)
        mask = self._in(self.node(gr), self.mask_src(self.node(gr).inputs[0])) if gr else None
        rows = dy.dims[0]
        a = N.operand(dy.ptr, inner=o, outer=rows, ld=dy.ld, mn_major=False)
        bo = N.operand(w.ptr, inner=o, outer=i, ld=w.ld, mn_major=False)
        flat_out = out if out.kind == "mat" else Tensor((rows, i), 0, int(np.prod(out.dims[1:])), out.buf, "mat")
        flat_mask = None
        if mask is not None:
            flat_mask = mask if mask.kind == "mat" else Tensor((rows, i), 0, int(np.prod(mask.dims[1:])), mask.buf,
                                                               "mat")
        self._gemm(n.id, rows, i, o, a, bo, flat_out, mask=flat_mask)

    def _lower_conv_x(self, n: Node) -> None:
        dy = self._in(n, n.inputs[0])
        w = self._in(n, n.inputs[1])
        conv = self._conv_of_weight(n.inputs[1])
        cn = self.node(conv)
        kk, _, ci, co = w.dims
        s, p = conv_geometry(cn, kk)
        gr = self.bwd_mask.get(n.id)
        out = self._out(gr if gr else n.id)
        mask = self._in(self.node(gr), self.mask_src(self.node(gr).inputs[0])) if gr else None
        b, ho, wo, _ = self.dims(conv)
        if self.strategy[conv] == "shifted":
            P = dy.pad
            assert out.pad == P and (mask is None or (mask.pad == P and mask.ld == out.ld))
            wp = out.dims[2] + P
            shifts = [(u - p) * wp + (v - p) for u in range(kk) for v in range(kk)]
            a = self._operand(dy, False, inner=co, tap_period=co, offsets=tuple(-s_ for s_ in shifts))
            bo = N.operand(w.ptr, inner=co, outer=kk * kk * ci, ld=w.ld, mn_major=False, tap_period=co,
                           offsets=tuple(t * ci for t in range(kk * kk)))
            bits = self.mask_bits.get(self.mask_src(self.node(gr).inputs[0])) if gr else None
            self._gemm(n.id, dy.rows, ci, kk * kk * co, a, bo, out, mask=None if bits is not None else mask,
                       halo=(P, out.dims[1], out.dims[2]), mbits_in=bits, mask_fallback=mask)
        else:
            P = dy.pad
            K = kk * kk * ci
            ldcol = _ceil4(K)
            rows = dy.rows
            dcol = self.torch.empty(rows * ldcol, dtype=self.torch.float32, device=self.device)
            dct = Tensor((rows, K), 0, ldcol, dcol, "mat")
            a = self._operand(dy, False, inner=co)
            bo = N.operand(w.ptr, inner=co, outer=K, ld=w.ld, mn_major=False)
            self._gemm(n.id + "/dcol", rows, K, co, a, bo, dct)
            ml = mask.layout() if mask is not None else N.wap_layout_t()
            self._emit(n.id + "/col2im", self.L.wap_col2im,
                       (dcol.data_ptr(), ldcol, kk, s, p, ho, wo, P, out.ptr, out.layout(),
                        mask.ptr if mask is not None else None, ml), "col2im", keep=[dcol],
                       alg_bytes=4 * b * ho * wo * K + self._nbytes(out, mask))

    def _lower_conv_w(self, n: Node) -> None:
        x = self._in(n, n.inputs[0])
        dy = self._in(n, n.inputs[1])
        dw = self._out(n.id)
        conv = self._conv_of_wgrad(n)
        kk, _, ci, co = self.dims(n.id)
        if self.strategy[conv] == "s2d":
            s_, p_, ks, hs, ws, ldc, halo = self._s2d_geometry(self.node(conv))
            xs = self.t[f"{conv}::s2d"]
            assert dy.rows == xs.rows and dy.pad == halo, (n.id, dy.rows, xs.rows)
            dws = self.torch.zeros(ks * ks * ldc * dw.ld, dtype=self.torch.float32, device=self.device)
            a = N.operand(xs.ptr, inner=ldc, outer=xs.rows, ld=ldc, mn_major=True, tap_period=ldc,
                          offsets=tuple(u * ws + v for u in range(ks) for v in range(ks)))
            bo = N.operand(dy.ptr, inner=co, outer=dy.rows, ld=dy.ld, mn_major=True)
            self._gemm(n.id, ks * ks * ldc, co, xs.rows, a, bo, Tensor((ks * ks * ldc, co), 0, dw.ld, dws, "mat"))
            self._emit(n.id + "/fold", self.L.wap_s2d_weight,
                       (dws.data_ptr(), dw.ptr, kk, ci, co, dw.ld, s_, ldc, dw.ld, 1), "s2d weight-gradient fold",
                       keep=[dws], alg_bytes=4 * (kk * kk * ci + kk * kk * ci) * co)
            return
        if self.strategy[conv] == "shifted":
            P = x.pad
            assert dy.pad == P
            p = kk // 2
            wp = x.dims[2] + P
            shifts = [(u - p) * wp + (v - p) for u in range(kk) for v in range(kk)]
            a = N.operand(x.ptr, inner=ci, outer=x.rows, ld=x.ld, mn_major=True, tap_period=ci,
                          offsets=tuple(shifts))
            bo = N.operand(dy.ptr, inner=co, outer=dy.rows, ld=dy.ld, mn_major=True)
            self._gemm(n.id, kk * kk * ci, co, x.rows, a, bo, dw)
        else:
            if self.strategy[conv] == "direct":
                cn = self.node(conv)
                x_in = self._in(cn, cn.inputs[0])
                s_, p_ = conv_geometry(cn, kk)
                _, ho, wo, _ = self.dims(conv)
                if (kk == 3 and s_ == 1 and p_ == 1 and ci == 3 and x_in.ld == 4 and (ho, wo) == tuple(x_in.dims[1:3])
                        and os.environ.get("WAP_WGRAD_DIRECT", "0") == "1"):
                    # 3-channel first layer: CUDA-core direct weight gradient, no im2col and no
                    # M = 27 GEMM (csrc/ops.cu wgrad_direct_3x3_kernel). Opt-in: measured r02 on
                    # VGG-16 conv1_1, 0.47 ms vs 0.34 ms for im2col + the tcgen05 GEMM
                    work = self.torch.empty(int(self.L.wap_conv_wgrad_direct_work_floats(dy.layout())),
                                            dtype=self.torch.float32, device=self.device)
                    self._emit(n.id, self.L.wap_conv_wgrad_direct,
                               (x_in.ptr, x_in.layout(), dy.ptr, dy.layout(), kk, p_, dw.ptr, dw.ld,
                                work.data_ptr()), "direct weight gradient (3-channel first layer)",
                               keep=[work], alg_bytes=self._nbytes(x_in, dy, dw))
                    return
                # the forward never built columns: im2col here, on the weight-gradient stream
                K = kk * kk * ci
                ldcol = _ceil4(K)
                colb = self.torch.empty(dy.rows * ldcol, dtype=self.torch.float32, device=self.device)
                self.t[f"{conv}::col"] = Tensor((dy.rows, K), 0, ldcol, colb, "mat")
                self._emit(n.id + "/im2col", self.L.wap_im2col,
                           (x_in.ptr, x_in.layout(), kk, s_, p_, ho, wo, dy.pad, colb.data_ptr(), ldcol),
                           "im2col (weight gradient)", alg_bytes=self._nbytes(x_in) + 4 * dy.rows * K)
            col = self.t[f"{conv}::col"]
            K = kk * kk * ci
            assert col.rows == dy.rows, (n.id, col.rows, dy.rows)
            a = N.operand(col.ptr, inner=K, outer=col.rows, ld=col.ld, mn_major=True)
            bo = N.operand(dy.ptr, inner=co, outer=dy.rows, ld=dy.ld, mn_major=True)
            self._gemm(n.id, K, co, col.rows, a, bo, dw)

    # -- pooling / LRN -------------------------------------------------------
    def _lower_pool(self, n: Node) -> None:
        ln = self._lrn_pool.pop(n.id, None)
        if ln is not None:
            x = self._in(ln, ln.inputs[0])
            y = self._out(n.id)
            arg = self.torch.zeros(y.numel_storage(), dtype=self.torch.uint8, device=self.device)
            self.t[f"{n.id}::argmax"] = Tensor(y.dims, y.pad, y.ld, arg, "nhwc")
            a = ln.attrs
            self._emit(n.id, self.L.wap_lrn_maxpool_fwd,
                       (x.ptr, x.layout(), a["size"], C.c_float(a["alpha"]), C.c_float(a["beta"]),
                        C.c_float(a["bias"]), n.attr("window"), n.attr("stride"), y.ptr, y.layout(),
                        arg.data_ptr()), "LRN+MaxPool", keep=[arg],
                       alg_bytes=self._nbytes(x, y) + self._nbytes(y) // 4)
            return
        x = self._in(n, n.inputs[0])
        y = self._out(n.id)
        if x.ld != y.ld:
            raise EvalError("MaxPool needs equal channel strides")
        arg = self.torch.zeros(y.numel_storage(), dtype=self.torch.uint8, device=self.device)
        self.t[f"{n.id}::argmax"] = Tensor(y.dims, y.pad, y.ld, arg, "nhwc")
        flags = N.POOL_RELU_FUSED if n.id in self.pool_relu_fused else 0
        self._emit(n.id, self.L.wap_maxpool_fwd_ex,
                   (x.ptr, x.layout(), n.attr("window"), n.attr("stride"), y.ptr, y.layout(), arg.data_ptr(), flags),
                   "MaxPool", keep=[arg], alg_bytes=self._nbytes(x, y) + self._nbytes(y) // 4)

    def _lower_pool_grad(self, n: Node) -> None:
        x_id, dy_id = n.inputs
        pool = self.pool_of.get((x_id, n.attr("window"), n.attr("stride")))
        if pool is None:
            raise EvalError(f"{n.id!r}: no matching MaxPool forward for its argmax")
        arg = self.t[f"{pool}::argmax"]
        dy = self._in(n, dy_id)
        gr = self.bwd_mask.get(n.id)
        lrn = self._pool_lrn_fusable(n, gr, dy)
        if lrn is not None:
            # GradMaxPool -> GradLRN as one kernel (wap_maxpool_lrn_bwd), emitted at the GradLRN
            self._pool_lrn[lrn] = (arg, dy, n.attr("window"), n.attr("stride"))
            return
        out = self._out(gr if gr else n.id)
        mask = self._in(self.node(gr), self.mask_src(self.node(gr).inputs[0])) if gr else None
        if pool in self.pool_relu_fused:
            mask = None  # the forward argmax already encodes the GradReLU mask
        ml = mask.layout() if mask is not None else N.wap_layout_t()
        if dy.pad != arg.pad:
            raise EvalError("MaxPool gradient must share the pooled output layout")
        self._emit(n.id, self.L.wap_maxpool_bwd,
                   (arg.ptr, dy.ptr, dy.layout(), n.attr("window"), n.attr("stride"), out.ptr, out.layout(),
                    mask.ptr if mask is not None else None, ml), "GradMaxPool",
                   alg_bytes=self._nbytes(dy, out, mask) + self._nbytes(dy) // 4)

    def _lrn_pool_fusable(self, n: Node) -> str | None:
        """The MaxPool reading this LRN's output when the pair can run as one forward
        kernel: the LRN output is read by nothing else (GradMaxPool nodes only name it
        as the key of the pool's argmax), is not a graph output, LRN size 5 over
        C = 64 / 192 compact channels, window 2/3."""
        if os.environ.get("WAP_FUSE_LRN_POOL", "1") == "0" or n.id in self.g.outputs or n.attr("size") != 5:
            return None
        users = self.users.get(n.id, [])
        pools = [u for u in users if self.kind(u) is OpKind.MAX_POOL]
        if len(pools) != 1 or any(self.kind(u) not in (OpKind.MAX_POOL, OpKind.GRAD_MAX_POOL) for u in users):
            return None
        pn = self.node(pools[0])
        if pn.inputs[0] != n.id or pn.attr("window") not in (2, 3) or pn.id in self.pool_relu_fused:
            return None
        x, y = self.t.get(n.inputs[0]), self.t.get(n.id)
        py = self.t.get(pn.id)
        if x is None or y is None or py is None or x.kind != "nhwc" or x.dims[-1] not in (64, 192):
            return None
        if x.ld != x.dims[-1] or py.ld != x.ld:
            return None
        return pn.id

    def _lower_lrn(self, n: Node) -> None:
        pool = self._lrn_pool_fusable(n)
        if pool is not None:
            self._lrn_pool[pool] = n  # emitted by _lower_pool as wap_lrn_maxpool_fwd
            return
        x = self._in(n, n.inputs[0])
        y = self._out(n.id)
        a = n.attrs
        self._emit(n.id, self.L.wap_lrn_fwd,
                   (x.ptr, x.layout(), a["size"], C.c_float(a["alpha"]), C.c_float(a["beta"]), C.c_float(a["bias"]),
                    y.ptr, y.layout()), "LRN", alg_bytes=self._nbytes(x, y))

    def _pool_lrn_fusable(self, n: Node, gr, dy) -> str | None:
        """The GradLRN consuming this GradMaxPool's output when the pair can run fused:
        sole consumer, not a graph output, no GradReLU on the pool gradient, stride 2,
        window 2/3, LRN size 5 over C = 64 / 192 compact channels."""
        if os.environ.get("WAP_FUSE_POOL_LRN", "1") == "0" or gr or n.id in self.g.outputs:
            return None
        users = self.users.get(n.id, [])
        if len(users) != 1 or self.kind(users[0]) is not OpKind.GRAD_LRN:
            return None
        ln = self.node(users[0])
        if ln.inputs[1] != n.id or ln.inputs[0] == n.id or ln.attr("size") != 5:
            return None
        if n.attr("stride") != 2 or n.attr("window") not in (2, 3):
            return None
        x = self.t.get(ln.inputs[0])
        if x is None or x.kind != "nhwc" or x.dims[-1] not in (64, 192) or x.ld != x.dims[-1] or dy.ld != x.ld:
            return None
        return ln.id

    def _lower_lrn_grad(self, n: Node) -> None:
        x = self._in(n, n.inputs[0])
        gr = self.bwd_mask.get(n.id)
        out = self._out(gr if gr else n.id)
        mask = self._in(self.node(gr), self.mask_src(self.node(gr).inputs[0])) if gr else None
        ml = mask.layout() if mask is not None else N.wap_layout_t()
        a = n.attrs
        fused = self._pool_lrn.pop(n.id, None)
        if fused is not None and out.ld == x.ld and (mask is None or mask.ld == x.ld):
            arg, pdy, window, stride = fused
            self._emit(n.id, self.L.wap_maxpool_lrn_bwd,
                       (arg.ptr, pdy.ptr, pdy.layout(), window, stride, x.ptr, x.layout(), a["size"],
                        C.c_float(a["alpha"]), C.c_float(a["beta"]), C.c_float(a["bias"]), out.ptr, out.layout(),
                        mask.ptr if mask is not None else None, ml), "GradMaxPool+GradLRN",
                       alg_bytes=self._nbytes(pdy, x, out) + self._nbytes(pdy) // 4
                       + (0 if mask is None or mask.ptr == x.ptr else self._nbytes(mask)))
            return
        if fused is not None:
            raise EvalError(f"{n.id!r}: fused MaxPool+LRN backward needs compact channel layouts")
        dy = self._in(n, n.inputs[1])
        self._emit(n.id, self.L.wap_lrn_bwd,
                   (x.ptr, x.layout(), dy.ptr, dy.layout(), a["size"], C.c_float(a["alpha"]), C.c_float(a["beta"]),
                    C.c_float(a["bias"]), out.ptr, out.layout(), mask.ptr if mask is not None else None, ml),
                   "GradLRN", alg_bytes=self._nbytes(x, dy, out) + (0 if mask is None or mask.ptr == x.ptr
                                                                     else self._nbytes(mask)))

    # -- aggregation / update ------------------------------------------------
    def _lower_add_n(self, n: Node) -> None:
        ins = [self._in(n, i) for i in n.inputs]
        out = self._out(n.id)
        for t in ins:
            if t.numel_storage() != out.numel_storage() or t.ld != out.ld or t.pad != out.pad:
                raise EvalError(f"{n.id!r}: AddN operands must share one layout")
        # wap_add_n folds at most 16 sources left to right (interp.py:115-119): the first
        # launch takes ins[0:16], every later one the running sum plus the next 15 operands
        lo = 0
        while lo < len(ins):
            srcs = ins[0:16] if lo == 0 else [out] + ins[lo:lo + 15]
            arr = (C.c_void_p * len(srcs))(*[t.ptr for t in srcs])
            self._emit(f"{n.id}#{lo}", self.L.wap_add_n, (arr, len(srcs), out.layout(), out.ptr), "AddN",
                       keep=[arr])
            lo += len(srcs) - (0 if lo == 0 else 1)

    def _lower_allreduce(self, n: Node) -> None:
        if len(n.inputs) >= 2:  # all replicas in this process: left fold (interp.py:181-182)
            self._lower_add_n(n)
            return
        # rank-local view: the sum crosses processes. Recorded here, bucketed in
        # _schedule_collectives once every producer's position is known.
        src = self._in(n, n.inputs[0])
        if self.collective is not None or self.fused is not None:
            self._collectives.append((len(self.steps), n.id, src))

    def _lower_concat(self, n: Node) -> None:
        out = self._out(n.id)
        if n.attr("axis") != 0:
            raise EvalError("Concat is supported along the batch axis (0) only")
        per = out.numel_storage() // len(n.inputs)
        for k, i in enumerate(n.inputs):
            src = self._in(n, i)
            dst = Tensor(src.dims, out.pad, out.ld, out.buf[k * per:(k + 1) * per], out.kind)
            xl, yl = self._as_compat(src, dst)
            self._emit(f"{n.id}#{k}", self.L.wap_elementwise, (4, src.ptr, xl, None, N.wap_layout_t(), None,
                                                                dst.ptr, yl), "Concat copy")

    def _lower_sgd(self, n: Node) -> None:
        v = self._in(n, n.inputs[0])
        gsrc = self._in(n, n.inputs[1])
        out = self._out(n.id)
        lr = float(n.attr("learning_rate"))
        if gsrc.numel_storage() != v.numel_storage():
            raise EvalError(f"{n.id!r}: gradient layout does not match the variable")
        self.update_steps.append(Step(n.id, self.L.wap_sgd,
                                      (v.ptr, gsrc.ptr, C.c_float(lr), out.ptr, v.numel_storage()), "SgdUpdate"))

    # ------------------------------------------------------------- execution
    def run(self, stream=None) -> None:
        s = N.stream_ptr(stream)
        if self.graph_exec is not None:
            self.graph_exec.replay()
            return
        for st in self.steps:
            st(s)

    def capture(self) -> None:
        """Record the whole step as one CUDA graph (replayed by run())."""
        torch = self.torch
        if any(isinstance(s, _CollectiveStep) and not s.capturable for s in self.steps):
            raise EvalError("steps with non-capturable (gloo) collectives are not captured")
        side = torch.cuda.Stream(device=self.device)
        # the warm-up pass is a real training step (in-place SGD): keep the variables
        # as they were, so capture() + the first replay is exactly one step. The
        # snapshot is queued before the side stream forks, so the warm-up's in-place
        # update is ordered after it.
        saved = self.var_arena.clone() if self.in_place else None
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            for st in self.steps:  # warm-up on the capture stream
                st(N.stream_ptr(side))
        torch.cuda.current_stream(self.device).wait_stream(side)
        if saved is not None:
            torch.cuda.current_stream(self.device).synchronize()
            self.var_arena.copy_(saved)
            torch.cuda.current_stream(self.device).synchronize()
            del saved
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for st in self.steps:
                st(N.stream_ptr(side))
        self.graph_exec = g

    def capture_with(self, pre=(), post=()):
        """One CUDA graph of `pre` callables + the whole step + `post` callables (each
        called with the capture stream's pointer). No warm-up: capture() already ran
        one, so kernels are loaded and GEMM plans tuned."""
        torch = self.torch
        if any(isinstance(s, _CollectiveStep) and not s.capturable for s in self.steps):
            raise EvalError("steps with non-capturable (gloo) collectives are not captured")
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            sp = N.stream_ptr(side)
            for f in pre:
                f(sp)
            for st in self.steps:
                st(sp)
            for f in post:
                f(sp)
        torch.cuda.current_stream(self.device).wait_stream(side)
        return g

    # ----------------------------------------------------------- host binding
    def h2d_staged(self, values: dict, copy_stream, slot: int, after=None) -> dict:
        """H2D of this step's shard into staging buffer `slot` on `copy_stream` (after
        event `after`, the last reader of that slot); the compute stream waits for it.
        Returns {input id: staging tensor}."""
        torch = self.torch
        staged = self.staging(values, slot)
        if after is not None:
            copy_stream.wait_event(after)
        with torch.cuda.stream(copy_stream):
            for k, v in values.items():
                if isinstance(v, np.ndarray):
                    v = torch.from_numpy(v)
                if v.dtype != torch.float32:
                    raise EvalError(f"binding {k!r} must be float32 for the async path")
                staged[k].copy_(v.reshape(-1), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(copy_stream)
        torch.cuda.current_stream(self.device).wait_event(ev)
        return staged

    def staging(self, values: dict, slot: int) -> dict:
        """The dense device staging buffers of `slot` for the inputs in `values`."""
        torch = self.torch
        if not hasattr(self, "_stg2"):
            self._stg2 = [{}, {}]
        for k in values:
            if k not in self._stg2[slot]:
                n = int(np.prod(self.t[k].dims))
                self._stg2[slot][k] = torch.empty(n, dtype=torch.float32, device=self.device)
        return {k: self._stg2[slot][k] for k in values}

    def pack_staged(self, staged: dict, stream_ptr) -> None:
        """Staging -> input layouts (the step's first launches; capturable). Dense
        inputs (labels) are a device copy on the current stream (the capture stream)."""
        for k, st in staged.items():
            t = self.t[k]
            n = st.numel()
            if t.pad == 0 and t.ld == t.dims[-1]:
                t.buf[:n].copy_(st, non_blocking=True)
            else:
                N.check(self.L.wap_pack(st.data_ptr(), t.layout(), t.ptr, 0, stream_ptr), "pack")

    def input_ids(self) -> list[str]:
        return [nid for nid in self.order if self.kind(nid) is OpKind.INPUT]

    def _upload(self, t: Tensor, value, stream=None) -> None:
        torch = self.torch
        src = value if isinstance(value, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(value))
        src = src.to(dtype=torch.float32)
        dev_src = src.to(self.device, non_blocking=True).contiguous()
        dims = t.dims
        lay = t.layout()
        if t.kind == "nhwc" and tuple(dev_src.shape) != dims:
            raise EvalError(f"binding has shape {tuple(dev_src.shape)}, expected {dims}")
        N.check(self.L.wap_pack(dev_src.data_ptr(), lay, t.ptr, 0, N.stream_ptr(stream)), "pack")
        self._keep_alive = dev_src

    def bind(self, values: dict, stream=None) -> None:
        """Copy host/torch arrays into Input (and optionally Variable) buffers."""
        for k, v in values.items():
            if k not in self.t or self.kind(k) not in (OpKind.INPUT, OpKind.VARIABLE):
                continue
            self._upload(self.t[k], v, stream)
        self.torch.cuda.current_stream(self.device).synchronize()

    def bind_async(self, values: dict, stream=None) -> None:
        """Stream-ordered binding for the training loop: pinned host (or device)
        tensors -> preallocated dense staging -> layout pack; no synchronisation."""
        torch = self.torch
        if not hasattr(self, "_staging"):
            self._staging = {}
        s = N.stream_ptr(stream)
        for k, v in values.items():
            t = self.t[k]
            n = int(np.prod(t.dims))
            dense_ok = (t.pad == 0 and t.ld == t.dims[-1])
            if isinstance(v, np.ndarray):
                v = torch.from_numpy(v)
            if v.dtype != torch.float32:
                raise EvalError(f"binding {k!r} must be float32 for the async path")
            if dense_ok:
                t.buf[:n].copy_(v.reshape(-1), non_blocking=True)
                continue
            st = self._staging.get(k)
            if st is None:
                st = self._staging[k] = torch.empty(n, dtype=torch.float32, device=self.device)
            if v.device.type == "cuda":
                src = v.reshape(-1)
            else:
                st.copy_(v.reshape(-1), non_blocking=True)
                src = st
            N.check(self.L.wap_pack(src.data_ptr(), t.layout(), t.ptr, 0, s), "pack")

    def bind_overlapped(self, values: dict, copy_stream) -> None:
        """Training-loop input path with the host->device copy off the critical path.

        The H2D copy of this step's shard runs on `copy_stream` into a dense staging
        buffer, so it overlaps the previous step still running on the compute
        stream; the compute stream then waits for it and packs / copies staging
        into the input buffers the step's kernels (or captured graph) read. The
        next call's H2D waits only until this pack has consumed the staging."""
        torch = self.torch
        if not hasattr(self, "_ov_staging"):
            self._ov_staging = {}
            self._ov_free = None
        compute = torch.cuda.current_stream(self.device)
        if self._ov_free is not None:
            copy_stream.wait_event(self._ov_free)
        staged = {}
        with torch.cuda.stream(copy_stream):
            for k, v in values.items():
                t = self.t[k]
                n = int(np.prod(t.dims))
                if isinstance(v, np.ndarray):
                    v = torch.from_numpy(v)
                if v.dtype != torch.float32:
                    raise EvalError(f"binding {k!r} must be float32 for the async path")
                st = self._ov_staging.get(k)
                if st is None:
                    st = self._ov_staging[k] = torch.empty(n, dtype=torch.float32, device=self.device)
                st.copy_(v.reshape(-1), non_blocking=True)
                staged[k] = st
        ev = torch.cuda.Event()
        ev.record(copy_stream)
        compute.wait_event(ev)
        s = N.stream_ptr(compute)
        for k, st in staged.items():
            t = self.t[k]
            n = st.numel()
            if t.pad == 0 and t.ld == t.dims[-1]:
                t.buf[:n].copy_(st, non_blocking=True)
            else:
                N.check(self.L.wap_pack(st.data_ptr(), t.layout(), t.ptr, 0, s), "pack")
        self._ov_free = torch.cuda.Event()
        self._ov_free.record(compute)

    def fetch(self, nid: str) -> np.ndarray:
        torch = self.torch
        t = self.t[nid]
        dims = t.dims
        dense = torch.empty(int(np.prod(dims)), dtype=torch.float32, device=self.device)
        N.check(self.L.wap_pack(dense.data_ptr(), t.layout(), t.ptr, 1, N.stream_ptr()), "unpack")
        return dense.cpu().numpy().reshape(dims)

    def outputs(self) -> dict[str, np.ndarray]:
        return {o: self.fetch(o) for o in self.g.outputs}

    def launches_per_step(self) -> int:
        before = N.launch_count()
        self.run()
        self.torch.cuda.synchronize()
        return N.launch_count() - before


def name_out_of(prog, buf) -> str | None:
    """Key of a mask-bits buffer in prog.mask_bits."""
    for k, v in prog.mask_bits.items():
        if v is buf:
            return k
    return None


class _CollectiveStep:
    """Marker base for steps that call into a cross-process collective.
    `capturable`: the step can be recorded into a CUDA graph (event waits, our
    kernels, NCCL); a gloo collective cannot."""

    capturable = True


class _BucketStep(_CollectiveStep):
    def __init__(self, name, fn, buf, side, torch, par=None, capturable=False):
        self.capturable = capturable
        self.name = name
        self.fn = fn
        self.buf = buf
        self.side = side
        self.torch = torch
        self.par = par  # stream producing weight gradients (may hold this bucket's grads)

    def __call__(self, stream: int) -> None:
        torch = self.torch
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.side.wait_event(ev)
        if self.par is not None:
            self.side.wait_stream(self.par)
        with torch.cuda.stream(self.side):
            self.fn(self.buf)


class _ParallelStep:
    """A native step issued on the weight-gradient stream, forked from the current
    stream at this point (capturable: the fork is an event wait)."""

    def __init__(self, step, side, torch):
        self.inner = step
        self.name = step.name
        self.side = side
        self.torch = torch
        for a in ("alg_flops", "alg_bytes", "shape", "desc", "call"):
            if hasattr(step, a):
                setattr(self, a, getattr(step, a))

    def __call__(self, stream: int) -> None:
        torch = self.torch
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.side.wait_event(ev)
        from . import _native as N

        self.inner(N.stream_ptr(self.side))


class _JoinParallel:
    def __init__(self, side, torch):
        self.name = "join(wgrad)"
        self.side = side
        self.torch = torch

    def __call__(self, stream: int) -> None:
        self.torch.cuda.current_stream().wait_stream(self.side)


class _SideStep(_CollectiveStep):
    """A native step issued on the comm stream after the compute stream reaches it."""

    def __init__(self, step, side, torch):
        self.name = step.name
        self.step = step
        self.alg_bytes = step.alg_bytes
        self.side = side
        self.torch = torch

    def __call__(self, stream: int) -> None:
        torch = self.torch
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.side.wait_event(ev)
        from . import _native as N

        self.step(N.stream_ptr(self.side))


class _FusedBucketStep:
    """wap_allreduce_sgd of one gradient bucket on the comm stream, after the
    compute stream reaches this point and the weight-gradient stream drained.
    Capturable: event waits plus one kernel launch."""

    def __init__(self, name, fused, offset, n, lr, slot, side, torch, par=None):
        self.name = f"allreduce_sgd[{name}]"
        self.fused, self.offset, self.n, self.lr, self.slot = fused, offset, n, lr, slot
        self.side, self.torch, self.par = side, torch, par
        self.alg_bytes = 12 * n  # local grad read + var read + var write (peer traffic on NVLink)

    def __call__(self, stream: int) -> None:
        torch = self.torch
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.side.wait_event(ev)
        if self.par is not None:
            self.side.wait_stream(self.par)
        from . import _native as N

        self.fused.launch(self.offset, self.n, self.lr, self.slot, N.stream_ptr(self.side))


class _JoinFused:
    def __init__(self, side, torch):
        self.name = "join(comm)"
        self.side = side
        self.torch = torch

    def __call__(self, stream: int) -> None:
        self.torch.cuda.current_stream().wait_stream(self.side)


class _JoinStep(_CollectiveStep):
    def __init__(self, side, torch):
        self.name = "join(comm)"
        self.side = side
        self.torch = torch

    def __call__(self, stream: int) -> None:
        self.torch.cuda.current_stream().wait_stream(self.side)
