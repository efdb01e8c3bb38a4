"""Host side of the on-device Workload Analysis Unit (csrc/wau.cu).

`layer_descriptors(graph)` turns a shape-inferred training graph into the
per-layer shape records the kernel consumes (the kernel itself derives the
FLOPs, weight bytes, Eq. (1) terms and the decision). `select` runs it on the
current CUDA device and returns (d, [CostEstimate...]) in candidate order.
"""

from __future__ import annotations

import ctypes as C
import sys

from . import _native as N
from .errors import WorkloadError
from .ir import GRAD_COMPANION_KINDS, PRIMARY_KINDS, Graph, OpKind, infer_shapes, topo_order
from .planner import CostEstimate, DeviceProfile
from .workloads import NetworkWorkload

ALGO_CODES = {"ring": 0, "naive_all_to_all": 1}
# planner.py:191-192 sums with the builtin sum(): Neumaier-compensated from CPython 3.12
# on, a plain left fold before. The device kernel follows the interpreter it runs under.
PLAIN_SUM = 0x100 if sys.version_info < (3, 12) else 0


def layer_descriptors(graph: Graph) -> tuple[list[N.wap_wau_layer_t], int]:
    """Shape records for every primary layer in topological order, plus G."""
    g = graph if all(n.output_shape is not None for n in graph) else infer_shapes(graph)
    users = g.consumers()
    n_grad: dict[str, int] = {}
    for n in g:
        if n.kind in GRAD_COMPANION_KINDS and n.attr("layer") is not None:
            n_grad[n.attr("layer")] = n_grad.get(n.attr("layer"), 0) + 1
    out = []
    batches = set()
    for nid in topo_order(g):
        n = g.node(nid)
        if n.kind not in PRIMARY_KINDS:
            continue
        rec = N.wap_wau_layer_t()
        rec.n_grad = n_grad.get(nid, 0)
        wnode = g.node(n.inputs[1])
        welems = wnode.output_shape.elements() if wnode.kind is OpKind.VARIABLE else 0
        for c in users[nid]:
            cn = g.node(c)
            if cn.kind is OpKind.BIAS_ADD and g.node(cn.inputs[1]).kind is OpKind.VARIABLE:
                welems += g.node(cn.inputs[1]).output_shape.elements()
        rec.weight_elems = welems
        if n.kind is OpKind.MATMUL:
            i, o = wnode.output_shape.dims
            rec.kind, rec.batch, rec.cin, rec.cout = 0, n.output_shape.dims[0], i, o
            rec.out_h = rec.out_w = rec.k = 1
        else:
            bsz, ho, wo, co = n.output_shape.dims
            k, _, ci, _ = wnode.output_shape.dims
            rec.kind, rec.batch, rec.out_h, rec.out_w, rec.cin, rec.cout, rec.k = 1, bsz, ho, wo, ci, co, k
        batches.add(n.output_shape.batch)
        out.append(rec)
    if len(batches) > 1:
        raise WorkloadError(f"inconsistent layer batch sizes: {sorted(batches)}")
    G = batches.pop() if batches else max(
        (n.output_shape.batch for n in g if n.kind is OpKind.INPUT), default=1)
    return out, G


def workload_descriptors(workload: NetworkWorkload) -> list[N.wap_wau_layer_t]:
    """Pre-counted records (kind 2) for a NetworkWorkload built elsewhere."""
    out = []
    for l in workload.layers:
        rec = N.wap_wau_layer_t()
        rec.kind, rec.batch, rec.cin = 2, l.flops_fwd, l.flops_bwd
        if l.weight_bytes % 4:
            raise WorkloadError(f"weight bytes of {l.layer!r} not a multiple of 4")
        rec.weight_elems = l.weight_bytes // 4
        out.append(rec)
    return out


def run(records, G: int, n_devices: int, profile: DeviceProfile, algo: str = "ring", device=None):
    """Launch the WAU kernel; returns (d, estimates, per-layer (fwd, bwd) FLOPs)."""
    import torch

    if algo not in ALGO_CODES:
        raise WorkloadError(f"unknown aggregation algorithm {algo!r}")
    if n_devices < 1:
        raise WorkloadError("device set is empty")
    dev = device or torch.device("cuda", torch.cuda.current_device())
    n = len(records)
    arr = (N.wap_wau_layer_t * max(n, 1))(*records)
    host = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8)
    d_layers = host.to(dev)
    flops = torch.zeros(2 * max(n, 1), dtype=torch.int64, device=dev)
    t_c = torch.empty(n_devices, dtype=torch.float64, device=dev)
    t_s = torch.empty_like(t_c)
    thr = torch.empty_like(t_c)
    d_out = torch.zeros(1, dtype=torch.int32, device=dev)
    prof = N.wap_wau_profile_t(profile.peak_flops, profile.efficiency_knee_flops, profile.link_bandwidth,
                               profile.link_latency, profile.allreduce_chunk_latency)
    with torch.cuda.device(dev):
        N.check(N.lib().wap_wau_select(C.cast(C.c_void_p(d_layers.data_ptr()), C.POINTER(N.wap_wau_layer_t)),
                                       n, G, n_devices, prof, ALGO_CODES[algo] | PLAIN_SUM, flops.data_ptr(),
                                       t_c.data_ptr(), t_s.data_ptr(), thr.data_ptr(), d_out.data_ptr(),
                                       N.stream_ptr()), "wap_wau_select", WorkloadError)
        torch.cuda.current_stream().synchronize()
    tc, ts, th = t_c.cpu().tolist(), t_s.cpu().tolist(), thr.cpu().tolist()
    ests = [CostEstimate(d, tc[d - 1], ts[d - 1], th[d - 1]) for d in range(1, n_devices + 1) if G % d == 0]
    fl = flops.cpu().tolist()
    return int(d_out.item()), ests, [(fl[2 * i], fl[2 * i + 1]) for i in range(n)]


def select(workload: NetworkWorkload, n_devices: int, profile: DeviceProfile, algo: str = "ring",
           graph: Graph | None = None):
    """(d, estimates); from the graph's shapes when given, else from the workload counts."""
    if graph is not None:
        recs, G = layer_descriptors(graph)
    else:
        recs, G = workload_descriptors(workload), workload.global_batch
    d, ests, _ = run(recs, G, n_devices, profile, algo)
    return d, ests
