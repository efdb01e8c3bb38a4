"""`execute` / `compare` with the reference's signatures, evaluated on the GPU.

Drop-in for wap.interp (interp.py:44-66, 122-215, 242-309): same deterministic
variable/input bindings (PCG64 keyed by crc32 of the base id, 0.1*N(0,1)
weights), same output dictionary (loss per replica = shard mean, updated
variables), same equivalence report. The arithmetic runs in the sm_100a
kernels through `runtime.Program` (fp32 storage; GEMMs in 3xTF32 by default,
which is fp32-accurate). Results come back as float64 numpy arrays like the
reference's.
"""

from __future__ import annotations

import logging
import zlib
from dataclasses import dataclass

import numpy as np

from .errors import EvalError
from .ir import Graph, OpKind, base_id, infer_shapes, replica_index

logger = logging.getLogger(__name__)

INIT_SCALE = 0.1


def _rng(seed: int, namespace: str, name: str) -> np.random.Generator:
    return np.random.default_rng((int(seed) & 0xFFFFFFFF, zlib.crc32(f"{namespace}:{name}".encode("utf-8"))))


def initial_variables(graph: Graph, seed: int) -> dict[str, np.ndarray]:
    """0.1 * N(0,1) per Variable, stream keyed by the base id (replicas share it)."""
    return {n.id: INIT_SCALE * _rng(seed, "var", base_id(n.id)).standard_normal(tuple(n.attr("shape")))
            for n in graph if n.kind is OpKind.VARIABLE}


def generate_inputs(graph: Graph, seed: int) -> dict[str, np.ndarray]:
    """Standard-normal binding for every Input (same stream scheme, namespace 'in')."""
    return {n.id: _rng(seed, "in", base_id(n.id)).standard_normal(tuple(n.attr("shape")))
            for n in graph if n.kind is OpKind.INPUT}


_PROGRAMS: dict[tuple, object] = {}


def _program(graph: Graph, precision: int):
    from .ir import serialize
    from .runtime import Program

    key = (serialize(graph), precision)
    prog = _PROGRAMS.get(key)
    if prog is None:
        if len(_PROGRAMS) > 8:
            _PROGRAMS.clear()
        prog = Program(graph, precision=precision)
        _PROGRAMS[key] = prog
    return prog


def execute(graph: Graph, inputs: dict[str, np.ndarray], seed: int = 0, precision: int = 3) -> dict[str, np.ndarray]:
    """Evaluate the graph on the GPU and return its outputs (float64 arrays)."""
    for n in graph:
        if n.kind is OpKind.INPUT and n.id not in inputs:
            raise EvalError(f"missing input binding for {n.id!r}")
    prog = _program(graph, precision)
    binding = {}
    for n in graph:
        if n.kind is OpKind.INPUT:
            binding[n.id] = inputs[n.id]
        elif n.kind is OpKind.VARIABLE:
            binding[n.id] = inputs[n.id] if n.id in inputs else \
                INIT_SCALE * _rng(seed, "var", base_id(n.id)).standard_normal(tuple(n.attr("shape")))
    prog.bind(binding)
    prog.run()
    out = {k: v.astype(np.float64) for k, v in prog.outputs().items()}
    for k, v in out.items():
        if not np.all(np.isfinite(v)):
            logger.warning("numeric overflow: node %r produced non-finite values", k)
    return out


@dataclass(frozen=True)
class EquivalenceReport:
    deviations: dict[str, float]
    tolerance: float

    @property
    def passed(self) -> bool:
        return all(d <= self.tolerance for d in self.deviations.values())

    @property
    def max_deviation(self) -> float:
        return max(self.deviations.values(), default=0.0)

    def failures(self) -> list[str]:
        return sorted(o for o, d in self.deviations.items() if d > self.tolerance)


def relative_deviation(a: np.ndarray, b: np.ndarray) -> float:
    if a.shape != b.shape:
        raise EvalError(f"output shapes differ: {a.shape} vs {b.shape}")
    scale = max(float(np.abs(a).max(initial=0.0)), float(np.abs(b).max(initial=0.0)), 1e-30)
    return float(np.abs(a - b).max(initial=0.0)) / scale


def _reassemble(graph_b: Graph, replicas: list[str], vals: dict[str, np.ndarray]):
    kind = graph_b.node(replicas[0]).kind
    parts = [vals[r] for r in replicas]
    if kind in (OpKind.SGD_UPDATE, OpKind.VARIABLE, OpKind.ALL_REDUCE_SUM):
        return parts
    if kind is OpKind.SOFTMAX_XENT_LOSS:
        acc = parts[0].copy()
        for p in parts[1:]:
            acc = acc + p
        return acc / len(parts)
    shape = graph_b.node(replicas[0]).output_shape
    return np.concatenate(parts, axis=shape.batch_axis if shape is not None else 0)


def compare(graph_a: Graph, graph_b: Graph, inputs: dict[str, np.ndarray], seed: int = 0,
            tol: float = 1e-6, precision: int = 3) -> EquivalenceReport:
    """Execute both graphs on the GPU and compare matched outputs (interp.py:267-309)."""
    va = execute(graph_a, inputs, seed, precision)
    vb = execute(graph_b, inputs, seed, precision)
    sb = infer_shapes(graph_b)
    groups: dict[str, list[str]] = {}
    for o in graph_b.outputs:
        groups.setdefault(base_id(o), []).append(o)
    for grp in groups.values():
        grp.sort(key=lambda o: replica_index(o) or 0)
    devs: dict[str, float] = {}
    matched: set[str] = set()
    for o in graph_a.outputs:
        grp = groups.get(o)
        if not grp:
            raise EvalError(f"output mismatch: {o!r} has no counterpart in {graph_b.name!r}")
        matched.update(grp)
        if grp == [o]:
            devs[o] = relative_deviation(va[o], vb[o])
            continue
        rebuilt = _reassemble(sb, grp, vb)
        if isinstance(rebuilt, list):
            devs[o] = max(relative_deviation(va[o], r) for r in rebuilt)
        else:
            devs[o] = relative_deviation(va[o], rebuilt)
    extra = set(graph_b.outputs) - matched
    if extra:
        raise EvalError(f"output mismatch: {sorted(extra)} have no counterpart in {graph_a.name!r}")
    return EquivalenceReport(devs, tol)
