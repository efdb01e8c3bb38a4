"""B200-native WAP: workload-aware data-parallel training (arXiv 1811.01532).

Drop-in for the reference `wap` package's hot path: describe a
single-device training graph, let the WAU choose the GPU count, replicate the
graph across that many ranks, and run replicated-variables SGD steps on
hand-written sm_100a kernels (tcgen05 implicit-GEMM conv/FC, vectorised
elementwise/reduction kernels, NCCL gradient allreduce).

The public names mirror `wap/__init__.py:10-67`; the heavy submodules load
lazily so the host-side API works on machines without a GPU.
"""

from .errors import (
    BuildError,
    CycleError,
    EvalError,
    ParseError,
    ShapeError,
    SimError,
    TransformError,
    WapError,
    WorkloadError,
)

__version__ = "0.1.0"

_LAZY = {
    # ir
    "BYTES_PER_ELEMENT": "ir", "Finding": "ir", "Graph": "ir", "GraphBuilder": "ir", "Node": "ir",
    "OpKind": "ir", "TensorShape": "ir", "ValidationReport": "ir", "base_id": "ir",
    "deserialize": "ir", "infer_shapes": "ir", "replica_index": "ir", "serialize": "ir",
    "topo_order": "ir", "validate": "ir",
    # training / models
    "TrainingGraphSpec": "training", "build_training_graph": "training",
    # workloads
    "LayerWorkload": "workloads", "NetworkWorkload": "workloads", "extract_workloads": "workloads",
    "flops_of": "workloads", "node_flops": "workloads",
    # planner
    "CostEstimate": "planner", "DeviceProfile": "planner", "ParallelPlan": "planner",
    "comm_time": "planner", "compute_time": "planner", "estimate_power": "planner",
    "estimate_total": "planner", "load_profile": "planner", "plan_for_degree": "planner",
    "select_parallelism": "planner",
    # transform
    "TransformReport": "graph_modifier", "check_parallel_structure": "graph_modifier",
    "localize_auxiliary": "graph_modifier", "optimize_gradient_aggregation": "graph_modifier",
    "replicate_primary": "graph_modifier", "transform": "graph_modifier",
    # execution (GPU)
    "EquivalenceReport": "interp", "compare": "interp", "execute": "interp",
    "generate_inputs": "interp", "initial_variables": "interp",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    import importlib

    value = getattr(importlib.import_module(f".{mod}", __name__), name)
    globals()[name] = value
    return value


def __dir__():
    return sorted(list(globals()) + list(_LAZY))
