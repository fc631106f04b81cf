"""B200-native (sm_100a) ROAM planner hot path (arXiv 2310.19295).

Drop-in, GPU-backed versions of the reference ``memplan`` hot-path functions
(see DESIGN.md for the reference file:line each one replaces) plus the batched
candidate-evaluation API.  All compute runs in ``libroam.so`` (include/roam.h);
there is no CPU fallback.
"""

from .graph import (ConfigError, Graph, GraphError, GraphFormatError, OpKind, OpNode, Schedule,
                    ScheduleError, StructuralError, TensorCategory, TensorInfo, classify_tensors,
                    load_graph)
from .evaluator import (argmin_orders, evaluate_orders, generate_orders, live_bytes_by_timestep,
                        peak_memory, sequential_schedule, tensor_lifetimes, validate_schedule)

__all__ = [
    "ConfigError", "Graph", "GraphError", "GraphFormatError", "OpKind", "OpNode", "Schedule",
    "ScheduleError", "StructuralError", "TensorCategory", "TensorInfo", "classify_tensors",
    "load_graph", "argmin_orders",
    "evaluate_orders", "generate_orders", "live_bytes_by_timestep", "peak_memory",
    "sequential_schedule", "tensor_lifetimes", "validate_schedule",
]
