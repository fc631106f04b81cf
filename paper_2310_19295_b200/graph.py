"""Graph IR for the planner hot path: the host-side mirror of the reference's
``memplan.graph`` types (reference: pkg/src/memplan/graph.py).

Same public names, argument meaning and exceptions as the reference so a caller
can switch imports; the evaluation functions themselves (``peak_memory``,
``tensor_lifetimes``, ``live_bytes_by_timestep``, ``validate_schedule``) live in
:mod:`.evaluator` and run on the GPU through ``libroam``.

Marshalling (``graph_arrays``) turns any object with the reference's shape
(``.ops[i].inputs/.outputs/.kind``, ``.tensors[t].size/.producer/.consumers``)
into flat CSR numpy arrays -- so graphs built by the reference library itself
can be passed straight in.
"""

from __future__ import annotations

import heapq
import json
import weakref
from dataclasses import dataclass
from enum import Enum
from functools import cached_property
from typing import Mapping

import numpy as np


class GraphError(Exception):
    """Base error (reference graph.py:19)."""


class GraphFormatError(GraphError):
    """Malformed interchange document (graph.py:23)."""


class StructuralError(GraphError):
    """Structural precondition violated (graph.py:27)."""


class ScheduleError(GraphError):
    """Schedule invalid for its graph (graph.py:31)."""


class ConfigError(GraphError):
    """Invalid solver configuration (graph.py:35)."""


class OpKind(str, Enum):
    FORWARD = "forward"
    BACKWARD = "backward"
    WEIGHT_UPDATE = "weight_update"
    LOSS = "loss"


class TensorCategory(str, Enum):
    ACTIVATION = "activation"
    TEMPORARY_BUFFER = "temporary_buffer"
    GRADIENT = "gradient"
    WEIGHT = "weight"
    OPTIMIZER_STATE = "optimizer_state"


_PINNED = (TensorCategory.WEIGHT, TensorCategory.OPTIMIZER_STATE)
KIND_CODE = {OpKind.FORWARD: 0, OpKind.BACKWARD: 1, OpKind.WEIGHT_UPDATE: 2, OpKind.LOSS: 3}


@dataclass(frozen=True)
class OpNode:
    id: int
    name: str
    kind: OpKind
    inputs: tuple[int, ...]
    outputs: tuple[int, ...]


@dataclass(frozen=True)
class TensorInfo:
    id: int
    size: int
    producer: int
    consumers: tuple[int, ...]
    category: TensorCategory = TensorCategory.TEMPORARY_BUFFER


@dataclass(frozen=True)
class Graph:
    """Immutable DAG with dense ids (reference graph.py:77-135)."""

    ops: tuple[OpNode, ...]
    tensors: tuple[TensorInfo, ...]

    @property
    def n_ops(self) -> int:
        return len(self.ops)

    @property
    def n_tensors(self) -> int:
        return len(self.tensors)

    @cached_property
    def direct_preds(self) -> tuple[tuple[int, ...], ...]:
        # producers of the op's inputs, deduplicated, self discarded (graph.py:97-104)
        return tuple(
            tuple(sorted({self.tensors[t].producer for t in op.inputs} - {op.id}))
            for op in self.ops
        )

    @cached_property
    def direct_succs(self) -> tuple[tuple[int, ...], ...]:
        out = []
        for op in self.ops:
            s: set[int] = set()
            for t in op.outputs:
                s.update(self.tensors[t].consumers)
            s.discard(op.id)
            out.append(tuple(sorted(s)))
        return tuple(out)

    def topological_order(self) -> tuple[int, ...]:
        """Kahn with smallest-id ties; StructuralError on a cycle (graph.py:118-135)."""
        indeg = [len(p) for p in self.direct_preds]
        ready = [v for v in range(self.n_ops) if indeg[v] == 0]
        heapq.heapify(ready)
        order = []
        while ready:
            v = heapq.heappop(ready)
            order.append(v)
            for w in self.direct_succs[v]:
                indeg[w] -= 1
                if indeg[w] == 0:
                    heapq.heappush(ready, w)
        if len(order) != self.n_ops:
            raise StructuralError("graph contains a cycle")
        return tuple(order)


@dataclass(frozen=True)
class Schedule:
    """Order plus a timestep per op (reference graph.py:150-167)."""

    order: tuple[int, ...]
    timesteps: tuple[int, ...]
    ops_per_step: int = 1

    @property
    def n_steps(self) -> int:
        return max(self.timesteps) + 1 if self.timesteps else 0


@dataclass(frozen=True)
class Violation:
    kind: str
    message: str


@dataclass(frozen=True)
class ValidationReport:
    violations: tuple[Violation, ...] = ()

    @property
    def ok(self) -> bool:
        return not self.violations

    def kinds(self) -> tuple[str, ...]:
        return tuple(v.kind for v in self.violations)


def load_graph(doc: Mapping) -> Graph:
    """Interchange document -> Graph with dense ids (reference graph.py:188-278).

    Consumers get one entry per input occurrence (graph.py:227-231), which the
    peak evaluator and the greedy scorer treat differently.
    """
    if not isinstance(doc, Mapping) or "ops" not in doc or "tensors" not in doc:
        raise GraphFormatError("document must contain 'ops' and 'tensors' arrays")
    raw_t, raw_o = doc["tensors"], doc["ops"]
    tindex: dict[int, int] = {}
    for pos, e in enumerate(raw_t):
        tid = e.get("id")
        if not isinstance(tid, int):
            raise GraphFormatError(f"tensor at position {pos} has no integer id")
        if tid in tindex:
            raise GraphFormatError(f"duplicate tensor id {tid}")
        tindex[tid] = pos
    oindex: dict[int, int] = {}
    for pos, e in enumerate(raw_o):
        oid = e.get("id")
        if not isinstance(oid, int):
            raise GraphFormatError(f"op at position {pos} has no integer id")
        if oid in oindex:
            raise GraphFormatError(f"duplicate op id {oid}")
        oindex[oid] = pos

    producer: dict[int, int] = {}
    consumers: list[list[int]] = [[] for _ in raw_t]
    ops = []
    for pos, e in enumerate(raw_o):
        try:
            kind = OpKind(e.get("kind", "forward"))
        except ValueError:
            raise GraphFormatError(f"op {e['id']}: unknown kind {e.get('kind')!r}")
        ins = []
        for t in e.get("inputs", []):
            if t not in tindex:
                raise GraphFormatError(f"op {e['id']}: input tensor {t} does not exist")
            ins.append(tindex[t])
            consumers[tindex[t]].append(pos)
        outs = []
        for t in e.get("outputs", []):
            if t not in tindex:
                raise GraphFormatError(f"op {e['id']}: output tensor {t} does not exist")
            d = tindex[t]
            if d in producer:
                raise GraphFormatError(f"tensor {t} has multiple producers")
            producer[d] = pos
            outs.append(d)
        ops.append(OpNode(pos, str(e.get("name", f"op{e['id']}")), kind, tuple(ins), tuple(outs)))

    tensors = []
    for pos, e in enumerate(raw_t):
        size = e.get("size_bytes")
        if not isinstance(size, int):
            raise GraphFormatError(f"tensor {e['id']}: size_bytes must be an integer")
        if pos not in producer:
            raise GraphFormatError(f"tensor {e['id']} has no producer op")
        cat = TensorCategory.TEMPORARY_BUFFER
        if e.get("category") is not None:
            try:
                cat = TensorCategory(e["category"])
            except ValueError:
                raise GraphFormatError(f"tensor {e['id']}: unknown category {e['category']!r}")
        tensors.append(TensorInfo(pos, size, producer[pos], tuple(consumers[pos]), cat))
    g = Graph(tuple(ops), tuple(tensors))
    g.topological_order()
    return g


def graph_to_doc(g) -> dict:
    return {
        "ops": [
            {"id": o.id, "name": o.name, "kind": OpKind(o.kind).value,
             "inputs": list(o.inputs), "outputs": list(o.outputs)}
            for o in g.ops
        ],
        "tensors": [
            {"id": t.id, "size_bytes": t.size, "category": TensorCategory(t.category).value}
            for t in g.tensors
        ],
    }


def load_graph_json(text: str) -> Graph:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise GraphFormatError(f"invalid JSON: {exc}") from exc
    return load_graph(doc)


def validate_graph(g) -> ValidationReport:
    """Structural invariants as report entries (reference graph.py:309-332)."""
    v: list[Violation] = []
    seen: dict[int, int] = {}
    for op in g.ops:
        for t in op.outputs:
            if t in seen:
                v.append(Violation("multi_producer", f"tensor {t} produced by ops {seen[t]} and {op.id}"))
            seen[t] = op.id
    for t in g.tensors:
        if t.size <= 0:
            v.append(Violation("zero_size", f"tensor {t.id} has size {t.size}"))
        if t.producer != g.ops[t.producer].id or t.id not in g.ops[t.producer].outputs:
            v.append(Violation("producer_mismatch", f"tensor {t.id} producer link broken"))
        for c in t.consumers:
            if t.id not in g.ops[c].inputs:
                v.append(Violation("consumer_mismatch", f"tensor {t.id} consumer {c} link broken"))
    try:
        g.topological_order()
    except StructuralError:
        v.append(Violation("cycle", "graph contains a cycle"))
    return ValidationReport(tuple(v))


def classify_tensors(g) -> dict[int, TensorCategory]:
    """Activation / gradient / temporary taxonomy (reference graph.py:471-492),
    computed once per graph; each call returns its own dict."""
    ent = graph_cache(g)
    hit = ent.get("categories")
    if hit is None:
        hit = ent["categories"] = _classify(g)
    return dict(hit)


_KIND_OF = {k.value: k for k in OpKind}          # str-valued enums hash as their value,
_CAT_OF = {c.value: c for c in TensorCategory}   # so the reference's members look up too


def _classify(g) -> dict[int, TensorCategory]:
    kinds = [_KIND_OF.get(o.kind) or OpKind(o.kind) for o in g.ops]
    fwd, bwd, wu = OpKind.FORWARD, OpKind.BACKWARD, OpKind.WEIGHT_UPDATE
    out: dict[int, TensorCategory] = {}
    for t in g.tensors:
        cat = _CAT_OF.get(t.category) or TensorCategory(t.category)
        if cat in _PINNED:
            out[t.id] = cat
            continue
        pk = kinds[t.producer]
        if pk is fwd and any(kinds[c] is bwd for c in t.consumers):
            out[t.id] = TensorCategory.ACTIVATION
        elif pk is bwd and any(kinds[c] is wu for c in t.consumers):
            out[t.id] = TensorCategory.GRADIENT
        else:
            out[t.id] = TensorCategory.TEMPORARY_BUFFER
    return out


# --------------------------------------------------------------------------
# CSR marshalling: once per graph, cached by object identity.


@dataclass(frozen=True)
class GraphArrays:
    n_ops: int
    n_tensors: int
    size: np.ndarray       # int64[T]
    producer: np.ndarray   # int32[T]
    cons_ptr: np.ndarray   # int32[T+1]
    cons_idx: np.ndarray   # int32[E]  one entry per input occurrence
    in_ptr: np.ndarray     # int32[n+1]
    in_idx: np.ndarray     # int32[E]  op inputs in document order (duplicates kept)
    out_ptr: np.ndarray    # int32[n+1]
    out_idx: np.ndarray    # int32[sum outputs]
    op_kind: np.ndarray    # uint8[n]
    is_act: np.ndarray     # uint8[T] classify_tensors(g) is ACTIVATION


_CACHE: dict[int, dict] = {}


def graph_cache(g) -> dict:
    """Per-graph scratch dict (CSR arrays, device handle), dropped with the graph."""
    ent = _CACHE.get(id(g))
    if ent is not None and ent["ref"]() is g:
        return ent
    ent = {"ref": weakref.ref(g)}
    _CACHE[id(g)] = ent
    weakref.finalize(g, _drop_cache, id(g))
    return ent


def _drop_cache(key: int) -> None:
    ent = _CACHE.pop(key, None)
    if ent and "close" in ent:
        ent["close"]()


def graph_arrays(g) -> GraphArrays:
    """Flatten a (reference-shaped) graph into CSR numpy arrays."""
    ent = graph_cache(g)
    if "arrays" in ent:
        return ent["arrays"]
    n, T = len(g.ops), len(g.tensors)
    size = np.fromiter((t.size for t in g.tensors), dtype=np.int64, count=T)
    producer = np.fromiter((t.producer for t in g.tensors), dtype=np.int32, count=T)
    cons_len = np.fromiter((len(t.consumers) for t in g.tensors), dtype=np.int64, count=T)
    cons_ptr = np.zeros(T + 1, dtype=np.int64)
    np.cumsum(cons_len, out=cons_ptr[1:])
    cons_idx = np.fromiter((c for t in g.tensors for c in t.consumers), dtype=np.int32,
                           count=int(cons_ptr[-1]))
    in_len = np.fromiter((len(o.inputs) for o in g.ops), dtype=np.int64, count=n)
    in_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(in_len, out=in_ptr[1:])
    in_idx = np.fromiter((t for o in g.ops for t in o.inputs), dtype=np.int32, count=int(in_ptr[-1]))
    out_len = np.fromiter((len(o.outputs) for o in g.ops), dtype=np.int64, count=n)
    out_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(out_len, out=out_ptr[1:])
    out_idx = np.fromiter((t for o in g.ops for t in o.outputs), dtype=np.int32, count=int(out_ptr[-1]))
    op_kind = np.fromiter((KIND_CODE[_KIND_OF.get(o.kind) or OpKind(o.kind)] for o in g.ops),
                          dtype=np.uint8, count=n)
    cats = classify_tensors(g)
    is_act = np.fromiter((cats[t] is TensorCategory.ACTIVATION for t in range(T)), dtype=np.uint8, count=T)
    if max(int(cons_ptr[-1]), int(in_ptr[-1]), int(out_ptr[-1])) >= 2**31:
        raise GraphError("graph too large for int32 CSR offsets")
    arr = GraphArrays(n, T, size, producer, cons_ptr.astype(np.int32), cons_idx,
                      in_ptr.astype(np.int32), in_idx, out_ptr.astype(np.int32), out_idx,
                      op_kind, is_act)
    ent["arrays"] = arr
    return arr
