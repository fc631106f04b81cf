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

import weakref
from dataclasses import dataclass
from enum import Enum
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
    """Immutable DAG with dense ids: the attribute shape of the reference's
    Graph (graph.py:77-95) that this package reads -- ops and tensors by
    position.  The plug-in passes the reference's own graphs; this type only
    serves standalone use (benchmarks, tests, the C-ABI examples)."""

    ops: tuple[OpNode, ...]
    tensors: tuple[TensorInfo, ...]

    @property
    def n_ops(self) -> int:
        return len(self.ops)

    @property
    def n_tensors(self) -> int:
        return len(self.tensors)


@dataclass(frozen=True)
class Schedule:
    """Order plus a timestep per op (reference graph.py:150-167)."""

    order: tuple[int, ...]
    timesteps: tuple[int, ...]
    ops_per_step: int = 1

    @property
    def n_steps(self) -> int:
        return max(self.timesteps) + 1 if self.timesteps else 0


def _dense(ids: list, what: str) -> dict[int, int]:
    """document id -> position; GraphFormatError for a missing / repeated id
    (the reference's messages, graph.py:199-215)."""
    index: dict[int, int] = {}
    for pos, i in enumerate(ids):
        if not isinstance(i, int):
            raise GraphFormatError(f"{what} at position {pos} has no integer id")
        if index.setdefault(i, pos) != pos:
            raise GraphFormatError(f"duplicate {what} id {i}")
    return index


def load_graph(doc: Mapping) -> Graph:
    """Interchange document -> Graph with dense ids, built CSR-first: each
    op's tensor ids become positions (a tensor's producer recorded as its
    outputs are read), then the flattened input list gives every tensor's
    consumers -- one entry per input occurrence, graph.py:227-231; the peak
    evaluator and the greedy scorer treat them differently, SURVEY §8a h1 --
    by one stable argsort, and acyclicity is a level-by-level peel of the
    predecessor in-degree array.  Malformed documents raise GraphFormatError /
    StructuralError with the reference's messages, in its order
    (graph.py:188-278)."""
    if not isinstance(doc, Mapping) or "ops" not in doc or "tensors" not in doc:
        raise GraphFormatError("document must contain 'ops' and 'tensors' arrays")
    raw_t, raw_o = doc["tensors"], doc["ops"]
    tpos = _dense([e.get("id") for e in raw_t], "tensor")
    _dense([e.get("id") for e in raw_o], "op")
    n, T = len(raw_o), len(raw_t)

    producer = np.full(T, -1, np.int64)

    def positions(e, key, what):
        out = []
        for t in e.get(key, []):
            p = tpos.get(t)
            if p is None:
                raise GraphFormatError(f"op {e['id']}: {what} tensor {t} does not exist")
            out.append(p)
        return out

    kinds, ins, outs = [], [], []
    for pos, e in enumerate(raw_o):
        try:
            kinds.append(OpKind(e.get("kind", "forward")))
        except ValueError:
            raise GraphFormatError(f"op {e['id']}: unknown kind {e.get('kind')!r}") from None
        ins.append(positions(e, "inputs", "input"))
        o = []
        for t in e.get("outputs", []):   # existence, then a second producer, per output
            p = positions({"id": e["id"], "outputs": [t]}, "outputs", "output")[0]
            if producer[p] >= 0:
                raise GraphFormatError(f"tensor {t} has multiple producers")
            producer[p] = pos
            o.append(p)
        outs.append(o)
    # consumers: the flattened inputs grouped by tensor, in op order
    in_t = np.fromiter((t for i in ins for t in i), np.int64)
    in_op = np.repeat(np.arange(n, dtype=np.int64), [len(i) for i in ins])
    by_t = np.argsort(in_t, kind="stable")
    cptr = np.zeros(T + 1, np.int64)
    np.cumsum(np.bincount(in_t, minlength=T), out=cptr[1:])
    cons_op = in_op[by_t].tolist()
    tensors = []
    for pos, e in enumerate(raw_t):
        size = e.get("size_bytes")
        if not isinstance(size, int):
            raise GraphFormatError(f"tensor {e['id']}: size_bytes must be an integer")
        if producer[pos] < 0:
            raise GraphFormatError(f"tensor {e['id']} has no producer op")
        cat = e.get("category")
        try:
            cat = TensorCategory.TEMPORARY_BUFFER if cat is None else TensorCategory(cat)
        except ValueError:
            raise GraphFormatError(f"tensor {e['id']}: unknown category {cat!r}") from None
        tensors.append(TensorInfo(pos, size, int(producer[pos]),
                                  tuple(cons_op[cptr[pos]:cptr[pos + 1]]), cat))
    ops = tuple(OpNode(pos, str(e.get("name", f"op{e['id']}")), kinds[pos], tuple(ins[pos]), tuple(outs[pos]))
                for pos, e in enumerate(raw_o))
    # acyclic: peel zero in-degree ops level by level over the deduplicated,
    # self-free predecessor edges (graph.py:97-104, 118-135)
    src, dst = producer[in_t], in_op
    keep = src != dst
    edges = np.unique(np.stack([src[keep], dst[keep]], axis=1), axis=0) if keep.any() else np.zeros((0, 2), np.int64)
    indeg = np.bincount(edges[:, 1], minlength=n) if len(edges) else np.zeros(n, np.int64)
    eo = np.argsort(edges[:, 0], kind="stable") if len(edges) else np.zeros(0, np.int64)
    sptr = np.zeros(n + 1, np.int64)
    if len(edges):
        np.cumsum(np.bincount(edges[:, 0], minlength=n), out=sptr[1:])
    succ = edges[eo, 1] if len(edges) else np.zeros(0, np.int64)
    level = np.flatnonzero(indeg == 0)
    seen = 0
    while len(level):
        seen += len(level)
        nxt = np.concatenate([succ[sptr[v]:sptr[v + 1]] for v in level]) if len(succ) else np.zeros(0, np.int64)
        np.subtract.at(indeg, nxt, 1)
        level = np.unique(nxt[indeg[nxt] == 0])
    if seen != n:
        raise StructuralError("graph contains a cycle")
    return Graph(ops, tuple(tensors))


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
    # one pass per object list (attribute reads dominate on 10k-op graphs)
    size_l, prod_l, clen, cons = [], [], [], []
    for t in g.tensors:
        size_l.append(t.size)
        prod_l.append(t.producer)
        clen.append(len(t.consumers))
        cons.extend(t.consumers)
    ilen, ins, olen, outs, kinds = [], [], [], [], []
    for o in g.ops:
        ilen.append(len(o.inputs))
        ins.extend(o.inputs)
        olen.append(len(o.outputs))
        outs.extend(o.outputs)
        kinds.append(KIND_CODE[_KIND_OF.get(o.kind) or OpKind(o.kind)])

    def ptr_of(lens):
        p = np.zeros(len(lens) + 1, dtype=np.int64)
        np.cumsum(np.asarray(lens, dtype=np.int64), out=p[1:])
        return p

    size = np.asarray(size_l, dtype=np.int64).reshape(T)
    producer = np.asarray(prod_l, dtype=np.int32).reshape(T)
    cons_ptr, in_ptr, out_ptr = ptr_of(clen), ptr_of(ilen), ptr_of(olen)
    cons_idx = np.asarray(cons, dtype=np.int32).reshape(-1)
    in_idx = np.asarray(ins, dtype=np.int32).reshape(-1)
    out_idx = np.asarray(outs, dtype=np.int32).reshape(-1)
    op_kind = np.asarray(kinds, dtype=np.uint8).reshape(n)
    cats = classify_tensors(g)
    is_act = np.fromiter((cats[t] is TensorCategory.ACTIVATION for t in range(T)), dtype=np.uint8, count=T)
    if max(int(cons_ptr[-1]), int(in_ptr[-1]), int(out_ptr[-1])) >= 2**31:
        raise GraphError("graph too large for int32 CSR offsets")
    arr = GraphArrays(n, T, size, producer, cons_ptr.astype(np.int32), cons_idx,
                      in_ptr.astype(np.int32), in_idx, out_ptr.astype(np.int32), out_idx,
                      op_kind, is_act)
    ent["arrays"] = arr
    return arr
