"""Layout checks and the greedy (LLFB) packer on the GPU -- drop-ins for the
reference's ``memplan.layout`` / ``memplan.simulator`` hot-path functions.

  LayoutItem / LayoutProblem / MemoryLayout   layout.py:20-58 (same fields)
  layout_violations      layout.py:305-329   -> rm_layout_violations (K2)
  items_from_schedule    layout.py:332-346
  validate_layout        layout.py:349-352   -> K2
  replay_static          simulator.py:129-145 -> K2 (actual = max extent)
  conflict_pairs         layout.py:420-429   -> K2 (repair_conflicts' detector)
  llfb_layout            layout.py:100-118   -> rm_llfb_batch PLAIN (K3)
  constrained_llfb_layout layout.py:121-146  -> rm_llfb_batch CONSTRAINED (K3)
  solve_layouts          planner.py:134-138 batch dispatch (_pool_map of _solve_layout)
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib, ptr
from .graph import Schedule, TensorCategory, classify_tensors


@dataclass(frozen=True)
class LayoutItem:
    tensor: int
    size: int
    start: int
    end: int  # inclusive timestep
    is_activation: bool = False

    def overlaps(self, other: "LayoutItem") -> bool:
        return self.start <= other.end and other.start <= self.end


@dataclass(frozen=True)
class LayoutProblem:
    items: tuple[LayoutItem, ...]
    activations_at_bottom: bool = False
    time_budget: float = 60.0
    node_cap: int | None = None


@dataclass(frozen=True)
class LayoutStats:
    nodes: int
    wall_time: float


@dataclass(frozen=True)
class MemoryLayout:
    offsets: dict[int, int]
    capacity: int
    activation_block: int = 0
    optimal: bool = True
    stats: LayoutStats = LayoutStats(0, 0.0)


def _item_arrays(items: Sequence):
    N = len(items)
    start = np.fromiter((i.start for i in items), np.int64, N)
    end = np.fromiter((i.end for i in items), np.int64, N)
    size = np.fromiter((i.size for i in items), np.int64, N)
    if N and (start.min() < -(2**31) or end.max() >= 2**31 or start.max() >= 2**31 or end.min() < -(2**31)):
        raise ValueError("item timesteps exceed int32")
    return start.astype(np.int32), end.astype(np.int32), size


def _k2(items: Sequence, offsets: Mapping[int, int], capacity: int, max_pairs: int):
    _lib.require_device()
    N = len(items)
    start, end, size = _item_arrays(items)
    has = np.fromiter((i.tensor in offsets for i in items), np.uint8, N)
    off = np.fromiter((offsets.get(i.tensor, 0) for i in items), np.int64, N)
    flags = np.empty(N, np.uint8)
    cap = max(int(max_pairs), 0)
    pairs = np.empty(2 * max(cap, 1), np.int64)
    npairs = C.c_int64(0)
    mx = C.c_int64(0)
    check(lib().rm_layout_violations(N, ptr(start), ptr(end), ptr(size), ptr(off), ptr(has),
                                     int(capacity), ptr(flags), ptr(pairs), cap, C.byref(npairs),
                                     C.byref(mx), None), "rm_layout_violations")
    if npairs.value > cap:   # pairs buffer too small: fetch all
        return _k2(items, offsets, capacity, npairs.value)
    return flags, off, pairs[: 2 * npairs.value].reshape(-1, 2), mx.value


def layout_violations(items: Sequence, offsets: Mapping[int, int], capacity: int) -> list[str]:
    """Overlap / extent / missing-offset violations (layout.py:305-329): the
    per-item messages in item order, then each overlapping pair (i < j)."""
    flags, off, pairs, _ = _k2(items, offsets, capacity, 1024)
    return _messages(items, capacity, flags, off, pairs)


def _messages(items, capacity, flags, off, pairs) -> list[str]:
    out: list[str] = []
    for k in np.flatnonzero(flags):
        it = items[k]
        f = int(flags[k])
        if f & 1:
            out.append(f"tensor {it.tensor} has no offset")
            continue
        o = int(off[k])
        if f & 2:
            out.append(f"tensor {it.tensor} has negative offset {o}")
        if f & 4:
            out.append(f"tensor {it.tensor} extent {o + it.size} exceeds capacity {capacity}")
    for i, j in pairs.tolist():
        out.append(f"tensors {items[i].tensor} and {items[j].tensor} overlap in time and address")
    return out


def conflict_pairs(items: Sequence, offsets: Mapping[int, int]) -> list[tuple[int, int]]:
    """repair_conflicts' detector (layout.py:420-429) over items sorted by
    tensor id: every (a, b) index pair overlapping in time and address."""
    _, _, pairs, _ = _k2(items, offsets, 2**62, 1024)
    return [tuple(p) for p in pairs.tolist()]


def items_from_schedule(g, s: Schedule) -> tuple[LayoutItem, ...]:
    """layout.py:332-346 (lifetimes from the GPU evaluator)."""
    from .evaluator import tensor_lifetimes
    cats = classify_tensors(g)
    spans = tensor_lifetimes(g, s)
    return tuple(LayoutItem(t.id, t.size, spans[t.id][0], spans[t.id][1],
                            cats[t.id] is TensorCategory.ACTIVATION) for t in g.tensors)


def validate_layout(g, s: Schedule, m) -> list[str]:
    """Empty iff the layout is valid for the schedule (layout.py:349-352)."""
    return layout_violations(items_from_schedule(g, s), m.offsets, m.capacity)


def replay_static(g, s: Schedule, m) -> tuple[int, list[str]]:
    """(actual peak extent, violations) (simulator.py:129-145)."""
    from .evaluator import validate_schedule
    validate_schedule(g, s)
    items = items_from_schedule(g, s)
    flags, off, pairs, mx = _k2(items, m.offsets, m.capacity, 1024)
    return int(mx), _messages(items, m.capacity, flags, off, pairs)
