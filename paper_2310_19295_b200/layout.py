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
  exact_layout           layout.py:153-302   -> rm_llfb_batch COMPONENTS (K3; the
                                              search only if incumbent > bound)
  pack_batch             planner.py:250-252 batch dispatch (_pool_map of _solve_layout)
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from . import _lib
from ._lib import RM_ERR_GRAPH, check, lib, ptr
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


# ------------------------------------------------------ K3: batched packer

PLAIN, CONSTRAINED, COMPONENTS, COMPONENTS_FREE = (_lib.RM_LLFB_PLAIN, _lib.RM_LLFB_CONSTRAINED,
                                                   _lib.RM_LLFB_COMPONENTS, 3)


@dataclass(frozen=True)
class PackResult:
    """One problem's K3 output: offsets by tensor id, capacity, and for the
    component modes whether every component's incumbent met its bound."""
    offsets: dict[int, int]
    capacity: int
    bound_met: bool = True
    comp_cap: dict[int, int] = field(default_factory=dict)  # component root -> incumbent cap


def set_pack_form(form: int) -> None:
    """K3 placement form on this thread: 0 auto (DAG rounds for problems of
    1,024+ items), 1 the placed-list path only, 2 DAG rounds wherever they
    qualify (rm_set_pack_form).  Same offsets either way."""
    check(lib().rm_set_pack_form(int(form)), "rm_set_pack_form")


def pack_batch(problems: Sequence[Sequence], mode: int) -> list[PackResult]:
    """Run K3 over many independent item lists in ONE launch (one CTA per
    problem): the batch form of the planner's ``_pool_map(_solve_layout)``
    (planner.py:250-252)."""
    _lib.require_device()
    P = len(problems)
    if P == 0:
        return []
    counts = np.fromiter((len(p) for p in problems), np.int64, P)
    item_ptr = np.zeros(P + 1, np.int64)
    np.cumsum(counts, out=item_ptr[1:])
    flat = [it for p in problems for it in p]
    NI = len(flat)
    start, end, size = _item_arrays(flat)
    tensor = np.fromiter((i.tensor for i in flat), np.int64, NI)
    if NI and (tensor.min() < 0 or tensor.max() >= 2**31):
        raise ValueError("tensor ids must fit int32")
    tensor = tensor.astype(np.int32)
    is_act = np.fromiter((bool(i.is_activation) for i in flat), np.uint8, NI)
    offset = np.empty(max(NI, 1), np.int64)
    cap = np.empty(P, np.int64)
    comps = mode in (COMPONENTS, COMPONENTS_FREE)
    met = np.ones(P, np.uint8) if comps else None
    comp = np.empty(max(NI, 1), np.int32) if comps else None
    ccap = np.empty(max(NI, 1), np.int64) if comps else None
    check(lib().rm_llfb_batch(P, ptr(item_ptr), ptr(tensor), ptr(start), ptr(end), ptr(size),
                              ptr(is_act), int(mode), ptr(offset), ptr(cap), ptr(met), ptr(comp),
                              ptr(ccap), None), "rm_llfb_batch")
    out = []
    off_l, ten_l = offset[:NI].tolist(), tensor.tolist()
    for p in range(P):
        a, b = int(item_ptr[p]), int(item_ptr[p + 1])
        offs = dict(zip(ten_l[a:b], off_l[a:b]))
        if comps:
            cc = {int(r): int(c) for r, c in zip(comp[a:b].tolist(), ccap[a:b].tolist()) if r >= 0}
            out.append(PackResult(offs, int(cap[p]), bool(met[p]), cc))
        else:
            out.append(PackResult(offs, int(cap[p])))
    return out


def _act_block(items) -> int:
    return sum(i.size for i in items if i.is_activation)


def llfb_layout(p) -> MemoryLayout:
    """Long-lived-first best fit (layout.py:100-118) on the GPU (K3 PLAIN)."""
    t0 = time.monotonic()
    r = pack_batch([p.items], PLAIN)[0]
    return MemoryLayout(offsets=r.offsets, capacity=r.capacity, activation_block=_act_block(p.items),
                        optimal=False, stats=LayoutStats(len(p.items), time.monotonic() - t0))


def constrained_llfb_layout(p) -> MemoryLayout:
    """Long-lived-first fallback keeping the activation block at the bottom
    (layout.py:121-146) on the GPU (K3 CONSTRAINED)."""
    t0 = time.monotonic()
    r = pack_batch([p.items], CONSTRAINED)[0]
    return MemoryLayout(offsets=r.offsets, capacity=r.capacity, activation_block=_act_block(p.items),
                        optimal=False, stats=LayoutStats(len(p.items), time.monotonic() - t0))


def exact_layout(p) -> MemoryLayout:
    """exact_layout (layout.py:153-302): K3 decides every problem whose overlap
    components' long-lived-first incumbents meet their lower bounds (then the
    reference returns that incumbent without search, and so does this); the
    other components run the reference's branch-and-bound node for node in
    libroam (``rm_layout_search``, masks of up to 256 words: components of
    any size the planner forms)."""
    if p.time_budget <= 0:
        from .graph import ConfigError
        raise ConfigError("time budget must be positive")
    if not p.items:
        return MemoryLayout(offsets={}, capacity=0, stats=LayoutStats(0, 0.0))
    return exact_layout_batch([p])[0]


def exact_layout_batch(problems: Sequence, search: bool = True) -> list[MemoryLayout | None]:
    """K3 component pass over many exact_layout problems in one launch, then
    the branch-and-bound (rm_layout_search) for the problems whose incumbent
    missed its bound (None for those when ``search`` is False: the K3 pass
    alone, for tests)."""
    t0 = time.monotonic()
    out: list[MemoryLayout | None] = [None] * len(problems)
    for bottom in (True, False):
        idx = [k for k, p in enumerate(problems) if bool(p.activations_at_bottom) == bottom]
        if not idx:
            continue
        res = pack_batch([problems[k].items for k in idx], COMPONENTS if bottom else COMPONENTS_FREE)
        for k, r in zip(idx, res):
            p = problems[k]
            if not p.items:
                out[k] = MemoryLayout(offsets={}, capacity=0, stats=LayoutStats(0, 0.0))
            elif r.bound_met:
                out[k] = MemoryLayout(offsets=r.offsets, capacity=r.capacity,
                                      activation_block=_act_block(p.items), optimal=True,
                                      stats=LayoutStats(0, time.monotonic() - t0))
            elif search:
                out[k] = _branch_and_bound(p, r, t0)
    return out


def _branch_and_bound(p, r: PackResult, t0: float) -> MemoryLayout:
    """layout.py:226-290 over K3's incumbent: one rm_layout_search call.  The
    deadline is the reference's (t0 + time_budget on the monotonic clock)."""
    items = p.items
    N = len(items)
    start, end, size = _item_arrays(items)
    tensor = np.fromiter((i.tensor for i in items), np.int64, N).astype(np.int32)
    is_act = np.fromiter((bool(i.is_activation) for i in items), np.uint8, N)
    inc = np.fromiter((r.offsets[i.tensor] for i in items), np.int64, N)
    offset = np.empty(N, np.int64)
    cap, nodes, opt = C.c_int64(0), C.c_int64(0), C.c_int32(0)
    check(lib().rm_layout_search(N, ptr(tensor), ptr(start), ptr(end), ptr(size), ptr(is_act),
                                 1 if p.activations_at_bottom else 0, ptr(inc),
                                 -1 if p.node_cap is None else int(p.node_cap), t0 + p.time_budget,
                                 ptr(offset), C.byref(cap), C.byref(nodes), C.byref(opt)),
          "rm_layout_search")
    return MemoryLayout(offsets=dict(zip(tensor.tolist(), offset.tolist())), capacity=int(cap.value),
                        activation_block=_act_block(items), optimal=bool(opt.value),
                        stats=LayoutStats(int(nodes.value), time.monotonic() - t0))


# --------------------------------------------------------- conflict repair

def repair_conflicts(m, p):
    """Re-place the smaller, shorter-lived member of every conflicting pair
    (layout.py:409-470) in one libroam call (rm_repair_conflicts): per round
    the device tests every item pair for time x address overlap with the
    items resident and flags each pair's elected mover (K2's tiled geometry;
    91.5 s of 279 s at 10.8k ops in the reference); the host C++ places the
    movers (best-fit gap, strict < on gap size so the lowest-addressed
    smallest gap wins).  Returns ``dataclasses.replace(m, ...)`` so the
    caller's layout type is preserved."""
    from dataclasses import replace

    from .graph import StructuralError
    items = sorted(p.items, key=lambda i: i.tensor)
    offsets = dict(m.offsets)
    N = len(items)
    for it in items:                      # layout.py:424-426 reads every offset
        if it.tensor not in offsets:
            raise KeyError(it.tensor)
    if N < 2:
        return replace(m, offsets=offsets, capacity=m.capacity)
    _lib.require_device()
    tid = np.fromiter((i.tensor for i in items), np.int64, N)
    st, en, sz = _item_arrays(items)
    act = np.fromiter((bool(i.is_activation) for i in items), np.uint8, N)
    off = np.fromiter((offsets[t] for t in tid.tolist()), np.int64, N)
    before = off.copy()
    cap = C.c_int64(int(m.capacity))
    rounds = C.c_int32(0)
    rc = lib().rm_repair_conflicts(N, ptr(tid), ptr(st), ptr(en), ptr(sz), ptr(act), ptr(off),
                                   C.byref(cap), C.byref(rounds), None)
    if rc == RM_ERR_GRAPH:
        raise StructuralError("conflict repair did not converge")
    check(rc, "rm_repair_conflicts")
    for k in np.flatnonzero(off != before).tolist():
        offsets[int(tid[k])] = int(off[k])
    return replace(m, offsets=offsets, capacity=int(cap.value))
