"""Window ordering on the GPU -- drop-ins for the reference's
``memplan.ordering.greedy_order`` / ``exact_order`` plus their batch forms.

  OrderingProblem / OrderingSolution / SolverStats   ordering.py:35-66 (same fields)
  greedy_order(p)          ordering.py:126-180  -> rm_greedy_windows (K4), one window
  greedy_orders(problems)  the planner's _pool_map(_solve_window) over every
                           greedy window (planner.py:155-157) as ONE launch
  exact_order(p)           ordering.py:183-286  -> rm_exact_windows (K5): the
                           order-ideal DP, exact whenever the reference's
                           search cannot reach its node cap
  exact_orders(problems)   every exact window of the planner as ONE launch
"""

from __future__ import annotations

import ctypes as C
import itertools
import time
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import check, lib, ptr
from .graph import ConfigError


@dataclass(frozen=True)
class OrderingProblem:
    graph: object
    ops: tuple[int, ...]
    live_in: frozenset[int] = frozenset()
    live_out: frozenset[int] = frozenset()
    ops_per_step: int = 1
    time_budget: float = 60.0
    node_cap: int | None = None


@dataclass(frozen=True)
class SolverStats:
    nodes: int
    wall_time: float


@dataclass(frozen=True)
class OrderingSolution:
    order: tuple[int, ...]
    peak: int
    optimal: bool
    stats: SolverStats


def _check_problem(p) -> None:
    # _Local's own checks come first (ordering.py:86-89)
    if p.ops_per_step < 1:
        raise ConfigError("ops_per_step must be >= 1")
    if p.time_budget <= 0:
        raise ConfigError("time budget must be positive")


def _window_csr(problems: Sequence, who: str):
    """Device graph + window / live-in / live-out CSR of problems sharing one
    graph.  Entry order within a window is free: libroam sorts the ops and
    treats the tensor lists as sets."""
    from .evaluator import device_graph
    _lib.require_device()
    g = problems[0].graph
    if any(p.graph is not g for p in problems):
        raise ValueError(f"{who}: every problem must share one graph")
    W = len(problems)

    def csr(lists):
        lens = np.fromiter(map(len, lists), np.int64, W)
        p = np.zeros(W + 1, np.int64)
        np.cumsum(lens, out=p[1:])
        arrs = [getattr(x, "arr", None) for x in lists]
        if W and all(a is not None for a in arrs):   # windows.LiveSet: ids already as arrays
            return p, np.concatenate(arrs).astype(np.int32, copy=False)
        idx = np.fromiter(itertools.chain.from_iterable(lists), np.int32, int(p[-1]))
        return p, idx

    return (device_graph(g), csr([p.ops for p in problems]),
            csr([p.live_in for p in problems]), csr([p.live_out for p in problems]))


def greedy_windows(problems: Sequence) -> list[tuple[tuple[int, ...], int] | Exception]:
    """K4 over windows that share one graph: [(order, peak) | exception]."""
    if not problems:
        return []
    dg, (win_ptr, win_ops), (lin_ptr, lin_idx), (lout_ptr, lout_idx) = _window_csr(problems, "greedy_windows")
    W = len(problems)
    order = np.empty(max(len(win_ops), 1), np.int32)
    peak = np.empty(W, np.int64)
    status = np.empty(W, np.int32)
    bad = np.empty(W, np.int32)
    check(lib().rm_greedy_windows(dg.handle, W, ptr(win_ptr), ptr(win_ops), ptr(lin_ptr), ptr(lin_idx),
                                  ptr(lout_ptr), ptr(lout_idx), ptr(order), ptr(peak), ptr(status),
                                  ptr(bad), None), "rm_greedy_windows")
    out: list = []
    for w in range(W):
        if status[w] == 1:
            out.append(ConfigError(f"live-in tensor {int(bad[w])} has no consumer in the window "
                                   f"and is not live-out"))
        elif status[w] == 2:
            out.append(AssertionError("window precedence contains a cycle"))
        else:
            a, b = int(win_ptr[w]), int(win_ptr[w + 1])
            out.append((tuple(order[a:b].tolist()), int(peak[w])))
    return out


def greedy_orders(problems: Sequence, solution_type=OrderingSolution, stats_type=SolverStats) -> list:
    """greedy_order over many windows (grouped per graph, one K4 launch per
    graph).  Raises the first problem's error in problem order, like a
    sequential map would."""
    t0 = time.monotonic()
    for p in problems:
        _check_problem(p)
    res: list = [None] * len(problems)
    groups: dict[int, list[int]] = {}
    for k, p in enumerate(problems):
        groups.setdefault(id(p.graph), []).append(k)
    for idx in groups.values():
        for k, r in zip(idx, greedy_windows([problems[k] for k in idx])):
            res[k] = r
    out = []
    wall = time.monotonic() - t0
    for p, r in zip(problems, res):
        if isinstance(r, Exception):
            raise r
        order, peak = r
        out.append(solution_type(order=order, peak=peak, optimal=False,
                                 stats=stats_type(nodes=len(order), wall_time=wall)))
    return out


def greedy_order(p) -> OrderingSolution:
    """Least-memory-increase list scheduling (ordering.py:126-180) on the GPU;
    always flagged non-optimal."""
    return greedy_orders([p])[0]


# ------------------------------------------------------------------ exact

NEEDS_SEARCH = object()   # rm_exact_windows status 3: the capped DFS (search_window) decides


def exact_windows(problems: Sequence) -> list:
    """K5 over windows that share one graph: per window (order, peak, nodes),
    NEEDS_SEARCH, or the exception the reference raises."""
    if not problems:
        return []
    dg, (win_ptr, win_ops), (lin_ptr, lin_idx), (lout_ptr, lout_idx) = _window_csr(problems, "exact_windows")
    W = len(problems)
    cap = np.array([-1 if p.node_cap is None else int(p.node_cap) for p in problems], np.int64)
    order = np.empty(max(len(win_ops), 1), np.int32)
    peak = np.zeros(W, np.int64)
    nodes = np.zeros(W, np.int64)
    status = np.empty(W, np.int32)
    bad = np.empty(W, np.int32)
    check(lib().rm_exact_windows(dg.handle, W, ptr(win_ptr), ptr(win_ops), ptr(lin_ptr), ptr(lin_idx),
                                 ptr(lout_ptr), ptr(lout_idx), ptr(cap), ptr(order), ptr(peak),
                                 ptr(nodes), ptr(status), ptr(bad), None), "rm_exact_windows")
    out: list = []
    for w in range(W):
        if status[w] == 1:
            out.append(ConfigError(f"live-in tensor {int(bad[w])} has no consumer in the window "
                                   f"and is not live-out"))
        elif status[w] == 2:
            out.append(AssertionError("window precedence contains a cycle"))
        elif status[w] == 3:
            out.append(NEEDS_SEARCH)
        else:
            a, b = int(win_ptr[w]), int(win_ptr[w + 1])
            out.append((tuple(order[a:b].tolist()), int(peak[w]), int(nodes[w])))
    return out


BUDGET = object()   # rm_exact_order_search status 4: the reference returns its greedy incumbent


def search_window(p):
    """exact_order's capped DFS (ordering.py:183-286) on the host in libroam
    (rm_exact_order_search), node for node: (order, peak, nodes), BUDGET when
    the node cap or the deadline stops it, or the exception the reference
    raises.  The deadline is the reference's (t0 + time_budget, monotonic)."""
    from .evaluator import device_graph
    t0 = time.monotonic()
    dg = device_graph(p.graph)
    ops = np.asarray(sorted(p.ops), np.int32)
    lin = np.asarray(sorted(p.live_in), np.int32)
    lout = np.asarray(sorted(p.live_out), np.int32)
    order = np.empty(max(len(ops), 1), np.int32)
    peak, nodes = C.c_int64(0), C.c_int64(0)
    status, bad = C.c_int32(0), C.c_int32(-1)
    check(lib().rm_exact_order_search(dg.handle, len(ops), ptr(ops), len(lin), ptr(lin), len(lout), ptr(lout),
                                      -1 if p.node_cap is None else int(p.node_cap), t0 + p.time_budget,
                                      ptr(order), C.byref(peak), C.byref(nodes), C.byref(status),
                                      C.byref(bad)), "rm_exact_order_search")
    if status.value == 1:
        return ConfigError(f"live-in tensor {bad.value} has no consumer in the window and is not live-out")
    if status.value == 2:
        return AssertionError("window precedence contains a cycle")
    if status.value == 4:
        return BUDGET
    return tuple(order[:len(ops)].tolist()), int(peak.value), int(nodes.value)


def exact_orders(problems: Sequence, solution_type=OrderingSolution, stats_type=SolverStats) -> list:
    """exact_order over many windows (one K5 launch per graph).  Windows whose
    order ideals outnumber their node cap run the reference's capped DFS in
    libroam (``search_window``): its optimum, or -- when the cap stops it --
    the greedy incumbent (K4), flagged non-optimal, as the reference returns.
    ``stats.nodes`` is the DFS's node count for searched windows and the
    number of order ideals minus one for K5's (an upper bound on the
    reference's expansions; the plan documents never contain it)."""
    t0 = time.monotonic()
    for p in problems:
        _check_problem(p)
    res: list = [None] * len(problems)
    groups: dict[int, list[int]] = {}
    for k, p in enumerate(problems):
        groups.setdefault(id(p.graph), []).append(k)
    for idx in groups.values():
        for k, r in zip(idx, exact_windows([problems[k] for k in idx])):
            res[k] = r
    wall = time.monotonic() - t0
    out = []
    for p, r in zip(problems, res):
        if isinstance(r, Exception):
            raise r
        if r is NEEDS_SEARCH:
            r = search_window(p)
            if isinstance(r, Exception):
                raise r
            if r is BUDGET:
                out.append(greedy_orders([p], solution_type, stats_type)[0])
                continue
        order, peak, nodes = r
        out.append(solution_type(order=order, peak=peak, optimal=True,
                                 stats=stats_type(nodes=nodes, wall_time=wall)))
    return out


def exact_order(p) -> OrderingSolution:
    """Minimum-peak window order (ordering.py:183-286): K5 on the GPU, the
    capped DFS in libroam where the node cap can bind (any window width)."""
    return exact_orders([p])[0]
