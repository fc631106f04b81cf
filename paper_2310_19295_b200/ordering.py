"""Window greedy ordering on the GPU -- drop-in for the reference's
``memplan.ordering.greedy_order`` plus its batch form.

  OrderingProblem / OrderingSolution / SolverStats   ordering.py:35-66 (same fields)
  greedy_order(p)          ordering.py:126-180  -> rm_greedy_windows (K4), one window
  greedy_orders(problems)  the planner's _pool_map(_solve_window) over every
                           greedy window (planner.py:155-157) as ONE launch
"""

from __future__ import annotations

import ctypes as C
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


def greedy_windows(problems: Sequence) -> list[tuple[tuple[int, ...], int] | Exception]:
    """K4 over windows that share one graph: [(order, peak) | exception]."""
    if not problems:
        return []
    from .evaluator import device_graph
    _lib.require_device()
    g = problems[0].graph
    if any(p.graph is not g for p in problems):
        raise ValueError("greedy_windows: every problem must share one graph")
    dg = device_graph(g)
    W = len(problems)

    def csr(lists):
        lens = np.fromiter((len(x) for x in lists), np.int64, W)
        p = np.zeros(W + 1, np.int64)
        np.cumsum(lens, out=p[1:])
        idx = np.fromiter((v for x in lists for v in x), np.int64, int(p[-1]))
        return p, idx.astype(np.int32)

    win_ptr, win_ops = csr([sorted(p.ops) for p in problems])
    lin_ptr, lin_idx = csr([sorted(p.live_in) for p in problems])
    lout_ptr, lout_idx = csr([sorted(p.live_out) for p in problems])
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
