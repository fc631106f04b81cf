"""Drop-in of the B200 hot path into the reference planner (``memplan``).

The reference has no plugin registry: its planner resolves the hot-path
functions as module globals at call time (planner.py:16-51, simulator.py:15-16,
cli.py:14-40).  ``install()`` rebinds exactly those globals to the GPU
implementations in this package, so the reference's own ``plan(g, cfg)`` /
``compare_baselines`` / ``replay_static`` / CLI run unchanged on top of
libroam; ``uninstall()`` restores the originals.

Dispatch points rebound (reference file:line of the call site):
  planner.peak_memory            planner.py:212    weight-update candidate argmin
  planner.tensor_lifetimes       planner.py:227    layout item lifetimes
  planner.live_bytes_by_timestep planner.py:264    boundary peaks
  planner._pool_map              planner.py:155-157, 250-252  the batch dispatch:
        _solve_window jobs -> every greedy window in ONE K4 launch, every
                              exact window in ONE K5 launch (the reference's
                              exact_order DFS only where its node cap can bind)
        _solve_layout jobs -> every leaf in ONE K3 launch per mode
                              (constrained LLFB for big leaves, exact_layout's
                              incumbent+bound for small ones, its branch-and-
                              bound in libroam where incumbent > bound)
  planner.repair_conflicts       planner.py:259    K2 detection + mover placement
  planner.validate_layout        planner.py:260    K2
  ordering.weight_update_cost    ordering.py:310   event sweep once per (graph, bounds)
  planner/ordering.place_weight_updates  ordering.py:387-467  the branch loop in libroam
                                 C++ (rm_place_weight_updates) over one activation sweep
  ordering.asap_alap             ordering.py:405   C++ closure bitsets (graph.py:365-372)
  segmentation._region_between / _format_ig_ok / linearize (+ planner.linearize,
  ordering.linearize)            segmentation.py:174-201, 500-572: numpy over the
                                 C++ ancestor bit matrix (control.py)
  segmentation.build_subgraph_tree (+ planner's)  segmentation.py:343-448: core,
                                 _mi_over and residual ranks from the same matrix
  graph/segmentation/ordering.weight_update_branches  graph.py:513: once per graph
  graph/planner/ordering/segmentation.classify_tensors  graph.py:471: once per graph
  segmentation.assign_shared_tensors (+ planner's)  segmentation.py:598-639: one
                                 slot pass instead of one per floating op
  planner.build_window_problems  planner.py:141-149 interval stabbing on slot positions
                                                   (windows.py)
  layout.layout_violations / simulator.layout_violations / simulator.peak_memory
  cli.peak_memory / validate_schedule / tensor_lifetimes / validate_layout (memplan eval)
  the user-facing API in its home modules and as memplan's re-exports:
  peak_memory / tensor_lifetimes / live_bytes_by_timestep / asap_alap (graph),
  replay_static (simulator.py:129-145: K2's max-extent epilogue),
  validate_layout / repair_conflicts / llfb_layout / constrained_llfb_layout /
  exact_layout (layout), greedy_order / exact_order (ordering)

Results are bit-identical to the unpatched reference: the plan document bytes
(``plan_doc_bytes``) are the parity artefact (tests/test_gpu_plan.py).
"""

from __future__ import annotations

import functools
import importlib
import sys
import time
from pathlib import Path

from . import control as _ctl
from . import evaluator as _ev
from . import layout as _lay
from . import ordering as _ord
from . import windows as _win
from ._lib import RoamError
from .graph import GraphError

ROOT = Path(__file__).resolve().parents[1]


def load_memplan():
    """Import the reference package: an installed ``memplan`` or the copy the
    driver installs under baseline/_ref (pip --target)."""
    try:
        return importlib.import_module("memplan")
    except ImportError:
        ref = ROOT / "baseline" / "_ref"
        if (ref / "memplan").is_dir() and str(ref) not in sys.path:
            sys.path.insert(0, str(ref))
        return importlib.import_module("memplan")


def _translate(mp, fn):
    """Re-raise this package's errors as the reference's classes (same names,
    same messages), so callers' except clauses keep working."""

    @functools.wraps(fn)
    def wrapper(*a, **k):
        try:
            return fn(*a, **k)
        except GraphError as e:
            cls = getattr(mp.graph, type(e).__name__, None)
            if cls is None:
                raise
            raise cls(str(e)) from None
    return wrapper


def _raise(e):
    raise e


def _asap_alap_factory(mp):
    """graph.py:365-372 asap_alap (called by place_weight_updates,
    ordering.py:405) from libroam's C++ closure bitsets.  A cycle raises the
    reference's StructuralError (graph.py:133-134); graphs above libroam's
    closure limit (60k ops) raise RoamError -- there is no fallback."""

    def asap_alap(g):
        try:
            asap, alap = _ev.asap_alap(g)
        except RoamError as e:
            if "cycle" in str(e):
                raise mp.graph.StructuralError("graph contains a cycle") from None
            raise
        return mp.graph.ScheduleBounds(asap=asap, alap=alap)
    return asap_alap


class _State:
    installed = None  # (memplan module, {(module, name): original})


# dispatch counters since install(): how the planner's subtasks were served
# (every one by libroam: there is no reference fallback)
STATS = {"windows_k4": 0, "windows_k5": 0, "windows_dfs": 0, "windows_dfs_budget": 0,
         "leaves_k3_constrained": 0, "leaves_k3_exact": 0, "leaves_search": 0}


def install(mp=None):
    """Rebind the reference's hot-path globals to libroam; idempotent."""
    mp = mp or load_memplan()
    if _State.installed is not None:
        return mp
    for k in STATS:
        STATS[k] = 0
    pl, lay, sim, gr, ordm = mp.planner, mp.layout, mp.simulator, mp.graph, mp.ordering
    orig_solve_window = pl._solve_window
    orig_solve_layout = pl._solve_layout
    orig_pool_map = pl._pool_map

    def to_layout(m):
        return lay.MemoryLayout(offsets=m.offsets, capacity=m.capacity,
                                activation_block=m.activation_block, optimal=m.optimal,
                                stats=lay.LayoutStats(m.stats.nodes, m.stats.wall_time))

    def solve_windows(jobs):
        """Every greedy window in one K4 launch and every exact window in one
        K5 launch; a window with more order ideals than its node cap runs the
        reference's capped DFS restated in libroam (its answer depends on where
        that search stops).  Errors surface in job order, as the sequential map
        raises them."""
        greedy = [k for k, (p, limit) in enumerate(jobs) if len(p.ops) > limit]
        exact = [k for k, (p, limit) in enumerate(jobs) if len(p.ops) <= limit]
        exact_keys = set(exact)
        res = [None] * len(jobs)
        for idx, batch in ((greedy, _ord.greedy_windows), (exact, _ord.exact_windows)):
            groups = {}
            for k in idx:
                groups.setdefault(id(jobs[k][0].graph), []).append(k)
            for ks in groups.values():
                for k, r in zip(ks, batch([jobs[k][0] for k in ks])):
                    res[k] = r
        out = []
        check_problem = T(_ord._check_problem)   # wrap once, not per window
        for k, ((p, limit), r) in enumerate(zip(jobs, res)):
            check_problem(p)
            if isinstance(r, GraphError):
                T(functools.partial(_raise, r))()
            if isinstance(r, Exception):
                raise r
            if r is _ord.NEEDS_SEARCH:
                # more order ideals than the node cap: the capped DFS in libroam
                # (multi-word masks: windows of any node_limit)
                r = _ord.search_window(p)
                if isinstance(r, GraphError):
                    T(functools.partial(_raise, r))()
                if isinstance(r, Exception):
                    raise r
                if r is _ord.BUDGET:   # the reference returns its greedy incumbent
                    out.append(_ord.greedy_orders([p], ordm.OrderingSolution, ordm.SolverStats)[0])
                    STATS["windows_dfs_budget"] += 1
                else:
                    order, peak, nodes = r
                    out.append(ordm.OrderingSolution(order=order, peak=peak, optimal=True,
                                                      stats=ordm.SolverStats(nodes, 0.0)))
                    STATS["windows_dfs"] += 1
            elif k in exact_keys:
                order, peak, nodes = r
                out.append(ordm.OrderingSolution(order=order, peak=peak, optimal=True,
                                                  stats=ordm.SolverStats(nodes, 0.0)))
                STATS["windows_k5"] += 1
            else:
                order, peak = r
                out.append(ordm.OrderingSolution(order=order, peak=peak, optimal=False,
                                                  stats=ordm.SolverStats(len(order), 0.0)))
                STATS["windows_k4"] += 1
        return out

    def solve_layouts(jobs):
        out = [None] * len(jobs)
        big = [k for k, (p, limit) in enumerate(jobs) if len(p.items) > limit]
        small = [k for k, (p, limit) in enumerate(jobs) if len(p.items) <= limit]
        t0 = time.monotonic()
        if big:
            res = _lay.pack_batch([jobs[k][0].items for k in big], _lay.CONSTRAINED)
            wall = time.monotonic() - t0
            STATS["leaves_k3_constrained"] += len(big)
            for k, r in zip(big, res):
                p = jobs[k][0]
                out[k] = lay.MemoryLayout(offsets=r.offsets, capacity=r.capacity,
                                          activation_block=_lay._act_block(p.items), optimal=False,
                                          stats=lay.LayoutStats(len(p.items), wall))
        if small:
            for p in (jobs[k][0] for k in small):
                if p.time_budget <= 0:
                    raise gr.ConfigError("time budget must be positive")
            # K3 decides the leaves whose incumbents meet their bounds; the
            # others run the branch-and-bound in libroam (rm_layout_search)
            res = _lay.exact_layout_batch([jobs[k][0] for k in small])
            for k, r in zip(small, res):
                out[k] = to_layout(r)
                STATS["leaves_search" if r.stats.nodes else "leaves_k3_exact"] += 1
        return out

    def pool_map(fn, jobs, workers):
        jobs = list(jobs)
        if fn is orig_solve_window:
            return solve_windows(jobs)
        if fn is orig_solve_layout:
            return solve_layouts(jobs)
        return orig_pool_map(fn, jobs, workers)

    T = functools.partial(_translate, mp)

    def build_window_problems(g, lin, wu_plan=None, ops_per_step=1, time_budget=60.0, node_cap=None):
        return _win.build_window_problems(g, lin, wu_plan, ops_per_step, time_budget, node_cap,
                                          window_type=mp.segmentation.Window,
                                          problem_type=ordm.OrderingProblem)

    fast_linearize = _ctl.linearize_factory(mp)
    fast_tree = _ctl.subgraph_tree_factory(mp)
    fast_segments, fast_segment_tree = _ctl.segment_tree_factory(mp)
    wu_branches = _ctl.weight_update_branches_factory(mp)
    fast_assign = _ctl.assign_shared_tensors_factory(mp)
    cats = _ctl.classify_tensors_factory(mp)
    patches = {
        (mp.segmentation, "build_subgraph_tree"): fast_tree,
        (gr, "classify_tensors"): cats,
        (pl, "classify_tensors"): cats,
        (ordm, "classify_tensors"): cats,
        (mp.segmentation, "classify_tensors"): cats,
        (mp.segmentation, "assign_shared_tensors"): fast_assign,
        (pl, "assign_shared_tensors"): fast_assign,
        (pl, "build_subgraph_tree"): fast_tree,
        (mp.segmentation, "independent_segments"): fast_segments,
        (mp.segmentation, "build_segment_tree"): fast_segment_tree,
        (pl, "build_segment_tree"): fast_segment_tree,
        (gr, "weight_update_branches"): wu_branches,
        (mp.segmentation, "weight_update_branches"): wu_branches,
        (ordm, "weight_update_branches"): wu_branches,
        (mp.segmentation, "linearize"): fast_linearize,
        (pl, "linearize"): fast_linearize,
        (ordm, "linearize"): fast_linearize,
        (pl, "build_window_problems"): build_window_problems,
        (ordm, "weight_update_cost"): _weight_update_cost_factory(mp),
        (ordm, "place_weight_updates"): T(_ctl.place_weight_updates_factory(mp)),
        (pl, "place_weight_updates"): T(_ctl.place_weight_updates_factory(mp)),
        (ordm, "asap_alap"): _asap_alap_factory(mp),
        (mp.segmentation, "_region_between"): _ctl.region_between_factory(),
        (mp.segmentation, "_format_ig_ok"): _ctl.format_ig_ok_factory(mp),
        (pl, "peak_memory"): T(_ev.peak_memory),
        (pl, "tensor_lifetimes"): T(_ev.tensor_lifetimes),
        (pl, "live_bytes_by_timestep"): T(_ev.live_bytes_by_timestep),
        (pl, "_pool_map"): pool_map,
        (pl, "repair_conflicts"): T(_lay.repair_conflicts),
        (pl, "validate_layout"): T(_lay.validate_layout),
        (lay, "layout_violations"): T(_lay.layout_violations),
        (sim, "layout_violations"): T(_lay.layout_violations),
        (sim, "peak_memory"): T(_ev.peak_memory),
    }
    # the user-facing API: the same functions in their home modules and as
    # the package's re-exports (memplan/__init__.py), results in the
    # reference's own types
    def as_ref_layout(fn):
        return T(lambda p: to_layout(fn(p)))

    def as_ref_order(batch):
        return T(lambda p: batch([p], ordm.OrderingSolution, ordm.SolverStats)[0])

    api = {
        "peak_memory": (gr, T(_ev.peak_memory)),
        "tensor_lifetimes": (gr, T(_ev.tensor_lifetimes)),
        "live_bytes_by_timestep": (gr, T(_ev.live_bytes_by_timestep)),
        "replay_static": (sim, T(_lay.replay_static)),
        "validate_layout": (lay, T(_lay.validate_layout)),
        "repair_conflicts": (lay, T(_lay.repair_conflicts)),
        "llfb_layout": (lay, as_ref_layout(_lay.llfb_layout)),
        "constrained_llfb_layout": (lay, as_ref_layout(_lay.constrained_llfb_layout)),
        "exact_layout": (lay, as_ref_layout(_lay.exact_layout)),
        "greedy_order": (ordm, as_ref_order(_ord.greedy_orders)),
        "exact_order": (ordm, as_ref_order(_ord.exact_orders)),
        "asap_alap": (gr, patches[(ordm, "asap_alap")]),
        "independent_segments": (mp.segmentation, fast_segments),
    }
    for name, (home, fn) in api.items():
        patches.setdefault((home, name), fn)
        if hasattr(mp, name):
            patches[(mp, name)] = fn
    try:  # the CLI binds its own names at import (cli.py:14-40)
        cli = importlib.import_module(mp.__name__ + ".cli")
        patches.update({
            (cli, "peak_memory"): T(_ev.peak_memory),
            (cli, "validate_schedule"): T(_ev.validate_schedule),
            (cli, "tensor_lifetimes"): T(_ev.tensor_lifetimes),
            (cli, "validate_layout"): T(_lay.validate_layout),
        })
    except ImportError:
        pass
    saved = {}
    for (mod, name), fn in patches.items():
        saved[(mod, name)] = getattr(mod, name)
        setattr(mod, name, fn)
    _State.installed = (mp, saved)
    return mp


def _weight_update_cost_factory(mp):
    """Drop-in for ordering.weight_update_cost (ordering.py:310-338).

    The reference rescans every tensor for each (branch, timestep) query --
    1,162 queries x 7k tensors at GPT2-XL, 78 % of the planner's time once the
    hot path runs on the GPU.  Activations alive at t are those with
    asap(producer) <= t <= max alap(consumers) (horizon n-1 without
    consumers): one +size/-size event sweep per (graph, bounds) turns every
    query into a lookup.  Integer sums, same float expression for
    projected_use, so results are identical."""
    import weakref

    import numpy as np
    gr, ordm = mp.graph, mp.ordering
    cache: dict = {}

    def table(g, bounds):
        key = (id(g), id(bounds))
        ent = cache.get(key)
        if ent is not None and ent[0]() is g and ent[1]() is bounds:
            return ent[2], ent[3]
        cats = gr.classify_tensors(g)
        n = g.n_ops
        act = [t for t in g.tensors if cats[t.id] is gr.TensorCategory.ACTIVATION]
        total = sum(t.size for t in act)
        diff = np.zeros(n + 1, dtype=object if total >= 2**62 else np.int64)
        for t in act:
            start = bounds.asap[t.producer]
            end = max((bounds.alap[c] for c in t.consumers), default=n - 1)
            if start <= end:
                diff[start] += t.size
                diff[end + 1] -= t.size
        alive = np.cumsum(diff)[:n].tolist()
        cache[key] = (weakref.ref(g), weakref.ref(bounds), total, alive)
        weakref.finalize(g, cache.pop, key, None)
        return total, alive

    def weight_update_cost(g, bounds, t, branch, alpha=None):
        total, alive_at = table(g, bounds)
        alive = alive_at[t] if 0 <= t < len(alive_at) else 0
        a = ordm.resolve_alpha(g, branch, ordm.DEFAULT_ALPHA if alpha is None else alpha)
        projected = alive + a * branch.grad_bytes
        return total, alive, projected

    return weight_update_cost


def uninstall() -> None:
    if _State.installed is None:
        return
    _, saved = _State.installed
    for (mod, name), fn in saved.items():
        setattr(mod, name, fn)
    _State.installed = None


def plan(g, cfg=None):
    """The reference's ``plan(g, cfg)`` (planner.py:180) with the B200 hot path
    installed; returns the reference's ExecutionPlan."""
    mp = install()
    return mp.planner.plan(g, cfg)
