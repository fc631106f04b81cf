"""Host-side drop-in plumbing (no GPU): the plugin rebinds exactly the
reference's hot-path module globals and restores them."""

from __future__ import annotations

import pytest

from paper_2310_19295_b200 import memplan_plugin as plug

try:
    mp = plug.load_memplan()
except ImportError:  # pragma: no cover
    mp = None


@pytest.mark.skipif(mp is None, reason="reference memplan not importable")
def test_install_uninstall_roundtrip():
    names = [(mp.planner, n) for n in ("peak_memory", "tensor_lifetimes", "live_bytes_by_timestep",
                                       "_pool_map", "repair_conflicts", "validate_layout")]
    names += [(mp.layout, "layout_violations"), (mp.simulator, "layout_violations"),
              (mp.segmentation, "build_subgraph_tree"), (mp.planner, "build_subgraph_tree"),
              (mp.ordering, "weight_update_branches"), (mp.planner, "assign_shared_tensors"),
              (mp.planner, "classify_tensors"), (mp.graph, "classify_tensors"),
              (mp.ordering, "weight_update_cost"), (mp.ordering, "asap_alap"),
              (mp.planner, "build_window_problems"), (mp.planner, "place_weight_updates"),
              (mp.ordering, "place_weight_updates"),
              (mp.simulator, "peak_memory")]
    before = {k: getattr(*k) for k in names}
    plug.install(mp)
    try:
        for k in names:
            assert getattr(*k) is not before[k], k
        plug.install(mp)  # idempotent
    finally:
        plug.uninstall()
    for k in names:
        assert getattr(*k) is before[k], k


@pytest.mark.skipif(mp is None, reason="reference memplan not importable")
def test_errors_translate_to_reference_classes():
    from paper_2310_19295_b200.graph import ScheduleError
    def boom():
        raise ScheduleError("schedule must contain every op exactly once")
    w = plug._translate(mp, boom)
    with pytest.raises(mp.graph.ScheduleError, match="exactly once"):
        w()


@pytest.mark.skipif(mp is None, reason="reference memplan not importable")
def test_repair_mover_placement_matches_reference():
    """repair_conflicts' mover placement (rm_repair_place, host C++ in
    libroam) against the reference: the rounds are driven here with the
    oracle's pair predicate and mover election standing in for the device
    detection (no GPU), placement goes through the C ABI."""
    import ctypes as C
    import random

    import numpy as np

    from oracle import memplan_oracle as O
    from paper_2310_19295_b200._lib import check, lib, ptr

    def repair(m, p):
        items = sorted(p.items, key=lambda i: i.tensor)
        rows = [(i.tensor, i.size, i.start, i.end, i.is_activation) for i in items]
        N = len(rows)
        st = np.array([r[2] for r in rows], np.int32)
        en = np.array([r[3] for r in rows], np.int32)
        sz = np.array([r[1] for r in rows], np.int64)
        off = np.array([m.offsets[r[0]] for r in rows], np.int64)
        has = np.ones(N, np.uint8)
        cap = C.c_int64(m.capacity)

        def pairs():
            return [(a, b) for a in range(N) for b in range(a + 1, N)
                    if O.overlaps(rows[a], rows[b]) and off[a] < off[b] + sz[b] and off[b] < off[a] + sz[a]]

        def mover(a, b):
            if rows[a][4] != rows[b][4]:
                return b if rows[a][4] else a
            ka = (sz[a], en[a] - st[a], -rows[a][0])
            kb = (sz[b], en[b] - st[b], -rows[b][0])
            return a if ka < kb else b

        for _ in range(N + 1):
            ps = pairs()
            if not ps:
                break
            mv = np.array(sorted({mover(a, b) for a, b in ps},
                                 key=lambda k: (sz[k], en[k] - st[k], rows[k][0])), np.int64)
            check(lib().rm_repair_place(N, ptr(st), ptr(en), ptr(sz), ptr(has), ptr(off), C.byref(cap),
                                        len(mv), ptr(mv)), "rm_repair_place")
        assert not pairs()
        offs = dict(m.offsets)
        offs.update({r[0]: int(o) for r, o in zip(rows, off)})
        return offs, cap.value

    rng = random.Random(11)
    for trial in range(150):
        n = rng.randint(1, 40)
        items = []
        for t in rng.sample(range(100), n):
            s = rng.randint(0, 15)
            items.append(mp.layout.LayoutItem(t, rng.choice([0, 1, 2, 4, 8, 16]), s,
                                              s + rng.randint(0, 6), rng.random() < 0.3))
        offs = {i.tensor: rng.choice([0, 1, 2, 4, 8, 12, 16, 24]) for i in items}
        cap = max(offs[i.tensor] + i.size for i in items) + rng.choice([0, 0, 5])
        m = mp.layout.MemoryLayout(offsets=offs, capacity=cap)
        p = mp.layout.LayoutProblem(items=tuple(items))
        want = mp.layout.repair_conflicts(m, p)
        got_offs, got_cap = repair(m, p)
        assert (got_offs, got_cap) == (want.offsets, want.capacity), trial


@pytest.mark.skipif(mp is None, reason="reference memplan not importable")
def test_weight_update_cost_sweep_matches_reference(monkeypatch):
    """The event-sweep weight_update_cost answers every query the reference
    planner makes exactly like the reference (host code, no GPU)."""
    import memplan.graphgen as rgen

    from paper_2310_19295_b200 import graphgen as gg
    fast = plug._weight_update_cost_factory(mp)
    orig = mp.ordering.weight_update_cost
    seen = []

    def both(g, bounds, t, branch, alpha=None):
        a, b = orig(g, bounds, t, branch, alpha), fast(g, bounds, t, branch, alpha)
        assert a == b and type(a[1]) is type(b[1])
        seen.append(t)
        return a

    monkeypatch.setattr(mp.ordering, "weight_update_cost", both)
    mp.planner.plan(mp.graph.load_graph(gg.config_doc("gpt2-small")))
    for arch in ("mlp", "residual", "transformer_block"):
        for opt in ("sgd", "adam"):
            mp.planner.plan(rgen.gen_training_graph(arch, 3, optimizer=opt))
    assert len(seen) > 100


@pytest.mark.skipif(mp is None, reason="reference memplan not importable")
def test_window_problems_interval_rule_matches_reference(monkeypatch):
    """build_window_problems as interval stabbing (windows.py) returns the
    reference's windows and live-in / live-out sets for every call the planner
    makes (host code, no GPU)."""
    import memplan.graphgen as rgen

    from paper_2310_19295_b200 import graphgen as gg
    from paper_2310_19295_b200 import windows as W
    orig = mp.planner.build_window_problems
    n_calls = []

    def both(g, lin, wu_plan=None, ops_per_step=1, time_budget=60.0, node_cap=None):
        want = orig(g, lin, wu_plan, ops_per_step, time_budget, node_cap)
        got = W.build_window_problems(g, lin, wu_plan, ops_per_step, time_budget, node_cap,
                                      window_type=mp.segmentation.Window,
                                      problem_type=mp.ordering.OrderingProblem)
        assert got == want
        n_calls.append(len(want))
        return want

    monkeypatch.setattr(mp.planner, "build_window_problems", both)
    for name in ("layered", "gpt2-small"):
        mp.planner.plan(mp.graph.load_graph(gg.config_doc(name)))
    for arch in ("mlp", "residual", "transformer_block"):
        for opt in ("sgd", "adam"):
            mp.planner.plan(rgen.gen_training_graph(arch, 4, optimizer=opt))
    assert sum(n_calls) > 20


@pytest.mark.skipif(mp is None, reason="reference memplan not importable")
def test_asap_alap_matches_reference():
    """graph.py:365-372 from libroam's C++ closure bitsets (host-only)."""
    rg = mp.graph
    gen_random_dag, gen_training_graph = mp.graphgen.gen_random_dag, mp.graphgen.gen_training_graph
    from paper_2310_19295_b200 import evaluator as ev
    from paper_2310_19295_b200 import graphgen as gg
    graphs = [rg.load_graph(gg.config_doc(name)) for name in ("layered", "gpt2-small")]
    graphs += [gen_random_dag(5 + k, density=0.1 + 0.05 * (k % 6), seed=40 + k) for k in range(20)]
    graphs += [gen_training_graph("transformer_block", 3, optimizer="adam")]
    for g in graphs:
        want = rg.asap_alap(g)
        asap, alap = ev.asap_alap(g)
        assert (asap, alap) == (want.asap, want.alap)


@pytest.mark.skipif(mp is None, reason="reference memplan not importable")
def test_control_plane_dropins_match_reference():
    """control.py restatements == the reference functions on the subgraph
    trees of training graphs (every _region_between / _format_ig_ok call the
    tree build makes, and linearize) -- host-only."""
    from paper_2310_19295_b200 import control
    seg = mp.segmentation
    ref_rb, ref_ok, ref_lin = seg._region_between, seg._format_ig_ok, seg.linearize
    fast_rb = control.region_between_factory()
    fast_ok = control.format_ig_ok_factory(mp)
    fast_lin = control.linearize_factory(mp)
    calls = {"rb": 0, "ok": 0}

    def rb(build, core, lo, hi):
        calls["rb"] += 1
        want = ref_rb(build, core, lo, hi)
        assert fast_rb(build, core, lo, hi) == want
        return want

    def ok(build, members, boundary):
        calls["ok"] += 1
        want = ref_ok(build, members, boundary)
        assert fast_ok(build, members, boundary) == want
        return want

    seg._region_between, seg._format_ig_ok = rb, ok
    try:
        for arch, blocks, opt in (("transformer_block", 4, "adam"), ("mlp", 3, "sgd"),
                                  ("residual", 5, "adam"), ("transformer_block", 12, "adam")):
            g = mp.graphgen.gen_training_graph(arch, blocks, optimizer=opt)
            for limit in (6, 20):
                tree = seg.build_subgraph_tree(g, limit)
                assert fast_lin(g, tree) == ref_lin(g, tree)
    finally:
        seg._region_between, seg._format_ig_ok = ref_rb, ref_ok
    assert calls["rb"] > 20 and calls["ok"] > 5


def _tree_key(node):
    return (node.id, node.kind, node.outer_fwd, node.inner_fwd, node.inner_bwd, node.outer_bwd,
            node.members, node.owned_tensors, node.unsplittable, node.tag, node.floating_ops,
            node.pinned_ops, tuple(_tree_key(c) for c in node.children))


@pytest.mark.skipif(mp is None, reason="reference memplan not importable")
def test_subgraph_tree_dropin_matches_reference():
    """build_subgraph_tree over the C++ ancestor matrix returns the reference's
    tree node for node (ids, boundaries, members, split flags) on the config
    graphs and the reference's own generators, across node limits; the
    weight-update-branch and linearize caches hand out equal, independent
    results (host-only)."""
    import memplan.graphgen  # noqa: F401  (mp.graphgen)

    from paper_2310_19295_b200 import control
    from paper_2310_19295_b200 import graphgen as gg
    seg = mp.segmentation
    ref_tree, ref_lin, ref_wu = seg.build_subgraph_tree, seg.linearize, mp.graph.weight_update_branches
    fast_tree = control.subgraph_tree_factory(mp)
    fast_lin = control.linearize_factory(mp)
    fast_wu = control.weight_update_branches_factory(mp)
    ref_assign, fast_assign = seg.assign_shared_tensors, control.assign_shared_tensors_factory(mp)
    graphs = [mp.graph.load_graph(gg.config_doc(name)) for name in ("gpt2-small", "bert-large")]
    for arch, blocks, opt in (("transformer_block", 6, "adam"), ("mlp", 5, "sgd"),
                              ("residual", 7, "adam"), ("transformer_block", 1, "sgd")):
        graphs.append(mp.graphgen.gen_training_graph(arch, blocks, optimizer=opt))
    fast_cats = control.classify_tensors_factory(mp)
    for g in graphs:
        assert fast_wu(g) == ref_wu(g) and fast_wu(g) is not fast_wu(g)
        assert fast_cats(g) == mp.graph.classify_tensors(g) and fast_cats(g) is not fast_cats(g)
        for limit in (2, 7, 20, 10**6):
            want = ref_tree(g, limit)
            got = fast_tree(g, limit)
            assert _tree_key(got) == _tree_key(want), (len(g.ops), limit)
            lin = fast_lin(g, got)
            assert lin == ref_lin(g, want)
            assert fast_lin(g, got).leaf_of_op is not lin.leaf_of_op
            # tensor routing on two copies of the tree (it records owned_tensors)
            leaf_of = dict(lin.leaf_of_op)
            if limit == 20:   # a routing that moves weight-update ops, as plan() does
                for v in want.floating_ops[::2]:
                    leaf_of[v] = want.leaves()[-1].id
            for lo in (None, leaf_of):
                t_ref, t_fast = ref_tree(g, limit), ref_tree(g, limit)
                assert fast_assign(t_fast, g, lo) == ref_assign(t_ref, g, lo)
                assert [x.owned_tensors for x in t_fast.leaves()] == [x.owned_tensors for x in t_ref.leaves()]
    inference = mp.graph.load_graph(gg.config_doc("layered"))
    for fn in (ref_tree, fast_tree):
        with pytest.raises(mp.graph.StructuralError, match="no backward pass"):
            fn(inference, 20)
        with pytest.raises(mp.graph.ConfigError, match="node_limit"):
            fn(graphs[0], 1)


def test_live_set_sweep_matches_interval_rule():
    """windows._sweep_live_sets against the interval rule it sweeps, on random
    (birth, last-use) intervals and slot sets, including empty sets, shared
    endpoints and tensors that never enter."""
    import random

    import numpy as np

    from paper_2310_19295_b200.windows import _sweep_live_sets
    rng = random.Random(5)
    for trial in range(200):
        T = rng.randint(0, 40)
        H = rng.randint(1, 30)
        b = np.array([rng.randint(0, H) for _ in range(T)], np.int64)
        L = np.array([min(H, bb + rng.randint(0, H)) for bb in b], np.int64)
        slots = sorted(rng.sample(range(H + 1), rng.randint(1, H + 1)))
        got = _sweep_live_sets(b, L, slots)
        for p in slots:
            want_in = {t for t in range(T) if b[t] < p <= L[t]}
            want_out = {t for t in range(T) if b[t] <= p < L[t]}
            li, lo = got[p]
            assert set(li) == want_in and set(lo) == want_out
            assert set(li.arr.tolist()) == want_in and set(lo.arr.tolist()) == want_out


@pytest.mark.skipif(mp is None, reason="reference memplan not importable")
def test_window_problems_op_in_two_windows_matches_reference():
    """A linearisation that lists ops in two windows (the reference then keeps
    the LAST listing window as the op's position, ordering.py:490-503): the
    non-owner windows get the reference's rule evaluated directly, the rest
    the interval rule -- equal to the reference on every window."""
    import dataclasses
    import random

    import memplan.graphgen as rgen

    from paper_2310_19295_b200 import windows as W
    rng = random.Random(5)
    n_shared = 0
    for arch, blocks in (("transformer_block", 3), ("mlp", 4), ("residual", 3)):
        g = rgen.gen_training_graph(arch, blocks, optimizer="adam")
        tree = mp.segmentation.build_subgraph_tree(g, 8)
        lin = mp.segmentation.linearize(g, tree)
        wu = mp.ordering.place_weight_updates(g, tree, 2.0)
        wins = [w for w in lin.windows if w.ops]
        for trial in range(12):
            a, b = rng.sample(range(len(wins)), 2)
            moved = tuple(rng.sample(wins[a].ops, min(len(wins[a].ops), rng.randint(1, 3))))
            new = list(lin.windows)
            k = new.index(wins[b])
            new[k] = dataclasses.replace(new[k], ops=tuple(sorted(set(new[k].ops) | set(moved))))
            lin2 = dataclasses.replace(lin, windows=tuple(new))
            want = mp.ordering.build_window_problems(g, lin2, wu)
            got = W.build_window_problems(g, lin2, wu, window_type=mp.segmentation.Window,
                                          problem_type=mp.ordering.OrderingProblem)
            assert got == want
            n_shared += 1
    assert n_shared >= 30


@pytest.mark.skipif(mp is None, reason="reference memplan not importable")
def test_region_between_with_custom_build_preds():
    """_region_between on a _TreeBuild whose preds are NOT the graph's closure
    (the core's induced closure): the drop-in unpacks build.preds itself --
    the reference's answer, without running reference code."""
    import memplan.graphgen as rgen

    from paper_2310_19295_b200 import control
    seg, rg = mp.segmentation, mp.graph
    fast = control.region_between_factory()
    for arch in ("transformer_block", "residual"):
        g = rgen.gen_training_graph(arch, 3, optimizer="adam")
        branches = rg.weight_update_branches(g)
        floating = {v for b in branches for v in b.ops}
        core = [v for v in range(g.n_ops) if v not in floating]
        for preds in (rg.predecessor_masks(g, core[: len(core) // 2]), rg.predecessor_masks(g)):
            build = seg._TreeBuild(g=g, node_limit=8, preds=preds, categories=rg.classify_tensors(g),
                                   branches=branches)
            for lo, hi in ((None, core[len(core) // 3]), (core[2], core[-3]), (core[5], None),
                           (core[len(core) // 4], core[len(core) // 3])):
                assert fast(build, core, lo, hi) == seg._region_between(build, core, lo, hi)


@pytest.mark.skipif(mp is None, reason="reference memplan not importable")
def test_segment_tree_dropin_matches_reference():
    """build_segment_tree / independent_segments (segmentation.py:120-136,
    451-476), the inference-graph decomposition plan() runs on graphs with no
    backward op, from the C++ closure: the reference's segments and tree node
    for node on the layered config graph, random DAGs and chains (host-only)."""
    import memplan.graphgen  # noqa: F401  (mp.graphgen)

    from paper_2310_19295_b200 import control
    from paper_2310_19295_b200 import graphgen as gg
    seg = mp.segmentation
    fast_segments, fast_tree = control.segment_tree_factory(mp)
    graphs = [mp.graph.load_graph(gg.config_doc("layered")),
              mp.graph.load_graph(gg.layered_dag_doc(layers=6, width=1))]
    graphs += [mp.graphgen.gen_random_dag(n, d, seed=seed) for n, d, seed in
               ((1, 0.3, 0), (12, 0.2, 1), (40, 0.1, 2), (60, 0.05, 3), (80, 0.3, 4))]
    graphs.append(mp.graphgen.gen_greedy_trap(0))
    for g in graphs:
        assert fast_segments(g) == seg.independent_segments(g)
        for limit in (2, 5, 20, 10**6):
            assert _tree_key(fast_tree(g, limit)) == _tree_key(seg.build_segment_tree(g, limit))
    with pytest.raises(mp.graph.ConfigError, match="node_limit"):
        fast_tree(graphs[0], 1)


@pytest.mark.skipif(mp is None, reason="reference memplan not importable")
def test_place_weight_updates_matches_reference(monkeypatch):
    """rm_place_weight_updates (host C++) returns the reference's
    WeightUpdatePlan exactly -- placements, delays, targets, ratios and
    projected uses bit for bit -- for every call the planner makes, and for
    the same trees under other delay radii, alpha maps and force_immediate;
    an unresolvable alpha raises the reference's ConfigError message."""
    import memplan.graphgen as rgen

    from paper_2310_19295_b200 import control as ctl
    from paper_2310_19295_b200 import graphgen as gg
    fast = ctl.place_weight_updates_factory(mp)
    orig = mp.ordering.place_weight_updates
    calls, delayed = [], []

    def both(g, tree, r, alpha=None, *, force_immediate=False):
        want = orig(g, tree, r, alpha, force_immediate=force_immediate)
        assert fast(g, tree, r, alpha, force_immediate=force_immediate) == want
        for rr in (0.0, 0.25, 1.0, 3.0):
            for al in (None, {"adam": 0.5, "sgd": 9.0}, {"default": 2.5, "ad": 1.0}, {"default": 40.0},
                       {"default": 400.0, "adam.": 3000.0}):
                for fi in (False, True):
                    assert fast(g, tree, rr, al, force_immediate=fi) == orig(g, tree, rr, al, force_immediate=fi)
        if want.placements:
            with pytest.raises(mp.graph.ConfigError) as e_ref:
                orig(g, tree, r, {"nomatch": 1.0})
            with pytest.raises(mp.graph.ConfigError) as e_got:
                fast(g, tree, r, {"nomatch": 1.0})
            assert str(e_got.value) == str(e_ref.value)
        calls.append(len(want.placements))
        delayed.append(sum(p.delayed for p in orig(g, tree, 0.0, {"default": 400.0}).placements))
        return want

    monkeypatch.setattr(mp.planner, "place_weight_updates", both)
    mp.planner.plan(mp.graph.load_graph(gg.config_doc("gpt2-small")))
    for arch in ("mlp", "residual", "transformer_block"):
        for opt in ("sgd", "adam"):
            mp.planner.plan(rgen.gen_training_graph(arch, 4, optimizer=opt))
    assert len(calls) >= 7 and sum(calls) > 100
    assert sum(delayed) > 20      # the delay rule and the later-window scan are exercised
