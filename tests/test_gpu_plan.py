"""End-to-end drop-in: the reference's own ``plan(g, cfg)`` with the B200 hot
path installed (memplan_plugin) must emit byte-identical plan documents
(planner.py:398-399) -- against the golden plans the reference produced in the
build container, and against the unpatched reference run live on the same box
(baseline/_ref) for the BASELINE config graphs."""

from __future__ import annotations

import pytest

from conftest import golden
from paper_2310_19295_b200 import graphgen as gg
from paper_2310_19295_b200 import memplan_plugin as plug
from paper_2310_19295_b200.evaluator import launch_count

pytestmark = pytest.mark.gpu

try:
    mp = plug.load_memplan()
except ImportError:  # pragma: no cover - baseline/_ref missing
    mp = None
needs_ref = pytest.mark.skipif(mp is None, reason="reference memplan not installed (baseline/_ref)")


@needs_ref
@pytest.mark.parametrize("name", sorted(golden("plans")))
def test_golden_plan_bytes(name):
    c = golden("plans")[name]
    g = mp.graph.load_graph(c["doc"])
    plug.install(mp)
    try:
        before = launch_count()
        got = mp.planner.plan_doc_bytes(mp.planner.plan(g)).decode()
        assert launch_count() > before          # the GPU path really ran
    finally:
        plug.uninstall()
    assert got == c["plan"]


def _config_graph(name):
    if name.startswith("ref-"):   # the reference's own generator, e.g. ref-transformer_block-100
        import memplan.graphgen as rgen
        _, arch, blocks = name.split("-")
        return rgen.gen_training_graph(arch, int(blocks), optimizer="adam")
    return mp.graph.load_graph(gg.config_doc(name))


@needs_ref
@pytest.mark.parametrize("name", ["layered", "gpt2-small", "bert-large", "gpt2-xl", "ref-transformer_block-100",
                                  "ref-residual-60", "ref-mlp-60"])
def test_config_plan_matches_live_reference(name, monkeypatch):
    """BASELINE configs 1-4 (and the reference's own generator at 100 blocks):
    plan documents byte-identical to the unpatched reference run live on the
    same box, with no reference solver reachable under the plug-in."""
    g = _config_graph(name)
    want = mp.planner.plan_doc_bytes(mp.planner.plan(g))
    _ban_reference_solvers(monkeypatch)
    plug.install(mp)
    try:
        got = mp.planner.plan_doc_bytes(mp.planner.plan(g))
    finally:
        plug.uninstall()
    assert got == want


@needs_ref
def test_replay_and_compare_through_plugin():
    c = golden("plans")["diamond"]
    g = mp.graph.load_graph(c["doc"])
    plug.install(mp)
    try:
        p = mp.planner.plan(g)
        assert mp.simulator.replay_static(g, p.schedule, p.layout) == (94371840, [])
        rows = mp.planner.compare_baselines(g)
        assert rows
    finally:
        plug.uninstall()


@needs_ref
def test_cli_plan_and_eval_through_plugin(tmp_path):
    """`python -m paper_2310_19295_b200 plan/eval` = the reference CLI on the
    GPU path: same plan file bytes, eval exit code 0."""
    import json
    from paper_2310_19295_b200.__main__ import main
    c = golden("plans")["transformer_block-2-adam"]
    gpath = tmp_path / "g.json"
    gpath.write_text(json.dumps(c["doc"]))
    out = tmp_path / "p.json"
    try:
        assert main(["plan", "--graph", str(gpath), "--out", str(out)]) == 0
        assert out.read_text() == c["plan"]
        assert main(["eval", "--graph", str(gpath), "--plan", str(out)]) == 0
    finally:
        plug.uninstall()


@needs_ref
def test_capped_searches_match_live_reference():
    """Node caps tight enough that the planner's windows and leaves reach the
    capped searches (exact_order's DFS where K5 hands a window back,
    exact_layout's branch-and-bound where K3's incumbent misses its bound):
    the libroam restatements stop where the reference stops, so the plan
    documents -- optimal_leaves included -- stay byte-identical."""
    import memplan.graphgen as rgen
    runs = {"windows_dfs": 0, "windows_dfs_budget": 0, "leaves_search": 0}
    for cfgkw in (dict(order_node_cap=3, layout_node_cap=5), dict(order_node_cap=40),
                  dict(node_limit=14, order_node_cap=400, layout_limit=16, layout_node_cap=60),
                  dict(node_limit=6, order_node_cap=2000, layout_node_cap=100_000)):
        cfg = mp.planner.PlannerConfig(**cfgkw)
        for arch, blocks in (("transformer_block", 2), ("mlp", 3), ("residual", 3)):
            g = rgen.gen_training_graph(arch, blocks, optimizer="adam")
            want = mp.planner.plan_doc_bytes(mp.planner.plan(g, cfg))
            plug.install(mp)
            try:
                got = mp.planner.plan_doc_bytes(mp.planner.plan(g, cfg))
                for k in runs:
                    runs[k] += plug.STATS[k]
            finally:
                plug.uninstall()
            assert got == want, (arch, cfgkw)
    # real plans reach the window DFS; their small leaves meet the layout bound
    # (SURVEY probe p12), so the branch-and-bound is pinned by
    # test_layout_search.py instead
    assert runs["windows_dfs"] + runs["windows_dfs_budget"] > 0, runs


# the reference functions no plan may run once the plug-in is installed
_BANNED = [("ordering", "exact_order"), ("planner", "exact_order"), ("ordering", "greedy_order"),
           ("planner", "greedy_order"), ("layout", "exact_layout"), ("planner", "exact_layout"),
           ("layout", "constrained_llfb_layout"), ("planner", "constrained_llfb_layout"),
           ("layout", "llfb_layout"), ("ordering", "build_window_problems"), ("graph", "asap_alap"),
           ("graph", "predecessor_masks"), ("segmentation", "predecessor_masks"),
           ("graph", "successor_masks"), ("segmentation", "successor_masks"),
           ("graph", "live_bytes_by_timestep"), ("graph", "peak_memory"), ("layout", "layout_violations"),
           ("ordering", "place_weight_updates"), ("planner", "place_weight_updates"),
           ("ordering", "weight_update_cost"), ("layout", "repair_conflicts"), ("planner", "repair_conflicts")]


def _ban_reference_solvers(monkeypatch):
    def banned(*a, **k):
        raise AssertionError("a reference solver ran under the plug-in")
    n = 0
    for mod, name in _BANNED:
        m = getattr(mp, mod)
        if hasattr(m, name):
            monkeypatch.setattr(m, name, banned)
            n += 1
    return n


WIDE = {
    "layered-80": (lambda: gg.layered_dag_doc(layers=10, width=8),
                   dict(node_limit=600, layout_limit=300, order_node_cap=5000, layout_node_cap=5000)),
    "layered-80-roomy": (lambda: gg.layered_dag_doc(layers=10, width=8),
                         dict(node_limit=100, layout_limit=100, order_node_cap=50_000, layout_node_cap=50_000)),
    "layered-96": (lambda: gg.layered_dag_doc(layers=8, width=12),
                   dict(node_limit=600, layout_limit=300, order_node_cap=5000, layout_node_cap=5000)),
    "gpt2-small-600": (lambda: gg.config_doc("gpt2-small"),
                       dict(node_limit=600, layout_limit=300, order_node_cap=5000, layout_node_cap=5000)),
    "gpt2-small-80": (lambda: gg.config_doc("gpt2-small"),
                      dict(node_limit=80, layout_limit=80, order_node_cap=20_000, layout_node_cap=20_000)),
}


@needs_ref
@pytest.mark.parametrize("name", sorted(WIDE))
def test_wide_limits_served_by_libroam(name, monkeypatch):
    """node_limit / layout_limit above 64: windows of 80-541 ops reach the
    exact search and leaves of 240-288 items the branch-and-bound.  Every one
    is served by libroam (multi-word masks) -- the reference's solvers,
    window builder and closure functions are replaced by raising stubs while
    the plug-in plans -- and the documents equal the live reference's."""
    mk, kw = WIDE[name]
    g = mp.graph.load_graph(mk())
    cfg = mp.planner.PlannerConfig(**kw)
    want = mp.planner.plan_doc_bytes(mp.planner.plan(g, cfg))
    assert _ban_reference_solvers(monkeypatch) >= 12
    plug.install(mp)
    try:
        got = mp.planner.plan_doc_bytes(mp.planner.plan(g, cfg))
        stats = dict(plug.STATS)
    finally:
        plug.uninstall()
    assert got == want
    served = stats["windows_k5"] + stats["windows_dfs"] + stats["windows_dfs_budget"]
    assert served > 0 and "windows_ref_dfs" not in stats and "leaves_ref_search" not in stats, stats


@needs_ref
@pytest.mark.parametrize("name", ["gpt2-small", "bert-large", "ref-transformer_block-20"])
def test_replay_static_dropin_matches_live_reference(name):
    """simulator.replay_static (simulator.py:129-145) rebound to K2's
    max-extent epilogue: (actual, violations) equal to the reference's
    O(steps x N) replay on a planned layout, on the same layout with a
    few tensors shifted into each other (violations in the reference's
    message order), with an offset missing, and through memplan's re-export."""
    import dataclasses
    g = _config_graph(name)
    p = mp.planner.plan(g)
    offs = dict(p.layout.offsets)
    ids = sorted(offs)[:: max(1, len(offs) // 7)]
    for t in ids[1:]:
        offs[t] = offs[ids[0]]
    broken = dataclasses.replace(p.layout, offsets=offs)
    missing = dataclasses.replace(p.layout, offsets={t: o for t, o in p.layout.offsets.items() if t != ids[0]})
    want = [mp.simulator.replay_static(g, p.schedule, m) for m in (p.layout, broken, missing)]
    assert want[0][1] == [] and want[1][1] and want[2][1]
    plug.install(mp)
    try:
        before = launch_count()
        got = [mp.simulator.replay_static(g, p.schedule, m) for m in (p.layout, broken, missing)]
        assert mp.replay_static(g, p.schedule, p.layout) == want[0]
        assert launch_count() > before
    finally:
        plug.uninstall()
    assert got == want
