"""K4 (batched window greedy) against the reference's golden greedy_order
vectors (tests/golden/greedy.json: whole graphs, edge fixtures incl. the
duplicate-input hazard h1, and the real window problems of the planner's own
decomposition) and the oracle on large windows; orders and peaks bit-exact."""

from __future__ import annotations

import random

import pytest

from conftest import golden
from oracle import memplan_oracle as O
from paper_2310_19295_b200 import graphgen as gg
from paper_2310_19295_b200.graph import ConfigError, load_graph
from paper_2310_19295_b200.ordering import OrderingProblem, greedy_order, greedy_orders

pytestmark = pytest.mark.gpu


def _cases():
    G = golden("greedy")
    graphs = {}
    for c in G["cases"]:
        key = c.get("graph") or id(c)
        if key not in graphs:
            graphs[key] = load_graph(c.get("doc") or G["graphs"][c["graph"]])
        yield graphs[key], c


def test_golden_one_by_one():
    for g, c in _cases():
        sol = greedy_order(OrderingProblem(g, tuple(c["ops"]), frozenset(c["live_in"]),
                                           frozenset(c["live_out"])))
        assert list(sol.order) == c["order"] and sol.peak == c["peak"], c.get("graph")
        assert not sol.optimal


def test_golden_batched():
    """All windows in one call: grouped per graph, one launch per graph."""
    probs, want = [], []
    for g, c in _cases():
        probs.append(OrderingProblem(g, tuple(c["ops"]), frozenset(c["live_in"]), frozenset(c["live_out"])))
        want.append((c["order"], c["peak"]))
    for sol, (o, pk) in zip(greedy_orders(probs), want):
        assert list(sol.order) == o and sol.peak == pk


@pytest.mark.parametrize("name", ["layered", "gpt2-small"])
def test_whole_config_graph_vs_oracle(name):
    g = load_graph(gg.config_doc(name))
    ops = tuple(range(len(g.ops)))
    sol = greedy_order(OrderingProblem(g, ops))
    assert (sol.order, sol.peak) == O.greedy_order(g, ops)


def test_random_subwindows_vs_oracle():
    g = load_graph(gg.config_doc("gpt2-small"))
    n = len(g.ops)
    rng = random.Random(5)
    probs = []
    for _ in range(12):
        a = rng.randrange(0, n - 50)
        ops = tuple(range(a, min(n, a + rng.randint(20, 400))))
        inside = set(ops)
        # boundary context like build_window_problems: inputs from outside are
        # live-in, products consumed outside are live-out
        lin = {t for v in ops for t in g.ops[v].inputs if g.tensors[t].producer not in inside}
        lout = {t for v in ops for t in g.ops[v].outputs
                if any(c not in inside for c in g.tensors[t].consumers)}
        probs.append(OrderingProblem(g, ops, frozenset(lin), frozenset(lout)))
    for p, sol in zip(probs, greedy_orders(probs)):
        assert (sol.order, sol.peak) == O.greedy_order(g, p.ops, p.live_in, p.live_out)


def test_config_error_live_in_unconsumed():
    g = load_graph(golden("greedy")["graphs"]["mlp2"])
    # a live-in tensor nobody in the window consumes, not live-out
    ops = (0,)
    unused = next(t.id for t in g.tensors if 0 not in t.consumers and t.producer != 0)
    with pytest.raises(ConfigError):
        greedy_order(OrderingProblem(g, ops, frozenset({unused})))
    with pytest.raises(ConfigError):
        greedy_order(OrderingProblem(g, ops, ops_per_step=0))


def test_scratch_forms_and_64bit_scores(monkeypatch):
    """The working set in global scratch (windows above the shared-memory
    budget, forced here by the RM_K4_SMEM_LIMIT test hook) next to windows in
    shared memory, in one call; and the 64-bit score form (one tensor of
    2^40 + 4 KiB bytes, above the 32-bit form's 2^30 units)."""
    import copy

    doc = gg.layered_dag_doc(layers=60, width=20)
    big = copy.deepcopy(doc)
    t = next(t for t in big["tensors"] if any(t["id"] in o["inputs"] for o in big["ops"]))
    t["size_bytes"] = 2 ** 40 + 4096
    for d in (doc, big):
        g = load_graph(d)
        n = len(g.ops)
        whole = tuple(range(n))
        sub = tuple(range(100, 180))
        inside = set(sub)
        lin = frozenset(t for v in sub for t in g.ops[v].inputs if g.tensors[t].producer not in inside)
        lout = frozenset(t for v in sub for t in g.ops[v].outputs
                         if any(c not in inside for c in g.tensors[t].consumers))
        probs = [OrderingProblem(g, whole), OrderingProblem(g, sub, lin, lout)]
        want = [O.greedy_order(g, whole), O.greedy_order(g, sub, lin, lout)]
        for limit in (None, "20000", "0"):
            if limit is None:
                monkeypatch.delenv("RM_K4_SMEM_LIMIT", raising=False)
            else:
                monkeypatch.setenv("RM_K4_SMEM_LIMIT", limit)
            got = [(s.order, s.peak) for s in greedy_orders(probs)]
            assert got == want, (limit, d is big)
