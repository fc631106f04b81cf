"""exact_order's capped DFS (ordering.py:183-286) in libroam
(rm_exact_order_search) against the reference on wide windows under node
caps from tiny to roomy (tests/golden/exact_search.json, made by
make_golden.py exact_search) and on every golden exact_order case: the same
order, peak and node count when the search finishes, the budget outcome
(the reference returns its greedy incumbent) when the cap stops it.  The
search is host code, so the host test needs no GPU; the GPU test runs the
product path (K5, then the DFS for the windows K5 hands back)."""

from __future__ import annotations

import pytest

from conftest import golden
from paper_2310_19295_b200.graph import load_graph
from paper_2310_19295_b200.ordering import BUDGET, OrderingProblem, search_window


def _cases(name):
    G = golden(name)
    graphs = {}
    for c in G["orders" if name == "wide_search" else "cases"]:
        key = c["graph"] if "doc" not in c else id(c)
        if key not in graphs:
            graphs[key] = load_graph(c["doc"] if "doc" in c else G["graphs"][c["graph"]])
        yield graphs[key], c


def _problem(g, c):
    return OrderingProblem(g, tuple(c["ops"]), frozenset(c["live_in"]), frozenset(c["live_out"]),
                           node_cap=c["node_cap"])


@pytest.mark.parametrize("name", ["exact_search", "exact", "wide_search"])
def test_dfs_matches_reference_host(name):
    n_opt = n_budget = 0
    for g, c in _cases(name):
        r = search_window(_problem(g, c))
        if c["optimal"]:
            assert r is not BUDGET, c
            assert (list(r[0]), r[1], r[2]) == (c["order"], c["peak"], c["nodes"]), c
            n_opt += 1
        else:
            assert r is BUDGET, c
            n_budget += 1
    assert n_opt > (30 if name == "wide_search" else 100) and n_budget >= 2


@pytest.mark.gpu
def test_exact_orders_with_dfs_fallback():
    from paper_2310_19295_b200.ordering import exact_orders
    cases = list(_cases("exact_search"))
    sols = exact_orders([_problem(g, c) for g, c in cases])
    for (g, c), s in zip(cases, sols):
        assert (list(s.order), s.peak, s.optimal) == (c["order"], c["peak"], c["optimal"]), c


@pytest.mark.gpu
def test_wide_windows_product_path():
    """Windows of 65-140 ops (node_limit > 64) through the product path: K5
    hands them back, the multi-word DFS decides (reference's order, peak,
    optimal flag)."""
    from paper_2310_19295_b200.ordering import exact_orders
    cases = list(_cases("wide_search"))
    assert min(len(c["ops"]) for _, c in cases) > 64
    sols = exact_orders([_problem(g, c) for g, c in cases])
    for (g, c), s in zip(cases, sols):
        assert (list(s.order), s.peak, s.optimal) == (c["order"], c["peak"], c["optimal"]), c["graph"]
