"""K3 (batched long-lived-first packer) against the reference's golden layout
vectors (tests/golden/layouts.json, produced by the reference itself) and the
oracle restatement; offsets and capacities bit-exact."""

from __future__ import annotations

import random

import pytest

from conftest import golden
from oracle import memplan_oracle as O
from paper_2310_19295_b200.layout import (COMPONENTS, CONSTRAINED, PLAIN, LayoutItem, LayoutProblem,
                                          constrained_llfb_layout, exact_layout,
                                          exact_layout_batch, llfb_layout, pack_batch)

pytestmark = pytest.mark.gpu
MB = 1 << 20


def _items(rows):
    return tuple(LayoutItem(*r) for r in rows)


def _offs(d):
    return {int(k): v for k, v in d.items()}


def test_spec_llfb_example():
    # x(8,[0,10]), y(4,[0,3]), z(4,[4,10]) -> x@0, y@8, z@8, cap 12
    spec = golden("layouts")["spec"][0]
    m = llfb_layout(LayoutProblem(items=_items(spec["items"])))
    assert m.offsets == _offs(spec["offsets"]) and m.capacity == spec["capacity"] == 12
    assert not m.optimal


def test_llfb_and_constrained_golden():
    cases = golden("layouts")["llfb"]
    for c in cases:
        p = LayoutProblem(items=_items(c["items"]), activations_at_bottom=True)
        a = llfb_layout(p)
        b = constrained_llfb_layout(p)
        assert (a.offsets, a.capacity) == (_offs(c["llfb"]["offsets"]), c["llfb"]["capacity"])
        assert (b.offsets, b.capacity) == (_offs(c["constrained"]["offsets"]), c["constrained"]["capacity"])
        assert a.activation_block == sum(i.size for i in p.items if i.is_activation)
    # the whole corpus as ONE batched launch per mode gives the same answers
    plain = pack_batch([_items(c["items"]) for c in cases], PLAIN)
    cons = pack_batch([_items(c["items"]) for c in cases], CONSTRAINED)
    for c, a, b in zip(cases, plain, cons):
        assert a.offsets == _offs(c["llfb"]["offsets"]) and a.capacity == c["llfb"]["capacity"]
        assert b.offsets == _offs(c["constrained"]["offsets"]) and b.capacity == c["constrained"]["capacity"]


def test_exact_golden_decided_without_search():
    """Every golden exact_layout case the reference closed at 0 nodes is decided
    by K3 alone (same offsets and capacity); the others need the search."""
    cases = golden("layouts")["exact"]
    probs = [LayoutProblem(items=_items(c["items"]), activations_at_bottom=True, node_cap=200_000)
             for c in cases]
    res = exact_layout_batch(probs, search=False)
    for c, p, r in zip(cases, probs, res):
        if c["nodes"] == 0:
            assert r is not None, c
            assert r.offsets == _offs(c["offsets"]) and r.capacity == c["capacity"] and r.optimal
        else:
            assert r is None, c
    # with the search (rm_layout_search) every case is the reference's answer
    for c, r in zip(cases, exact_layout_batch(probs)):
        assert (r.offsets, r.capacity, r.optimal, r.stats.nodes) == \
            (_offs(c["offsets"]), c["capacity"], c["optimal"], c["nodes"]), c


def test_exact_spec_examples():
    # disjoint 16 MB / 20 MB -> both @0, cap 20 MB; a 3-clique stacks
    m = exact_layout(LayoutProblem(items=(LayoutItem(0, 16 * MB, 0, 1), LayoutItem(1, 20 * MB, 2, 3))))
    assert m.offsets == {0: 0, 1: 0} and m.capacity == 20 * MB and m.optimal
    m = exact_layout(LayoutProblem(items=(LayoutItem(0, 4, 0, 5), LayoutItem(1, 2, 1, 5), LayoutItem(2, 1, 2, 5))))
    assert m.capacity == 7
    assert exact_layout(LayoutProblem(items=())).capacity == 0


def _rand_rows(rng, n, horizon, act_p):
    rows = []
    for t in rng.sample(range(4 * n), n):
        s = rng.randint(0, horizon - 1)
        e = min(horizon - 1, s + rng.randint(0, max(1, horizon // 3)))
        rows.append((t, rng.choice([0, 1, 3, 8, 64, 100]) * rng.choice([1, MB]), s, e, rng.random() < act_p))
    return rows


@pytest.mark.parametrize("n", [1, 2, 31, 255, 256, 257, 1000, 3000, 4095, 4096])
def test_random_vs_oracle(n):
    rng = random.Random(1000 + n)
    rows = _rand_rows(rng, n, max(4, n // 3), 0.3)
    items = _items(rows)
    a, b = pack_batch([items], PLAIN)[0], pack_batch([items], CONSTRAINED)[0]
    wa = O.llfb_layout(rows)
    wb = O.constrained_llfb_layout(rows)
    assert (a.offsets, a.capacity) == wa
    assert (b.offsets, b.capacity) == wb


def test_large_problem_global_scratch():
    """> shared-memory working set: the CTA works out of global scratch."""
    rng = random.Random(7)
    rows = _rand_rows(rng, 6000, 2000, 0.2)
    items = _items(rows)
    b = pack_batch([items], CONSTRAINED)[0]
    assert (b.offsets, b.capacity) == O.constrained_llfb_layout(rows)


@pytest.mark.parametrize("n,horizon", [(5000, 1500), (8191, 3000), (8192, 3000), (9035, 4000), (10239, 3000),
                                       (10240, 3000), (6000, 70000)])
def test_register_list_geometries(n, horizon):
    """Placed lists of 4k-8k items (512 threads, start | end packed in 16 bits),
    8k-10k items (1024 threads, 4 register + 6 shared-memory slots each, every
    working set in global scratch; a small leaf rides in the same launch),
    the first size past it (the shared-memory list) and timesteps beyond 16
    bits (routed to the 1024-thread path)."""
    rng = random.Random(n + horizon)
    rows = _rand_rows(rng, n, horizon, 0.2)
    small = _rand_rows(rng, 40, 30, 0.2)
    b, c = pack_batch([_items(rows), _items(small)], CONSTRAINED)
    assert (b.offsets, b.capacity) == O.constrained_llfb_layout(rows)
    assert (c.offsets, c.capacity) == O.constrained_llfb_layout(small)
    if n in (9035, 10239):
        p = pack_batch([_items(rows)], PLAIN)[0]
        assert (p.offsets, p.capacity) == O.llfb_layout(rows)


def test_components_vs_oracle():
    rng = random.Random(3)
    probs = []
    for k in range(200):
        probs.append(_rand_rows(rng, rng.randint(1, 24), rng.randint(3, 30), 0.3))
    res = pack_batch([_items(r) for r in probs], COMPONENTS)
    for rows, r in zip(probs, res):
        offs, cap, met, comps = O.component_incumbents(rows)
        assert r.offsets == offs and r.capacity == cap and r.bound_met == met
        assert r.comp_cap == {root: c[1] for root, c in comps.items()}


# ---- K3 DAG placement (items placed in rounds over the time-overlap relation)

@pytest.fixture
def pack_form():
    from paper_2310_19295_b200.layout import set_pack_form
    yield set_pack_form
    set_pack_form(0)


def _planner_like_rows(rng, n, horizon, act_p, long_p=0.005):
    """Mostly one-to-few-step temporaries plus a few long-lived tensors, sizes
    with duplicates and zeros (ties in lo / hi), like the planner's leaves."""
    rows = []
    for t in rng.sample(range(4 * n), n):
        s = rng.randint(0, horizon - 1)
        ln = rng.randint(0, horizon // 8) if rng.random() < long_p else rng.choice([0, 0, 1, 1, 2, 3, 5])
        e = min(horizon - 1, s + ln)
        rows.append((t, rng.choice([0, 1, 3, 8, 64, 100]) * rng.choice([1, MB]), s, e, rng.random() < act_p))
    return rows


@pytest.mark.parametrize("form", [1, 2])
def test_forms_on_golden_corpora(pack_form, form):
    """The placed-list path (1) and the DAG rounds (2, every problem) give the
    reference's golden layouts."""
    pack_form(form)
    cases = golden("layouts")["llfb"]
    plain = pack_batch([_items(c["items"]) for c in cases], PLAIN)
    cons = pack_batch([_items(c["items"]) for c in cases], CONSTRAINED)
    for c, a, b in zip(cases, plain, cons):
        assert a.offsets == _offs(c["llfb"]["offsets"]) and a.capacity == c["llfb"]["capacity"]
        assert b.offsets == _offs(c["constrained"]["offsets"]) and b.capacity == c["constrained"]["capacity"]
    spec = golden("layouts")["spec"][0]
    m = pack_batch([_items(spec["items"])], PLAIN)[0]
    assert m.offsets == _offs(spec["offsets"]) and m.capacity == 12


@pytest.mark.parametrize("form", [0, 1, 2])
@pytest.mark.parametrize("n,horizon", [(1, 3), (40, 20), (700, 300), (1023, 900), (1024, 900), (3000, 2500),
                                       (9035, 8000), (10240, 9000)])
def test_dag_rounds_vs_oracle(pack_form, form, n, horizon):
    """Planner-like problems (shallow time-overlap relation: the DAG rounds
    qualify) in every form, PLAIN and CONSTRAINED, with a small problem
    riding in the same launch."""
    pack_form(form)
    key = (n, horizon)
    if key not in _ORACLE:  # the same problems in every form: the oracle runs once
        rng = random.Random(17 * n + horizon)
        rows = _planner_like_rows(rng, n, horizon, 0.1)
        small = _planner_like_rows(rng, 30, 12, 0.2)
        _ORACLE[key] = (rows, small, O.constrained_llfb_layout(rows), O.constrained_llfb_layout(small),
                        O.llfb_layout(rows))
    rows, small, want_b, want_c, want_a = _ORACLE[key]
    b, c = pack_batch([_items(rows), _items(small)], CONSTRAINED)
    assert (b.offsets, b.capacity) == want_b
    assert (c.offsets, c.capacity) == want_c
    a = pack_batch([_items(rows)], PLAIN)[0]
    assert (a.offsets, a.capacity) == want_a


_ORACLE: dict = {}


def test_dag_rounds_fall_back_on_dense_problems(pack_form):
    """Heavily overlapping items (more obstacles per item than the lists
    hold) keep the placed-list path: same answers."""
    pack_form(2)
    rng = random.Random(5)
    rows = _rand_rows(rng, 2000, 600, 0.2)
    b = pack_batch([_items(rows)], CONSTRAINED)[0]
    assert (b.offsets, b.capacity) == O.constrained_llfb_layout(rows)


def test_dag_rounds_components(pack_form):
    pack_form(2)
    rng = random.Random(4)
    probs = [_planner_like_rows(rng, rng.randint(1, 40), rng.randint(3, 30), 0.3) for _ in range(200)]
    res = pack_batch([_items(r) for r in probs], COMPONENTS)
    for rows, r in zip(probs, res):
        offs, cap, met, comps = O.component_incumbents(rows)
        assert r.offsets == offs and r.capacity == cap and r.bound_met == met
        assert r.comp_cap == {root: c[1] for root, c in comps.items()}
