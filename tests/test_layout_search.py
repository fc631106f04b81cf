"""exact_layout's branch-and-bound (layout.py:226-290) in libroam
(rm_layout_search) against the reference's own results on problems whose
incumbent misses its bound (tests/golden/layout_search.json, made by
make_golden.py layout_search): same offsets, capacity, optimal flag and node
count, for full searches and node-capped ones.

The host test feeds the search the incumbent the oracle restates (the search
is host code: no GPU); the GPU test runs the product path, K3's COMPONENTS
pass followed by the search."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from conftest import golden
from oracle import memplan_oracle as O
from paper_2310_19295_b200 import _lib


def _offs(d):
    return {int(k): v for k, v in d.items()}


def _incumbent(rows, bottom):
    """K3 COMPONENTS' offsets, restated by the oracle (per-component long-lived
    first placement; without the activation rule that is llfb_layout)."""
    return O.component_incumbents(rows)[0] if bottom else O.llfb_layout(rows)[0]


def _search(rows, bottom, node_cap, incumbent):
    lib = _lib.lib()
    n = len(rows)
    tensor = np.array([r[0] for r in rows], np.int32)
    size = np.array([r[1] for r in rows], np.int64)
    start = np.array([r[2] for r in rows], np.int32)
    end = np.array([r[3] for r in rows], np.int32)
    act = np.array([1 if r[4] else 0 for r in rows], np.uint8)
    inc = np.array([incumbent[r[0]] for r in rows], np.int64)
    off = np.empty(n, np.int64)
    cap, nodes, opt = C.c_int64(0), C.c_int64(0), C.c_int32(0)
    _lib.check(lib.rm_layout_search(n, _lib.ptr(tensor), _lib.ptr(start), _lib.ptr(end), _lib.ptr(size),
                                    _lib.ptr(act), int(bottom), _lib.ptr(inc), node_cap, 0.0, _lib.ptr(off),
                                    C.byref(cap), C.byref(nodes), C.byref(opt)), "rm_layout_search")
    return dict(zip(tensor.tolist(), off.tolist())), cap.value, bool(opt.value), nodes.value


def test_search_matches_reference_host():
    cases = golden("layout_search")["cases"]
    assert len(cases) >= 100 and any(not c["optimal"] for c in cases) and any(c["optimal"] for c in cases)
    for c in cases:
        rows = [tuple(r) for r in c["items"]]
        got = _search(rows, c["bottom"], c["node_cap"], _incumbent(rows, c["bottom"]))
        assert got == (_offs(c["offsets"]), c["capacity"], c["optimal"], c["nodes"]), c


def test_search_argument_checks():
    lib = _lib.lib()
    cap, nodes, opt = C.c_int64(0), C.c_int64(0), C.c_int32(0)
    assert lib.rm_layout_search(0, None, None, None, None, None, 1, None, -1, 0.0, None,
                                C.byref(cap), C.byref(nodes), C.byref(opt)) == 0
    assert (cap.value, nodes.value, opt.value) == (0, 0, 1)
    assert lib.rm_layout_search(2, None, None, None, None, None, 1, None, -1, 0.0, None,
                                C.byref(cap), C.byref(nodes), C.byref(opt)) != 0


@pytest.mark.gpu
def test_exact_layout_searches_like_reference():
    from paper_2310_19295_b200.layout import LayoutItem, LayoutProblem, exact_layout, exact_layout_batch
    cases = golden("layout_search")["cases"]
    probs = [LayoutProblem(items=tuple(LayoutItem(*r) for r in c["items"]), activations_at_bottom=c["bottom"],
                           node_cap=c["node_cap"]) for c in cases]
    res = exact_layout_batch(probs)
    for c, r in zip(cases, res):
        assert (r.offsets, r.capacity, r.optimal, r.stats.nodes) == \
            (_offs(c["offsets"]), c["capacity"], c["optimal"], c["nodes"]), c
    one = exact_layout(probs[0])
    assert (one.offsets, one.capacity) == (_offs(cases[0]["offsets"]), cases[0]["capacity"])


def test_wide_components_match_reference_host():
    """Components of 65-120 items (layout_limit > 64): the search's masks span
    several 64-bit words; offsets, capacity, optimal flag and node count
    equal the reference's under node caps from 1 to 20k
    (tests/golden/wide_search.json)."""
    cases = golden("wide_search")["layouts"]
    assert len(cases) >= 40 and any(c["optimal"] for c in cases)
    assert min(len(c["items"]) for c in cases) > 64
    for c in cases:
        rows = [tuple(r) for r in c["items"]]
        got = _search(rows, c["bottom"], c["node_cap"], _incumbent(rows, c["bottom"]))
        assert got == (_offs(c["offsets"]), c["capacity"], c["optimal"], c["nodes"]), c["node_cap"]


@pytest.mark.gpu
def test_wide_exact_layout_product_path():
    from paper_2310_19295_b200.layout import LayoutItem, LayoutProblem, exact_layout_batch
    cases = golden("wide_search")["layouts"]
    probs = [LayoutProblem(items=tuple(LayoutItem(*r) for r in c["items"]), activations_at_bottom=c["bottom"],
                           node_cap=c["node_cap"]) for c in cases]
    for c, r in zip(cases, exact_layout_batch(probs)):
        assert (r.offsets, r.capacity, r.optimal, r.stats.nodes) == \
            (_offs(c["offsets"]), c["capacity"], c["optimal"], c["nodes"]), c["node_cap"]
