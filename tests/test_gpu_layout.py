"""K2 (pairwise time x address interference) against the reference's golden
layout vectors and the oracle; exact messages and order."""

from __future__ import annotations

import random

import pytest

from conftest import golden
from oracle import memplan_oracle as O
from paper_2310_19295_b200.layout import LayoutItem, conflict_pairs, layout_violations

pytestmark = pytest.mark.gpu


def _items(rows):
    return [LayoutItem(*r) for r in rows]


def test_violations_golden():
    for c in golden("layouts")["violations"]:
        items = _items(c["items"])
        offsets = {int(k): v for k, v in c["offsets"].items()}
        assert layout_violations(items, offsets, c["capacity"]) == c["messages"]


def test_spec_messages():
    spec = golden("layouts")["spec"][1]
    assert layout_violations([LayoutItem(0, 4, 0, 3), LayoutItem(1, 4, 2, 5)], {0: 0, 1: 2}, 8) == spec["a"]
    assert layout_violations([LayoutItem(0, 4, 0, 3)], {0: 2}, 4) == spec["b"]


@pytest.mark.parametrize("N", [1, 127, 128, 129, 700, 3000])
def test_large_random_vs_oracle(N):
    rng = random.Random(N)
    rows = []
    for t in range(N):
        s = rng.randint(0, 200)
        rows.append((t, rng.randint(1, 64), s, s + rng.randint(0, 40), False))
    offsets = {t: rng.randint(0, 4000) for t in range(N) if rng.random() > 0.01}
    items = _items(rows)
    cap = 3500
    assert layout_violations(items, offsets, cap) == O.layout_violations(rows, offsets, cap)
    pairs = conflict_pairs(items, {t: offsets.get(t, 0) for t in range(N)})
    want = [(i, j) for i in range(N) for j in range(i + 1, N)
            if O.overlaps(rows[i], rows[j]) and offsets.get(i, 0) < offsets.get(j, 0) + rows[j][1]
            and offsets.get(j, 0) < offsets.get(i, 0) + rows[i][1]] if N <= 700 else None
    if want is not None:
        assert pairs == want


def test_replay_extent_golden():
    """replay_static's actual extent (simulator.py:137-145: the max over steps
    of max(off + size) over live items with offsets = the max over all such
    items, never below 0) from K2's epilogue, on every golden layout."""
    from paper_2310_19295_b200.layout import _k2
    for c in golden("layouts")["violations"]:
        items = [LayoutItem(*r) for r in c["items"]]
        offs = {int(k): v for k, v in c["offsets"].items()}
        _, _, _, mx = _k2(items, offs, c["capacity"], 16)
        assert mx == max(c["replay_extent"], 0), c
