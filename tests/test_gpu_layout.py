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


def _memplan():
    from paper_2310_19295_b200 import memplan_plugin as plug
    try:
        return plug.load_memplan()
    except ImportError:  # pragma: no cover
        pytest.skip("reference memplan not installed (baseline/_ref)")


@pytest.mark.parametrize("seed", range(6))
def test_repair_conflicts_device_rounds_vs_reference(seed):
    """rm_repair_conflicts (device detection + mover election, host C++
    placement) equals the reference's repair_conflicts (layout.py:409-470):
    offsets, capacity and the dict the result carries, on random problems
    from a handful of items up to 1,500 (several rounds, activations, zero
    sizes, items sharing offsets), with the ids unsorted in the input."""
    from paper_2310_19295_b200 import layout as L
    mp = _memplan()
    rng = random.Random(seed)
    for trial in range(40 if seed < 4 else 3):
        n = rng.randint(2, 60) if seed < 4 else rng.randint(800, 1500)
        items = []
        for t in rng.sample(range(4 * n), n):
            s = rng.randint(0, 30 if seed < 4 else 400)
            items.append(mp.layout.LayoutItem(t, rng.choice([0, 1, 2, 4, 8, 16, 48]), s,
                                              s + rng.randint(0, 8 if seed < 4 else 60), rng.random() < 0.3))
        slots = [0, 1, 2, 4, 8, 12, 16, 24, 32, 64]
        offs = {i.tensor: rng.choice(slots) for i in items}
        cap = max(offs[i.tensor] + i.size for i in items) + rng.choice([0, 0, 7])
        m = mp.layout.MemoryLayout(offsets=offs, capacity=cap)
        p = mp.layout.LayoutProblem(items=tuple(items))
        want = mp.layout.repair_conflicts(m, p)
        got = L.repair_conflicts(m, p)
        assert got == want and list(got.offsets) == list(want.offsets), (seed, trial)
        assert not L.conflict_pairs(sorted(items, key=lambda i: i.tensor), got.offsets)


def test_repair_conflicts_missing_offset_raises_like_reference():
    from paper_2310_19295_b200 import layout as L
    mp = _memplan()
    items = (mp.layout.LayoutItem(3, 4, 0, 2), mp.layout.LayoutItem(1, 4, 0, 2), mp.layout.LayoutItem(2, 4, 0, 2))
    m = mp.layout.MemoryLayout(offsets={1: 0}, capacity=4)
    p = mp.layout.LayoutProblem(items=items)
    with pytest.raises(KeyError) as want:
        mp.layout.repair_conflicts(m, p)
    with pytest.raises(KeyError) as got:
        L.repair_conflicts(m, p)
    assert got.value.args == want.value.args
