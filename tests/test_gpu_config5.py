"""BASELINE config 5 at its full size on one GPU: 1,048,576 counter-RNG Kahn
candidate orders on the GPT2-XL graph (11,217 ops), evaluated in chunks with
the first strict minimum kept on the device.  Size-independent checks: every
generated row is a valid schedule, the winner re-evaluated by the C oracle
has exactly the reported peak, the result does not depend on the chunking,
and a sampled chunk agrees between K1 v4, K1 v2 and the C oracle row by row."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import coracle
from oracle import memplan_oracle as O
from paper_2310_19295_b200 import evaluator as ev
from paper_2310_19295_b200 import graphgen as gg
from paper_2310_19295_b200.graph import load_graph
from paper_2310_19295_b200.sharding import evaluate_sharded

pytestmark = pytest.mark.gpu


def test_config5_full_size_one_gpu():
    """All 1,048,576 candidates: every GPU (peak, argmax, valid) equals the C
    oracle's (event-sweep mode, every host core) row for row, and the sharded
    search's answer is the first strict minimum over the whole id range
    (tests/oracles.py:46-56; planner.py:209-216)."""
    g = load_graph(gg.config_doc("gpt2-xl"))
    total, chunk = 1 << 20, 1 << 16
    res = evaluate_sharded(g, total, seed=0, chunk=chunk)
    assert res.local_range == (0, total) and res.local_valid == total
    cg = coracle.CGraph(g)
    peaks = np.empty(total, np.int64)
    valid = np.empty(total, bool)
    for c0 in range(0, total, chunk):
        orders = ev.generate_orders(g, 0, c0, chunk)
        p, a, v = (x.cpu().numpy() for x in ev.evaluate_orders(g, orders))
        want = coracle.eval_orders(cg, orders.cpu().numpy(), events=True)
        assert np.array_equal(v, want[2]), c0
        assert np.array_equal(p[v], want[0][want[2]]) and np.array_equal(a[v], want[1][want[2]]), c0
        peaks[c0:c0 + chunk], valid[c0:c0 + chunk] = want[0], want[2]
    assert valid.all()
    best = int(np.argmin(peaks))          # first index attaining the minimum
    assert (res.best_peak, res.best_id) == (int(peaks[best]), best)
    print(f"config 5: {total} candidates, {len(np.unique(peaks))} distinct peaks, "
          f"first strict min {int(peaks[best])} at id {best}")


def test_chunking_does_not_change_the_answer():
    g = load_graph(gg.config_doc("gpt2-small"))
    a = evaluate_sharded(g, 50_000, seed=3, chunk=7_000)
    b = evaluate_sharded(g, 50_000, seed=3, chunk=1 << 16)
    orders = ev.generate_orders(g, 3, 0, 50_000)
    peak, _, valid = ev.evaluate_orders(g, orders)
    want = O.first_strict_min(peak.cpu().tolist(), valid.cpu().tolist())
    assert (a.best_peak, a.best_id) == (b.best_peak, b.best_id) == want


def test_gpt2xl_chunk_three_ways():
    g = load_graph(gg.config_doc("gpt2-xl"))
    orders = ev.generate_orders(g, 0, 777_000, 3_000)
    host = orders.cpu().numpy()
    host[::101] = host[::101][:, ::-1]                 # invalid rows mixed in
    want = coracle.eval_orders(coracle.CGraph(g), host)
    for variant in (5, 6, 4):
        ev.set_k1_variant(variant)
        try:
            p, a, v = (x.cpu().numpy() for x in ev.evaluate_orders(g, orders.new_tensor(host)))
        finally:
            ev.set_k1_variant(0)
        assert np.array_equal(v, want[2])
        assert np.array_equal(p[v], want[0][v]) and np.array_equal(a[v], want[1][v])
