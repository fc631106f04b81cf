"""Pin the CPU oracle against golden vectors frozen from the real reference
(tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden
from oracle import coracle
from oracle import memplan_oracle as O
from paper_2310_19295_b200 import graphgen as gg
from paper_2310_19295_b200.graph import load_graph


def _expect(e):
    return ("err", e["error"], e["message"]) if isinstance(e, dict) else ("ok", tuple(e))


def _oracle_peak(g, order):
    n = len(g.ops)
    try:
        if any((not isinstance(v, int)) or v < 0 or v >= n for v in order):
            raise IndexError("list assignment index out of range")
        return ("ok", O.peak_memory(g, order))
    except O.OracleScheduleError as e:
        return ("err", "ScheduleError", str(e))
    except IndexError as e:
        return ("err", "IndexError", str(e))


def test_fixture_peaks_match_reference():
    P = golden("peaks")
    graphs = {k: load_graph(v) for k, v in P["fixtures"].items()}
    for c in P["cases"]:
        got = _oracle_peak(graphs[c["graph"]], c["order"])
        want = _expect(c["expect"])
        if want[0] == "err" and want[1] == "IndexError":
            assert got[0] == "err"
        else:
            assert got == want, (c["graph"], c["order"])


def test_reference_unit_tests_known_answers():
    MB = 1 << 20
    g = load_graph(golden("peaks")["fixtures"]["diamond"])
    assert O.peak_memory(g, (0, 1, 2, 3)) == (120 * MB, 1)      # test_graph.py:124-128
    assert O.peak_memory(g, (0, 2, 1, 3))[0] == 90 * MB          # test_graph.py:130-132
    single = load_graph(golden("peaks")["fixtures"]["single"])
    assert O.peak_memory(single, (0,)) == (8, 0)                 # test_graph.py:135-140


@pytest.mark.parametrize("corpus", ["small_dags", "random_dags", "training"])
def test_corpus_peaks_match_reference(corpus):
    for entry in golden("peaks")[corpus]:
        g = load_graph(entry["doc"])
        for row in entry["rows"]:
            assert _oracle_peak(g, row["order"]) == _expect(row["expect"])


def test_config_graph_candidates_match_reference():
    for entry in golden("peaks")["configs"]:
        doc = gg.config_doc(entry["graph"])
        assert gg.doc_sha256(doc) == entry["doc_sha256"], "generator drifted from the frozen graph"
        g = load_graph(doc)
        preds, succs = O.direct_preds(g), O.direct_succs(g)
        cg = coracle.CGraph(g)
        for row in entry["rows"][:6]:
            o = O.kahn_candidate(len(g.ops), preds, succs, row["seed"], row["id"])
            assert hashlib.sha256(",".join(map(str, o)).encode()).hexdigest()[:16] == row["order_sha"]
            peak, arg, val = coracle.eval_orders(cg, np.array([o], np.int32))
            assert val[0] and (int(peak[0]), int(arg[0])) == tuple(row["expect"])


def test_c_oracle_matches_python_oracle():
    for entry in golden("peaks")["training"] + golden("peaks")["random_dags"]:
        g = load_graph(entry["doc"])
        cg = coracle.CGraph(g)
        orders = [r["order"] for r in entry["rows"]]
        peak, arg, val = coracle.eval_orders(cg, np.array(orders, np.int32), threads=2)
        for k, r in enumerate(entry["rows"]):
            want = _expect(r["expect"])
            if want[0] == "ok":
                assert val[k] and (int(peak[k]), int(arg[k])) == want[1]
            else:
                assert not val[k]


def test_event_sweep_oracle_matches_literal_oracle():
    """The C oracle's event-sweep mode (used to check million-row batches)
    returns what its literal per-step mode returns (graph.py:452-458) row for
    row: golden corpora, every config graph's candidates, corrupted rows."""
    from paper_2310_19295_b200 import graphgen as gg
    cases = []
    for entry in golden("peaks")["training"] + golden("peaks")["random_dags"]:
        cases.append((load_graph(entry["doc"]), np.array([r["order"] for r in entry["rows"]], np.int32)))
    rng = np.random.default_rng(0)
    for name in ("layered", "gpt2-small", "bert-large", "gpt2-xl"):
        g = load_graph(gg.config_doc(name))
        rows = coracle.kahn_orders(coracle.CGraph(g), 0, 0, 64)
        for r in range(0, 64, 5):
            i, j = rng.integers(0, rows.shape[1], 2)
            rows[r, [i, j]] = rows[r, [j, i]]
        rows[3, 0] = len(g.ops) + 2
        cases.append((g, rows))
    for g, rows in cases:
        cg = coracle.CGraph(g)
        a = coracle.eval_orders(cg, rows, threads=2)
        b = coracle.eval_orders(cg, rows, threads=2, events=True)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_schedules_match_reference():
    S = golden("schedules")
    fx = {k: load_graph(v) for k, v in golden("peaks")["fixtures"].items()}
    for c in S["packed"]:
        g = fx[c["graph"]]
        assert O.peak_memory(g, c["order"], c["timesteps"], c["ops_per_step"]) == tuple(c["peak"])
        assert [list(x) for x in O.tensor_lifetimes(g, c["timesteps"])] == c["lifetimes"]
        assert O.live_bytes_by_timestep(g, c["timesteps"]) == c["live"]
    for c in S["random"]:
        g = load_graph(c["doc"])
        assert O.peak_memory(g, c["order"], c["timesteps"], c["ops_per_step"]) == tuple(c["peak"])
        assert O.live_bytes_by_timestep(g, c["timesteps"]) == c["live"]
    g = fx["diamond"]
    for c in S["errors"]:
        try:
            O.validate_schedule(g, c["order"], c["timesteps"], c["ops_per_step"])
            got = None
        except O.OracleScheduleError as e:
            got = ("ScheduleError", str(e))
        except O.OracleConfigError as e:
            got = ("ConfigError", str(e))
        assert got == (None if c["error"] is None else (c["error"], c["message"]))


def _items(rows):
    return [tuple(r) for r in rows]


def test_layout_violations_match_reference():
    for c in golden("layouts")["violations"]:
        items = _items(c["items"])
        offsets = {int(k): v for k, v in c["offsets"].items()}
        assert O.layout_violations(items, offsets, c["capacity"]) == c["messages"]
        assert O.replay_static_extent(items, offsets) == c["replay_extent"]


def test_llfb_match_reference():
    for c in golden("layouts")["llfb"]:
        items = _items(c["items"])
        off, cap = O.llfb_layout(items)
        assert ({str(k): v for k, v in off.items()}, cap) == (c["llfb"]["offsets"], c["llfb"]["capacity"])
        off, cap = O.constrained_llfb_layout(items)
        assert ({str(k): v for k, v in off.items()}, cap) == (
            c["constrained"]["offsets"], c["constrained"]["capacity"])
    spec = golden("layouts")["spec"][0]
    off, cap = O.llfb_layout(_items(spec["items"]))
    assert cap == spec["capacity"] == 12 and off == {0: 0, 1: 8, 2: 8}


def test_component_incumbents_match_exact_layout_when_search_free():
    hit = 0
    for c in golden("layouts")["exact"]:
        items = _items(c["items"])
        off, cap, met, _ = O.component_incumbents(items)
        if met:  # reference returns the incumbent without search (layout.py:226)
            hit += 1
            assert cap == c["capacity"] and {str(k): v for k, v in off.items()} == c["offsets"]
            assert c["nodes"] == 0
    assert hit >= 20


def test_greedy_matches_reference():
    G = golden("greedy")
    for c in G["cases"]:
        doc = c.get("doc") or G["graphs"][c["graph"]]
        g = load_graph(doc)
        order, peak = O.greedy_order(g, c["ops"], c["live_in"], c["live_out"])
        assert list(order) == c["order"] and peak == c["peak"]
    trap = [c for c in G["cases"] if c.get("graph") == "greedy_trap0"][0]
    assert trap["exact_peak"] < trap["peak"]                       # SPEC AC7


def test_first_strict_min():
    assert O.first_strict_min([5, 3, 3, 1], [True, True, True, False]) == (3, 1)
    assert O.first_strict_min([5], [False]) == (None, -1)


def exact_cases():
    G = golden("exact")
    graphs = {k: load_graph(v) for k, v in G["graphs"].items()}
    for c in G["cases"]:
        yield (load_graph(c["doc"]) if "doc" in c else graphs[c["graph"]]), c


def test_exact_dp_matches_reference():
    """The order-ideal DP reproduces exact_order wherever the
    reference's search cannot hit its node cap (#ideals - 1 <= cap), and every
    case where the reference did hit it has more ideals than the cap."""
    decided = 0
    for g, c in exact_cases():
        dp = O.exact_order_dp(g, c["ops"], c["live_in"], c["live_out"], c["node_cap"])
        if dp is None:
            assert c["node_cap"] is not None
            continue
        decided += 1
        assert c["optimal"], c["graph"]
        assert (list(dp[0]), dp[1]) == (c["order"], c["peak"]), c["graph"]
        assert c["nodes"] <= dp[2] - 1            # each ideal expanded at most once
    assert decided >= 185
