"""Host-side logic, no GPU needed: the C-ABI library loads and exports every
symbol include/roam.h declares; the host half of rm_graph_create (transitive
reduction, maximal consumers, event classes) restated in numpy reproduces the
oracle's peaks; generators and marshalling are deterministic."""

from __future__ import annotations

import ctypes as C
import re

import numpy as np
import pytest

from conftest import ROOT, golden
from oracle import memplan_oracle as O
from paper_2310_19295_b200 import _lib
from paper_2310_19295_b200 import graphgen as gg
from paper_2310_19295_b200.evaluator import DeviceGraph
from paper_2310_19295_b200.graph import graph_arrays, load_graph


def header_symbols() -> set[str]:
    text = (ROOT / "include" / "roam.h").read_text()
    return set(re.findall(r"^\s*(?:const\s+)?\w[\w\s\*]*?\b(rm_\w+)\s*\(", text, re.M))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, f"{s} missing from the ctypes table"


def test_device_entry_points_fail_loudly_without_gpu():
    if _lib.device_count() > 0:
        pytest.skip("GPU present")
    g = load_graph(golden("peaks")["fixtures"]["diamond"])
    dg = DeviceGraph(g)           # host-only handle works
    assert dg.info()["n_ops"] == 4
    from paper_2310_19295_b200 import evaluate_orders, peak_memory
    from paper_2310_19295_b200.graph import Schedule
    with pytest.raises(_lib.RoamError):
        evaluate_orders(g, np.array([[0, 2, 1, 3]], np.int32))
    with pytest.raises(_lib.RoamError):
        peak_memory(g, Schedule((0, 2, 1, 3), (0, 2, 1, 3)))
    from paper_2310_19295_b200.ordering import OrderingProblem, exact_order, greedy_order
    with pytest.raises(_lib.RoamError):
        exact_order(OrderingProblem(g, (0, 1, 2, 3)))
    with pytest.raises(_lib.RoamError):
        greedy_order(OrderingProblem(g, (0, 1, 2, 3)))
    from paper_2310_19295_b200.layout import LayoutItem, repair_conflicts
    from types import SimpleNamespace
    with pytest.raises(_lib.RoamError):
        repair_conflicts(SimpleNamespace(offsets={0: 0, 1: 0}, capacity=4),
                         SimpleNamespace(items=(LayoutItem(0, 4, 0, 1), LayoutItem(1, 4, 0, 1))))


def k1_numpy(meta: dict, n: int, order) -> tuple[int, int, bool]:
    """The K1 reformulation (csrc/roam_internal.h K1Meta) in numpy."""
    o = np.asarray(order, np.int64)
    if n == 0:
        return 0, 0, len(o) == 0
    if len(o) != n or o.min() < 0 or o.max() >= n or len(np.unique(o)) != n:
        return 0, 0, False
    pos = np.empty(n, np.int64)
    pos[o] = np.arange(n)
    if len(meta["edge_u"]) and np.any(pos[meta["edge_u"]] >= pos[meta["edge_v"]]):
        return 0, 0, False
    mf = np.zeros(max(int(meta["slot"].max()) + 1, 1), np.int64)
    for m in range(len(meta["msize"])):
        cons = meta["mcons"][meta["mptr"][m]:meta["mptr"][m + 1]]
        c = cons[np.argmax(pos[cons])]
        mf[meta["slot"][c]] += meta["msize"][m]
    outb = meta["out_tab"][meta["vidx"][o]]
    freed = meta["fs_tab"][meta["vidx"][o]] + np.where(meta["slot"][o] >= 0, mf[meta["slot"][o]], 0)
    x = outb.copy()
    x[1:] -= freed[:-1]
    live = np.cumsum(x)
    k = int(np.argmax(live))
    return int(live[k]), k, True


def _check_graph(g, orders, reduce=True):
    dg = DeviceGraph(g, reduce=reduce)
    meta = dg.k1_export()
    preds = O.direct_preds(g)
    for order in orders:
        p, a, v = O.evaluate_order(g, list(order), preds=preds)
        got = k1_numpy(meta, len(g.ops), order)
        assert got[2] == v, order
        if v:
            assert got[:2] == (p, a), order
    return dg.info()


@pytest.mark.parametrize("reduce", [True, False])
def test_k1_reformulation_on_fixtures_and_corpora(reduce):
    P = golden("peaks")
    graphs = {k: load_graph(v) for k, v in P["fixtures"].items()}
    by_graph: dict[str, list] = {}
    for c in P["cases"]:
        by_graph.setdefault(c["graph"], []).append(c["order"])
    for name, orders in by_graph.items():
        _check_graph(graphs[name], orders, reduce)
    for corpus in ("small_dags", "random_dags", "training"):
        for e in P[corpus]:
            _check_graph(load_graph(e["doc"]), [r["order"] for r in e["rows"]], reduce)


def test_k1_reformulation_on_config_graphs():
    for name in ("layered", "gpt2-small"):
        g = load_graph(gg.config_doc(name))
        preds, succs = O.direct_preds(g), O.direct_succs(g)
        orders = [O.kahn_candidate(len(g.ops), preds, succs, 0, c) for c in range(3)]
        info = _check_graph(g, orders)
        assert info["reduced"] == 1
        assert info["n_check_edges"] <= info["n_pred_edges"]


def test_reduction_shrinks_training_graphs():
    g = load_graph(gg.config_doc("gpt2-small"))
    i = DeviceGraph(g).info()
    assert i["n_check_edges"] < i["n_pred_edges"]
    assert i["n_multi"] < sum(1 for t in g.tensors if len(set(t.consumers)) >= 2)
    assert i["wide_index"] == 0


def test_graph_create_rejects_bad_csr():
    L = _lib.lib()
    size = np.array([4], np.int64)
    producer = np.array([3], np.int32)  # out of range
    cp = np.array([0, 0], np.int32)
    ip = np.array([0, 0], np.int32)
    d = _lib.RmGraphDesc(1, 1, size.ctypes.data, producer.ctypes.data, cp.ctypes.data, None,
                         ip.ctypes.data, None, ip.ctypes.data, None)
    h = C.c_void_p()
    assert L.rm_graph_create(C.byref(d), 0, C.byref(h)) != 0
    assert b"producer" in L.rm_last_error()


def test_generators_deterministic():
    for name in ("layered", "gpt2-small", "bert-large", "gpt2-xl"):
        assert gg.doc_sha256(gg.config_doc(name)) == gg.doc_sha256(gg.config_doc(name))
    g = load_graph(gg.config_doc("gpt2-small"))
    a = graph_arrays(g)
    assert a.n_ops == len(g.ops) and a.cons_ptr[-1] == len(a.cons_idx)
    kinds = {op.kind.value for op in g.ops}
    assert kinds == {"forward", "backward", "weight_update", "loss"}


def test_kahn_candidates_are_topological():
    g = load_graph(gg.config_doc("layered"))
    preds, succs = O.direct_preds(g), O.direct_succs(g)
    seen = set()
    for c in range(4):
        o = O.kahn_candidate(len(g.ops), preds, succs, 0, c)
        O.validate_schedule(g, o, O.sequential_timesteps(len(g.ops), o))
        seen.add(tuple(o))
    assert len(seen) == 4


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the driver's reference arm) runs on the host
    alone and prints the contract's JSON line: impl, the metric of our arm,
    a cpu_baseline describing the run and an e2e object with zero copies."""
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "3",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "candidate plans evaluated/sec"
    assert line["unit"] == "candidates/s" and line["higher_is_better"] is True
    assert line["steps"] == 3 and line["warmup"] == 1 and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_load_graph_matches_reference_loader():
    """The CSR-first loader builds the reference's graph (graph.py:188-278):
    same ops, tensors, consumer entries and categories on the config graphs
    and the reference's own generators, and the same exception class and
    message, in the same order, on malformed documents."""
    import sys
    from pathlib import Path
    ref = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    rg = pytest.importorskip("memplan.graph")
    rgen = pytest.importorskip("memplan.graphgen")
    from paper_2310_19295_b200 import graphgen as gg
    docs = [gg.config_doc(n) for n in ("layered", "gpt2-small", "bert-large")]
    docs += [rg.graph_to_doc(rgen.gen_training_graph(a, 3, optimizer=o))
             for a in ("mlp", "residual", "transformer_block") for o in ("sgd", "adam")]
    docs += [rg.graph_to_doc(rgen.gen_random_dag(12 + k, density=0.3, seed=k)) for k in range(6)]
    for d in docs:
        a, b = rg.load_graph(d), load_graph(d)
        assert [(o.id, o.name, o.kind.value, o.inputs, o.outputs) for o in a.ops] == \
               [(o.id, o.name, o.kind.value, o.inputs, o.outputs) for o in b.ops]
        assert [(t.id, t.size, t.producer, t.consumers, t.category.value) for t in a.tensors] == \
               [(t.id, t.size, t.producer, t.consumers, t.category.value) for t in b.tensors]
    bad = [
        {"tensors": []},
        {"ops": [], "tensors": [{"id": 1, "size_bytes": 3}, {"id": 1, "size_bytes": 3}]},
        {"ops": [{"id": "a"}], "tensors": []},
        {"ops": [{"id": 0, "outputs": [5]}], "tensors": [{"id": 1, "size_bytes": 3}]},
        {"ops": [{"id": 0, "outputs": [1]}, {"id": 1, "outputs": [1]}], "tensors": [{"id": 1, "size_bytes": 3}]},
        {"ops": [{"id": 0, "outputs": [1, 1]}], "tensors": [{"id": 1, "size_bytes": 3}]},
        {"ops": [{"id": 0, "outputs": [1, 7]}, {"id": 1, "outputs": [1]}], "tensors": [{"id": 1, "size_bytes": 3}]},
        {"ops": [{"id": 0, "outputs": [1], "kind": "zz"}], "tensors": [{"id": 1, "size_bytes": 3}]},
        {"ops": [{"id": 0, "outputs": []}], "tensors": [{"id": 1, "size_bytes": 3}]},
        {"ops": [{"id": 0, "outputs": [1]}], "tensors": [{"id": 1, "size_bytes": "x"}]},
        {"ops": [{"id": 0, "outputs": [1]}], "tensors": [{"id": 1, "size_bytes": 3, "category": "nope"}]},
        {"ops": [{"id": 0, "outputs": [1], "inputs": [2]}, {"id": 1, "outputs": [2], "inputs": [1]}],
         "tensors": [{"id": 1, "size_bytes": 3}, {"id": 2, "size_bytes": 3}]},
    ]
    for d in bad:
        with pytest.raises(Exception) as want:
            rg.load_graph(d)
        with pytest.raises(Exception) as got:
            load_graph(d)
        assert (type(got.value).__name__, str(got.value)) == (type(want.value).__name__, str(want.value))
