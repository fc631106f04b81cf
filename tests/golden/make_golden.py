"""Freeze golden vectors from the REAL reference (pkg/src/memplan).

Run in the build container (the reference is importable there, not on the GPU
box):  python tests/golden/make_golden.py
Writes tests/golden/*.json; the tests check both the oracle and the CUDA path
against them.  Deterministic: every input comes from seeded generators.
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

from memplan import graph as rg  # noqa: E402
from memplan import layout as rl  # noqa: E402
from memplan import ordering as ro  # noqa: E402
from memplan import planner as rp  # noqa: E402
from memplan import simulator as rs  # noqa: E402
from memplan.graphgen import gen_random_dag, gen_training_graph, gen_greedy_trap  # noqa: E402

from oracle.memplan_oracle import direct_preds, direct_succs, kahn_candidate  # noqa: E402
from paper_2310_19295_b200 import graphgen as gg  # noqa: E402

MB = 1 << 20


def dump(name: str, obj) -> None:
    (HERE / name).write_text(json.dumps(obj, sort_keys=True, separators=(",", ":")) + "\n")
    print(f"wrote {name}: {(HERE / name).stat().st_size} bytes")


def diamond_doc():
    return {"ops": [
        {"id": 0, "name": "A", "kind": "forward", "inputs": [], "outputs": [0, 1]},
        {"id": 1, "name": "B", "kind": "forward", "inputs": [1], "outputs": [2]},
        {"id": 2, "name": "C", "kind": "forward", "inputs": [0], "outputs": [3]},
        {"id": 3, "name": "D", "kind": "forward", "inputs": [2, 3], "outputs": []}],
        "tensors": [{"id": 0, "size_bytes": 60 * MB}, {"id": 1, "size_bytes": 20 * MB},
                    {"id": 2, "size_bytes": 40 * MB}, {"id": 3, "size_bytes": 10 * MB}]}


def chain_doc(k, size=MB):
    ops, tensors = [], []
    for i in range(k):
        ops.append({"id": i, "name": f"n{i}", "kind": "forward",
                    "inputs": [i - 1] if i else [], "outputs": [i] if i < k - 1 else []})
        if i < k - 1:
            tensors.append({"id": i, "size_bytes": size})
    return {"ops": ops, "tensors": tensors}


def edge_docs():
    """h1 duplicate input, h2 self-consuming op, h3 zero-consumer outputs."""
    h1 = {"ops": [
        {"id": 0, "name": "a", "kind": "forward", "inputs": [], "outputs": [0]},
        {"id": 1, "name": "b", "kind": "forward", "inputs": [0, 0], "outputs": [1]},
        {"id": 2, "name": "c", "kind": "forward", "inputs": [1], "outputs": [2]},
        {"id": 3, "name": "d", "kind": "forward", "inputs": [2, 0], "outputs": []}],
        "tensors": [{"id": 0, "size_bytes": 30 * MB}, {"id": 1, "size_bytes": 20 * MB},
                    {"id": 2, "size_bytes": 10 * MB}]}
    h1b = {"ops": [
        {"id": 0, "name": "a", "kind": "forward", "inputs": [], "outputs": [0, 1]},
        {"id": 1, "name": "b", "kind": "forward", "inputs": [0, 0], "outputs": [2]},
        {"id": 2, "name": "c", "kind": "forward", "inputs": [1, 2, 1], "outputs": [3]},
        {"id": 3, "name": "d", "kind": "forward", "inputs": [3], "outputs": []}],
        "tensors": [{"id": 0, "size_bytes": 40 * MB}, {"id": 1, "size_bytes": 10 * MB},
                    {"id": 2, "size_bytes": 20 * MB}, {"id": 3, "size_bytes": 5 * MB}]}
    h2 = {"ops": [
        {"id": 0, "name": "a", "kind": "forward", "inputs": [], "outputs": [0]},
        {"id": 1, "name": "self", "kind": "forward", "inputs": [0, 1], "outputs": [1, 2]},
        {"id": 2, "name": "c", "kind": "forward", "inputs": [2], "outputs": [3]},
        {"id": 3, "name": "d", "kind": "forward", "inputs": [1, 3], "outputs": []}],
        "tensors": [{"id": 0, "size_bytes": 7}, {"id": 1, "size_bytes": 11},
                    {"id": 2, "size_bytes": 13}, {"id": 3, "size_bytes": 17}]}
    h3 = {"ops": [
        {"id": 0, "name": "a", "kind": "forward", "inputs": [], "outputs": [0, 1]},
        {"id": 1, "name": "b", "kind": "forward", "inputs": [0], "outputs": [2]},
        {"id": 2, "name": "c", "kind": "forward", "inputs": [], "outputs": [3]},
        {"id": 3, "name": "d", "kind": "forward", "inputs": [2], "outputs": []}],
        "tensors": [{"id": 0, "size_bytes": 5}, {"id": 1, "size_bytes": 100},
                    {"id": 2, "size_bytes": 3}, {"id": 3, "size_bytes": 50}]}
    single = {"ops": [{"id": 0, "name": "A", "kind": "forward", "inputs": [], "outputs": [0]}],
              "tensors": [{"id": 0, "size_bytes": 8}]}
    empty = {"ops": [], "tensors": []}
    no_tensors = {"ops": [{"id": 0, "name": "x", "kind": "forward", "inputs": [], "outputs": []},
                          {"id": 1, "name": "y", "kind": "forward", "inputs": [], "outputs": []}],
                  "tensors": []}
    return {"h1_dup_input": h1, "h1b_dup_input": h1b, "h2_self_consume": h2,
            "h3_zero_consumer": h3, "single": single, "empty": empty, "no_tensors": no_tensors,
            "diamond": diamond_doc(), "chain5": chain_doc(5)}


def small_dag_doc(rng: random.Random, max_ops=7):
    """test_graph.py:215-233 small_dags shape, drawn from a seeded RNG."""
    n = rng.randint(1, max_ops)
    ops, tensors = [], []
    for i in range(n):
        parents = sorted(rng.sample(range(i), rng.randint(0, min(i, 3)))) if i else []
        ops.append({"id": i, "name": f"v{i}", "kind": "forward", "inputs": parents, "outputs": [i]})
        tensors.append({"id": i, "size_bytes": rng.randint(1, 8) * MB})
    return {"ops": ops, "tensors": tensors}


def all_orders(g, cap=200):
    n = g.n_ops
    indeg = [len(p) for p in g.direct_preds]
    order, out = [], []

    def rec():
        if len(out) >= cap:
            return
        if len(order) == n:
            out.append(tuple(order))
            return
        for v in range(n):
            if indeg[v] == 0 and v not in order:
                order.append(v)
                for w in g.direct_succs[v]:
                    indeg[w] -= 1
                rec()
                for w in g.direct_succs[v]:
                    indeg[w] += 1
                order.pop()
    rec()
    return out


def ref_peak(g, order):
    try:
        return list(rg.peak_memory(g, rg.sequential_schedule(g, order)))
    except (rg.ScheduleError, IndexError) as e:  # out-of-range ids raise IndexError (graph.py:406)
        return {"error": type(e).__name__, "message": str(e)}


def order_hash(order) -> str:
    return hashlib.sha256(",".join(map(str, order)).encode()).hexdigest()[:16]


# ------------------------------------------------------------------ peaks

def make_peaks():
    rng = random.Random(20231029)
    cases = []
    docs = edge_docs()
    for name, doc in docs.items():
        g = rg.load_graph(doc)
        orders = all_orders(g, cap=50)
        n = g.n_ops
        bad = []
        if n >= 2:
            o = list(orders[0])
            bad.append(o[::-1])                       # usually pred-violating
            bad.append(o[:-1] + [o[0]])                # duplicate
            bad.append(o[:-1] + [n])                   # out of range
            bad.append(o[:-1])                         # short
        for order in orders + bad:
            cases.append({"graph": name, "order": list(order), "expect": ref_peak(g, order)})
    # hypothesis-style small DAG corpus: all orders (capped) of 150 DAGs
    small = []
    for k in range(150):
        doc = small_dag_doc(rng)
        g = rg.load_graph(doc)
        orders = all_orders(g, cap=24)
        rows = [{"order": list(o), "expect": ref_peak(g, o)} for o in orders]
        o = list(orders[0])
        if len(o) >= 2:
            rows.append({"order": o[::-1], "expect": ref_peak(g, o[::-1])})
        small.append({"doc": doc, "rows": rows})
    # random DAGs from the reference generator (denser, up to 14 ops)
    rdags = []
    for k in range(40):
        g = rg.load_graph(rg.graph_to_doc(gen_random_dag(6 + k % 9, density=0.3 + 0.1 * (k % 4), seed=k)))
        preds, succs = direct_preds(g), direct_succs(g)
        rows = []
        for cid in range(20):
            o = kahn_candidate(g.n_ops, preds, succs, seed=7, cand_id=cid)
            rows.append({"order": o, "expect": ref_peak(g, o)})
        rdags.append({"doc": rg.graph_to_doc(g), "rows": rows})
    # training graphs from the reference generator (duplicate consumers etc.)
    tg = []
    for arch in ("mlp", "residual", "transformer_block"):
        for opt in ("sgd", "adam"):
            g = gen_training_graph(arch, 3, optimizer=opt)
            preds, succs = direct_preds(g), direct_succs(g)
            rows = []
            for cid in range(16):
                o = kahn_candidate(g.n_ops, preds, succs, seed=11, cand_id=cid)
                rows.append({"order": o, "expect": ref_peak(g, o)})
            rows.append({"order": list(range(g.n_ops)), "expect": ref_peak(g, range(g.n_ops))})
            tg.append({"doc": rg.graph_to_doc(g), "rows": rows})
    # config graphs: candidates identified by (seed, id) and order hash
    cfg = []
    for name, count in (("layered", 24), ("gpt2-small", 16), ("bert-large", 6), ("gpt2-xl", 4)):
        doc = gg.config_doc(name)
        g = rg.load_graph(doc)
        preds, succs = direct_preds(g), direct_succs(g)
        rows = []
        for cid in range(count):
            o = kahn_candidate(g.n_ops, preds, succs, seed=0, cand_id=cid)
            rows.append({"seed": 0, "id": cid, "order_sha": order_hash(o), "expect": ref_peak(g, o)})
        cfg.append({"graph": name, "doc_sha256": gg.doc_sha256(doc), "n_ops": g.n_ops, "rows": rows})
    dump("peaks.json", {"fixtures": docs, "cases": cases, "small_dags": small,
                        "random_dags": rdags, "training": tg, "configs": cfg})


# ------------------------------------------------------- schedules (general)

def make_schedules():
    rng = random.Random(5)
    out = []
    docs = edge_docs()
    for name in ("diamond", "h1_dup_input", "h2_self_consume", "h3_zero_consumer", "chain5"):
        g = rg.load_graph(docs[name])
        for k in (1, 2, 3):
            for order in all_orders(g, cap=6):
                s = rg.pack_schedule(g, order, k)
                out.append({"graph": name, "order": list(s.order), "timesteps": list(s.timesteps),
                            "ops_per_step": k, "peak": list(rg.peak_memory(g, s)),
                            "lifetimes": [list(x) for x in rg.tensor_lifetimes(g, s)],
                            "live": rg.live_bytes_by_timestep(g, s)})
    # validation errors with messages, each check in turn
    g = rg.load_graph(docs["diamond"])
    bad = [((0, 1, 2, 3), (0, 1, 1, 2), 1), ((0, 1, 2, 3), (0, 2, 1, 3), 1), ((0, 1, 2, 3), (0, 1, 2), 1),
           ((0, 1, 2, 3), (0, 1, 2, 3), 0), ((0, 2, 1, 3), (0, 1, 1, 1), 2), ((3, 0, 1, 2), (1, 2, 3, 0), 1),
           ((0, 1, 1, 3), (0, 1, 2, 3), 1), ((0, 1, 2), (0, 1, 2, 3), 1), ((1, 0, 2, 3), (1, 0, 2, 3), 1),
           ((0, 3, 1, 2), (0, 2, 3, 1), 1), ((0, 1, 2, 3), (0, 0, 0, 0), 4), ((0, 1, 2, 3), (0, 0, 0, 0), 3)]
    errs = []
    for order, ts, k in bad:
        s = rg.Schedule(order=order, timesteps=ts, ops_per_step=k)
        try:
            rg.validate_schedule(g, s)
            errs.append({"order": list(order), "timesteps": list(ts), "ops_per_step": k, "error": None,
                         "peak": list(rg.peak_memory(g, s))})
        except rg.GraphError as e:
            errs.append({"order": list(order), "timesteps": list(ts), "ops_per_step": k,
                         "error": type(e).__name__, "message": str(e)})
    # random packed schedules on random DAGs
    rnd = []
    for k in range(30):
        g = gen_random_dag(8 + k % 7, density=0.3, seed=100 + k)
        o = kahn_candidate(g.n_ops, direct_preds(g), direct_succs(g), seed=3, cand_id=k)
        s = rg.pack_schedule(g, o, 1 + k % 3)
        rnd.append({"doc": rg.graph_to_doc(g), "order": list(s.order), "timesteps": list(s.timesteps),
                    "ops_per_step": s.ops_per_step, "peak": list(rg.peak_memory(g, s)),
                    "lifetimes": [list(x) for x in rg.tensor_lifetimes(g, s)],
                    "live": rg.live_bytes_by_timestep(g, s)})
    dump("schedules.json", {"packed": out, "errors": errs, "random": rnd})


# ----------------------------------------------------------------- layouts

def rand_items(rng, n, act_p=0.3, horizon=None):
    horizon = horizon or max(4, n)
    items = []
    ids = rng.sample(range(3 * n), n)
    for t in ids:
        s = rng.randint(0, horizon - 1)
        e = min(horizon - 1, s + rng.randint(0, horizon // 2))
        items.append(rl.LayoutItem(tensor=t,
                                   size=rng.choice([1, 2, 3, 4, 8, 16]) * MB // rng.choice([1, 2, 4]),
                                   start=s, end=e, is_activation=rng.random() < act_p))
    return items


def it_row(i):
    return [i.tensor, i.size, i.start, i.end, bool(i.is_activation)]


def make_layouts():
    rng = random.Random(99)
    viol = []
    for k in range(80):
        items = rand_items(rng, rng.randint(1, 40))
        offsets = {}
        for i in items:
            r = rng.random()
            if r < 0.05:
                continue
            offsets[i.tensor] = -rng.randint(1, 4) if r < 0.08 else rng.randint(0, 24) * MB // 2
        cap = rng.randint(8, 40) * MB
        msgs = rl.layout_violations(items, offsets, cap)
        viol.append({"items": [it_row(i) for i in items], "offsets": {str(a): b for a, b in offsets.items()},
                     "capacity": cap, "messages": msgs,
                     "replay_extent": max((offsets[i.tensor] + i.size for i in items if i.tensor in offsets),
                                          default=0)})
    # SPEC examples
    spec = []
    x, y, z = (rl.LayoutItem(0, 8, 0, 10), rl.LayoutItem(1, 4, 0, 3), rl.LayoutItem(2, 4, 4, 10))
    m = rl.llfb_layout(rl.LayoutProblem(items=(x, y, z)))
    spec.append({"kind": "llfb", "items": [it_row(i) for i in (x, y, z)],
                 "offsets": {str(a): b for a, b in m.offsets.items()}, "capacity": m.capacity})
    v1 = rl.layout_violations([rl.LayoutItem(0, 4, 0, 3), rl.LayoutItem(1, 4, 2, 5)], {0: 0, 1: 2}, 8)
    v2 = rl.layout_violations([rl.LayoutItem(0, 4, 0, 3)], {0: 2}, 4)
    spec.append({"kind": "violations", "a": v1, "b": v2})
    llfb = []
    for k in range(60):
        items = rand_items(rng, rng.randint(1, 60), act_p=0.35)
        p = rl.LayoutProblem(items=tuple(items), activations_at_bottom=True)
        a = rl.llfb_layout(p)
        b = rl.constrained_llfb_layout(p)
        llfb.append({"items": [it_row(i) for i in items],
                     "llfb": {"offsets": {str(t): o for t, o in a.offsets.items()}, "capacity": a.capacity},
                     "constrained": {"offsets": {str(t): o for t, o in b.offsets.items()},
                                     "capacity": b.capacity}})
    exact = []
    for k in range(60):
        items = rand_items(rng, rng.randint(1, 14), act_p=0.3)
        p = rl.LayoutProblem(items=tuple(items), activations_at_bottom=True, node_cap=200_000)
        m = rl.exact_layout(p)
        exact.append({"items": [it_row(i) for i in items], "offsets": {str(t): o for t, o in m.offsets.items()},
                      "capacity": m.capacity, "optimal": m.optimal, "nodes": m.stats.nodes})
    dump("layouts.json", {"violations": viol, "spec": spec, "llfb": llfb, "exact": exact})


# ---------------------------------------------------------- layout search

def make_layout_search():
    """exact_layout problems whose incumbent misses its bound, so the
    reference's branch-and-bound runs (layout.py:226-290): both activation
    modes, full searches and node-capped ones (optimal=False, partial best)."""
    rng = random.Random(23)
    cases = []
    tries = 0
    while len(cases) < 120 and tries < 20000:
        tries += 1
        n = rng.randint(3, 16)
        items = rand_items(rng, n, act_p=0.3, horizon=rng.choice([3, 4, 6, n]))
        bottom = rng.random() < 0.6
        p = rl.LayoutProblem(items=tuple(items), activations_at_bottom=bottom, node_cap=200_000)
        m = rl.exact_layout(p)
        if m.stats.nodes == 0:
            continue
        runs = [(200_000, m)]
        for cap in sorted({1, max(1, m.stats.nodes // 3), max(1, m.stats.nodes - 1)}):
            q = rl.LayoutProblem(items=tuple(items), activations_at_bottom=bottom, node_cap=cap)
            runs.append((cap, rl.exact_layout(q)))
        for cap, r in runs:
            cases.append({"items": [it_row(i) for i in items], "bottom": bottom, "node_cap": cap,
                          "offsets": {str(t): o for t, o in r.offsets.items()}, "capacity": r.capacity,
                          "optimal": r.optimal, "nodes": r.stats.nodes})
    dump("layout_search.json", {"cases": cases})


# ---------------------------------------------------------------- greedy

def make_greedy():
    out = []
    graphs = {}
    for k in range(30):
        g = gen_random_dag(5 + k % 12, density=0.25 + 0.05 * (k % 5), seed=500 + k)
        sol = ro.greedy_order(ro.whole_graph_problem(g))
        out.append({"doc": rg.graph_to_doc(g), "ops": list(range(g.n_ops)), "live_in": [], "live_out": [],
                    "order": list(sol.order), "peak": sol.peak})
    for name, doc in edge_docs().items():
        g = rg.load_graph(doc)
        sol = ro.greedy_order(ro.whole_graph_problem(g))
        out.append({"graph": name, "doc": doc, "ops": list(range(g.n_ops)), "live_in": [], "live_out": [],
                    "order": list(sol.order), "peak": sol.peak})
    # real window problems from the planner's own decomposition
    for arch in ("mlp", "residual", "transformer_block"):
        for blocks in (2, 4):
            g = gen_training_graph(arch, blocks, optimizer="adam")
            tree = rp.build_subgraph_tree(g, 20)
            lin = rp.linearize(g, tree)
            wu = rp.place_weight_updates(g, tree, 2.0)
            graphs[f"{arch}{blocks}"] = rg.graph_to_doc(g)
            for w, prob in ro.build_window_problems(g, lin, wu):
                sol = ro.greedy_order(prob)
                out.append({"graph": f"{arch}{blocks}", "ops": list(prob.ops),
                            "live_in": sorted(prob.live_in), "live_out": sorted(prob.live_out),
                            "order": list(sol.order), "peak": sol.peak})
    trap = gen_greedy_trap(0)
    sol = ro.greedy_order(ro.whole_graph_problem(trap))
    ex = ro.exact_order(ro.whole_graph_problem(trap))
    out.append({"graph": "greedy_trap0", "doc": rg.graph_to_doc(trap), "ops": list(range(trap.n_ops)),
                "live_in": [], "live_out": [], "order": list(sol.order), "peak": sol.peak,
                "exact_peak": ex.peak})
    dump("greedy.json", {"cases": out, "graphs": graphs})


# ------------------------------------------------------- exact order DFS

def make_exact_search():
    """exact_order's capped DFS (ordering.py:183-286) on wide windows -- the
    ones whose order ideals can outnumber a node cap -- under caps from tiny
    (the cap stops it: greedy incumbent, optimal=False) to roomy (the pruned
    search finishes: its order, peak and node count)."""
    from memplan.graphgen import gen_random_dag
    rng = random.Random(31)
    cases, graphs = [], {}
    for k in range(40):
        n = rng.randint(6, 18)
        g = gen_random_dag(n, density=rng.choice([0.05, 0.1, 0.15, 0.25]), seed=900 + k)
        name = f"dag{k}"
        graphs[name] = rg.graph_to_doc(g)
        windows = [(list(range(g.n_ops)), [], [])]
        for _ in range(2):
            ops, li, lo = random_window(g, rng)
            windows.append((ops, sorted(li), sorted(lo)))
        for ops, li, lo in windows:
            for cap in (rng.choice([1, 5, 20]), rng.choice([50, 200, 1000]), 500_000):
                prob = ro.OrderingProblem(graph=g, ops=tuple(ops), live_in=frozenset(li),
                                          live_out=frozenset(lo), node_cap=cap)
                try:
                    sol = ro.exact_order(prob)
                except rg.ConfigError as e:
                    cases.append({"graph": name, "ops": ops, "live_in": li, "live_out": lo,
                                  "node_cap": cap, "error": str(e)})
                    continue
                cases.append({"graph": name, "ops": ops, "live_in": li, "live_out": lo, "node_cap": cap,
                              "order": list(sol.order), "peak": sol.peak, "optimal": sol.optimal,
                              "nodes": sol.stats.nodes})
    dump("exact_search.json", {"cases": cases, "graphs": graphs})


# --------------------------------------- wide searches (beyond 64 bits)

def make_wide_search():
    """The two capped searches on problems wider than one 64-bit mask word
    (node_limit / layout_limit > 64): exact_order on windows of 65-140 ops
    (chain-like DAGs whose pruned DFS finishes, wide ones that a node cap
    stops) and exact_layout on overlap components of 65-120 items whose
    incumbent misses its bound, under node caps from 1 to 20k."""
    import time as _t
    rng = random.Random(47)
    orders, graphs = [], {}
    for k in range(24):
        n = rng.randint(65, 140)
        dens = rng.choice([0.02, 0.05, 0.3, 0.6, 0.9])
        g = gen_random_dag(n, density=dens, seed=1300 + k)
        name = f"wide{k}"
        graphs[name] = rg.graph_to_doc(g)
        for cap in (rng.choice([1, 10, 100]), rng.choice([1000, 5000]), 20_000):
            prob = ro.OrderingProblem(graph=g, ops=tuple(range(n)), node_cap=cap)
            t0 = _t.monotonic()
            sol = ro.exact_order(prob)
            orders.append({"graph": name, "ops": list(range(n)), "live_in": [], "live_out": [],
                           "node_cap": cap, "order": list(sol.order), "peak": sol.peak,
                           "optimal": sol.optimal, "nodes": sol.stats.nodes,
                           "ref_s": round(_t.monotonic() - t0, 3)})
    layouts = []
    tries = 0
    while len(layouts) < 48 and tries < 400:
        tries += 1
        n = rng.randint(65, 120)
        horizon = rng.choice([6, 10, 20])
        items = rand_items(rng, n, act_p=0.2, horizon=horizon)
        bottom = rng.random() < 0.5
        for cap in (1, rng.choice([50, 500]), 20_000):
            q = rl.LayoutProblem(items=tuple(items), activations_at_bottom=bottom, node_cap=cap)
            m = rl.exact_layout(q)
            if m.stats.nodes == 0:
                break
            layouts.append({"items": [it_row(i) for i in items], "bottom": bottom, "node_cap": cap,
                            "offsets": {str(t): o for t, o in m.offsets.items()}, "capacity": m.capacity,
                            "optimal": m.optimal, "nodes": m.stats.nodes})
    dump("wide_search.json", {"orders": orders, "graphs": graphs, "layouts": layouts})


# ---------------------------------------------------------------- exact

def random_window(g, rng):
    """A random op subset of g with its boundary liveness (live_in = consumed
    inside, produced outside; live_out = produced inside, consumed outside,
    plus a few extra held outputs)."""
    n = g.n_ops
    k = rng.randint(1, min(n, 14))
    ops = sorted(rng.sample(range(n), k))
    inside = set(ops)
    live_in, live_out = set(), set()
    for t in g.tensors:
        cons = set(t.consumers)
        if t.producer not in inside and cons & inside:
            live_in.add(t.id)
        if t.producer in inside and cons - inside:
            live_out.add(t.id)
        if t.producer in inside and rng.random() < 0.1:
            live_out.add(t.id)
    return ops, sorted(live_in), sorted(live_out)


def make_exact():
    """exact_order (ordering.py:183-286) on whole random DAGs, random windows
    with boundary liveness, the hazard fixtures and the planner's own windows
    (node_limit 20, node_cap 500k); plus cases whose node cap the search hits
    (the reference then returns the greedy incumbent, optimal=False)."""
    out, graphs = [], {}

    def case(name, g, ops, live_in, live_out, node_cap=500_000, doc=None):
        prob = ro.OrderingProblem(graph=g, ops=tuple(ops), live_in=frozenset(live_in),
                                  live_out=frozenset(live_out), node_cap=node_cap)
        sol = ro.exact_order(prob)
        ent = {"graph": name, "ops": list(ops), "live_in": list(live_in), "live_out": list(live_out),
               "node_cap": node_cap, "order": list(sol.order), "peak": sol.peak,
               "optimal": sol.optimal, "nodes": sol.stats.nodes}
        if doc is not None:
            ent["doc"] = doc
        out.append(ent)

    rng = random.Random(7)
    for k in range(60):
        g = gen_random_dag(2 + k % 13, density=0.15 + 0.05 * (k % 8), seed=2000 + k)
        case(f"rand{k}", g, range(g.n_ops), (), (), doc=rg.graph_to_doc(g))
    for k in range(60):
        g = gen_random_dag(8 + k % 12, density=0.2 + 0.05 * (k % 6), seed=3000 + k)
        ops, li, lo = random_window(g, rng)
        case(f"win{k}", g, ops, li, lo, doc=rg.graph_to_doc(g))
    for name, doc in edge_docs().items():
        g = rg.load_graph(doc)
        case(name, g, range(g.n_ops), (), (), doc=doc)
    trap = gen_greedy_trap(0)
    case("greedy_trap0", trap, range(trap.n_ops), (), (), doc=rg.graph_to_doc(trap))
    # caps the search hits: a 12-op antichain, and a random DAG under a tiny cap
    anti = {"ops": [{"id": i, "name": f"a{i}", "kind": "forward", "inputs": [], "outputs": [i]}
                    for i in range(12)] + [{"id": 12, "name": "z", "kind": "forward",
                                            "inputs": list(range(12)), "outputs": []}],
            "tensors": [{"id": i, "size_bytes": (i % 5 + 1) * MB} for i in range(12)]}
    g = rg.load_graph(anti)
    case("antichain12_cap100", g, range(g.n_ops), (), (), node_cap=100, doc=anti)
    case("antichain12_nocap", g, range(g.n_ops), (), (), node_cap=None, doc=anti)
    g = gen_random_dag(14, density=0.2, seed=77)
    case("rand14_cap20", g, range(g.n_ops), (), (), node_cap=20, doc=rg.graph_to_doc(g))
    # the planner's exact windows
    for arch in ("mlp", "residual", "transformer_block"):
        for blocks in (2, 4):
            g = gen_training_graph(arch, blocks, optimizer="adam")
            name = f"{arch}{blocks}"
            graphs[name] = rg.graph_to_doc(g)
            tree = rp.build_subgraph_tree(g, 20)
            lin = rp.linearize(g, tree)
            wu = rp.place_weight_updates(g, tree, 2.0)
            for w, prob in ro.build_window_problems(g, lin, wu):
                if len(prob.ops) <= 20:
                    case(name, g, sorted(prob.ops), sorted(prob.live_in), sorted(prob.live_out))
    dump("exact.json", {"cases": out, "graphs": graphs})


def make_plans():
    docs = {"diamond": diamond_doc()}
    for arch in ("mlp", "residual", "transformer_block"):
        for blocks in (1, 2, 4):
            for opt in ("sgd", "adam"):
                docs[f"{arch}-{blocks}-{opt}"] = rg.graph_to_doc(gen_training_graph(arch, blocks, optimizer=opt))
    out = {}
    for name, doc in docs.items():
        g = rg.load_graph(doc)
        out[name] = {"doc": doc, "plan": rp.plan_doc_bytes(rp.plan(g)).decode()}
    dump("plans.json", out)


if __name__ == "__main__":
    which = set(sys.argv[1:]) or {"peaks", "schedules", "layouts", "layout_search", "greedy", "exact",
                                  "exact_search", "plans", "wide_search"}
    for w in ("peaks", "schedules", "layouts", "layout_search", "greedy", "exact", "exact_search", "plans",
              "wide_search"):
        if w in which:
            globals()[f"make_{w}"]()
