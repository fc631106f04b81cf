"""K1 (batched order evaluator), the device candidate generator, argmin and the
single-schedule drop-ins, against the reference's golden vectors and the
CPU oracle.  Bit-exact (integer work)."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden
from oracle import coracle
from oracle import memplan_oracle as O
from paper_2310_19295_b200 import graphgen as gg
from paper_2310_19295_b200.evaluator import (argmin_orders, evaluate_orders, generate_orders,
                                             live_bytes_by_timestep, peak_memory, sequential_schedule,
                                             tensor_lifetimes, validate_schedule)
from paper_2310_19295_b200.graph import ConfigError, Schedule, ScheduleError, load_graph

pytestmark = pytest.mark.gpu


def _check_rows(g, rows):
    n = len(g.ops)
    ok_rows = [r for r in rows if len(r["order"]) == n]
    orders = np.array([r["order"] for r in ok_rows], np.int64).reshape(len(ok_rows), n)
    peak, arg, val = evaluate_orders(g, orders)
    for k, r in enumerate(ok_rows):
        e = r["expect"]
        if isinstance(e, dict):
            assert not val[k], r["order"]
        else:
            assert val[k] and (int(peak[k]), int(arg[k])) == tuple(e), r["order"]


def test_fixture_cases():
    P = golden("peaks")
    graphs = {k: load_graph(v) for k, v in P["fixtures"].items()}
    by: dict[str, list] = {}
    for c in P["cases"]:
        by.setdefault(c["graph"], []).append(c)
    for name, rows in by.items():
        _check_rows(graphs[name], rows)


@pytest.mark.parametrize("corpus", ["small_dags", "random_dags", "training"])
def test_corpora(corpus):
    for e in golden("peaks")[corpus]:
        _check_rows(load_graph(e["doc"]), e["rows"])


@pytest.mark.parametrize("name", ["layered", "gpt2-small", "bert-large", "gpt2-xl"])
def test_config_graphs_generator_and_golden(name):
    entry = [e for e in golden("peaks")["configs"] if e["graph"] == name][0]
    g = load_graph(gg.config_doc(name))
    B = len(entry["rows"])
    orders = generate_orders(g, 0, 0, B)
    peak, arg, val = evaluate_orders(g, orders)
    host = orders.cpu().numpy()
    for k, r in enumerate(entry["rows"]):
        assert hashlib.sha256(",".join(map(str, host[k].tolist())).encode()).hexdigest()[:16] == r["order_sha"]
        assert bool(val[k]) and (int(peak[k]), int(arg[k])) == tuple(r["expect"])


@pytest.mark.parametrize("name,B", [("layered", 4096), ("gpt2-small", 2048), ("gpt2-xl", 256)])
def test_large_batch_vs_c_oracle(name, B):
    g = load_graph(gg.config_doc(name))
    orders = generate_orders(g, 12345, 1000, B)
    host = orders.cpu().numpy()
    # corrupt a few rows: swap a pred/succ pair, duplicate, out-of-range
    host[1] = host[1][::-1]
    host[2, 5] = host[2, 6]
    host[3, 0] = len(g.ops)
    cg = coracle.CGraph(g)
    want = coracle.eval_orders(cg, host)
    got = evaluate_orders(g, host)
    assert np.array_equal(got[2], want[2])
    assert np.array_equal(got[0][want[2]], want[0][want[2]])
    assert np.array_equal(got[1][want[2]], want[1][want[2]])
    import torch
    dev = evaluate_orders(g, torch.from_numpy(host).cuda())
    assert np.array_equal(dev[2].cpu().numpy(), want[2])
    assert np.array_equal(dev[0].cpu().numpy()[want[2]], want[0][want[2]])
    # argmin == first strict minimum, on device and host paths
    best = O.first_strict_min(want[0].tolist(), want[2].tolist())
    assert argmin_orders(dev[0], dev[2], id_base=7) == (best[0], best[1] + 7)
    assert argmin_orders(got[0], got[2]) == best


def test_generator_matches_python_restatement():
    g = load_graph(gg.config_doc("gpt2-small"))
    preds, succs = O.direct_preds(g), O.direct_succs(g)
    orders = generate_orders(g, 99, 5, 8).cpu().numpy()
    for k in range(8):
        assert orders[k].tolist() == O.kahn_candidate(len(g.ops), preds, succs, 99, 5 + k)


@pytest.mark.parametrize("name", ["gpt2-small", "bert-large", "gpt2-xl", "layered", "wide", "fan-in"])
def test_generator_thread_form_equals_warp_form(name):
    """The thread-per-candidate generator (heap + counters per thread, rows it
    cannot finish rewritten by the warp form) gives the warp form's rows
    exactly: training graphs, the layered DAG (ready sets above the heap's
    32 entries: the hand-over path), a 300-wide antichain and an op with 12
    predecessors (the warp form only); a sample of
    rows against the Python restatement."""
    from paper_2310_19295_b200.evaluator import set_gen_form
    if name == "wide":
        doc = {"ops": [{"id": 0, "name": "s", "kind": "forward", "inputs": [], "outputs": list(range(300))}]
               + [{"id": 1 + k, "name": f"w{k}", "kind": "forward", "inputs": [k], "outputs": []}
                  for k in range(300)],
               "tensors": [{"id": k, "size_bytes": 4} for k in range(300)]}
    elif name == "fan-in":
        doc = {"ops": [{"id": k, "name": f"p{k}", "kind": "forward", "inputs": [], "outputs": [k]} for k in range(12)]
               + [{"id": 12, "name": "j", "kind": "forward", "inputs": list(range(12)), "outputs": []}],
               "tensors": [{"id": k, "size_bytes": 4} for k in range(12)]}
    else:
        doc = gg.config_doc(name)
    g = load_graph(doc)
    B = 3000 if name in ("gpt2-xl", "bert-large") else 5000
    got = generate_orders(g, 17, 123, B).cpu().numpy()
    set_gen_form(1)
    try:
        want = generate_orders(g, 17, 123, B).cpu().numpy()
    finally:
        set_gen_form(0)
    assert np.array_equal(got, want)
    if name in ("gpt2-xl", "layered"):   # the other heap capacities (A/B settings)
        for cap in (40, 64):
            set_gen_form(cap)
            try:
                assert np.array_equal(generate_orders(g, 17, 123, B).cpu().numpy(), want), cap
            finally:
                set_gen_form(0)
    preds, succs = O.direct_preds(g), O.direct_succs(g)
    for k in (0, 1, B // 2, B - 1):
        assert got[k].tolist() == O.kahn_candidate(len(g.ops), preds, succs, 17, 123 + k)


def test_argmin_ties_and_none_valid():
    peak = np.array([7, 3, 3, 1, 3], np.int64)
    valid = np.array([1, 1, 1, 0, 1], bool)
    assert argmin_orders(peak, valid) == (3, 1)
    assert argmin_orders(peak, np.zeros(5, bool)) == (2**63 - 1, -1)


def test_single_schedule_dropins():
    S = golden("schedules")
    fx = {k: load_graph(v) for k, v in golden("peaks")["fixtures"].items()}
    for c in S["packed"] + S["random"]:
        g = fx[c["graph"]] if "graph" in c else load_graph(c["doc"])
        s = Schedule(tuple(c["order"]), tuple(c["timesteps"]), c["ops_per_step"])
        assert peak_memory(g, s) == tuple(c["peak"])
        assert live_bytes_by_timestep(g, s) == c["live"]
        if "lifetimes" in c:
            assert [list(x) for x in tensor_lifetimes(g, s)] == c["lifetimes"]
    g = fx["diamond"]
    for c in S["errors"]:
        s = Schedule(tuple(c["order"]), tuple(c["timesteps"]), c["ops_per_step"])
        if c["error"] is None:
            validate_schedule(g, s)
            assert peak_memory(g, s) == tuple(c["peak"])
            continue
        exc = ConfigError if c["error"] == "ConfigError" else ScheduleError
        with pytest.raises(exc) as ei:
            validate_schedule(g, s)
        assert str(ei.value) == c["message"]


def test_reference_unit_answers_through_gpu():
    MB = 1 << 20
    fx = {k: load_graph(v) for k, v in golden("peaks")["fixtures"].items()}
    d = fx["diamond"]
    assert peak_memory(d, sequential_schedule(d, (0, 1, 2, 3))) == (120 * MB, 1)
    assert peak_memory(d, sequential_schedule(d, (0, 2, 1, 3)))[0] == 90 * MB
    assert peak_memory(fx["single"], sequential_schedule(fx["single"], (0,))) == (8, 0)
    assert peak_memory(fx["empty"], sequential_schedule(fx["empty"], ())) == (0, 0)
    with pytest.raises(ScheduleError):
        sequential_schedule(d, (3, 0, 1, 2))


@pytest.mark.parametrize("variant", [1, 4, 5, 6])
@pytest.mark.parametrize("name", ["layered", "gpt2-small", "bert-large", "gpt2-xl"])
def test_both_k1_variants_vs_c_oracle(name, variant):
    """Every K1 variant -- v5 (dynamic class bytes, the default on the training
    graphs up to 8k ops), v4 (the default where the classes do not fit --
    layered -- and on the 11k-op GPT2-XL), v5 with bulk-copied rows and the
    generic v1 -- agrees with the oracle, including on corrupted rows
    (invalid -> valid=False)."""
    from paper_2310_19295_b200.evaluator import device_graph, set_k1_variant
    g = load_graph(gg.config_doc(name))
    assert device_graph(g).info()["k1_variant"] == (4 if name == "layered" else 5)
    B = 1501
    host = generate_orders(g, 7, 0, B).cpu().numpy()
    rng = np.random.default_rng(0)
    n = len(g.ops)
    for r in range(0, B, 50):                   # swaps: mostly invalid
        i, j = rng.integers(0, n, 2)
        host[r, [i, j]] = host[r, [j, i]]
    for r in range(1, B, 97):                   # duplicates
        host[r, rng.integers(0, n)] = host[r, rng.integers(0, n)]
    for r in range(2, B, 131):                  # out of range
        host[r, rng.integers(0, n)] = n + 3
    want = coracle.eval_orders(coracle.CGraph(g), host)
    set_k1_variant(variant)
    try:
        got = evaluate_orders(g, host)
    finally:
        set_k1_variant(0)
    assert np.array_equal(got[2], want[2])
    v = want[2]
    assert np.array_equal(got[0][v], want[0][v]) and np.array_equal(got[1][v], want[1][v])


def test_unit_shift_and_v2_eligibility():
    from paper_2310_19295_b200.evaluator import device_graph
    MB = 1 << 20
    lay = load_graph(gg.config_doc("layered"))   # keep the graph alive: the handle is cached on it
    info = device_graph(lay).info()
    assert info["k1_variant"] == 4 and info["unit_shift"] >= 20   # MB-rounded sizes
    # an odd byte count forces unit 1; a 2^33-byte output forces the generic path
    doc = {"ops": [{"id": 0, "name": "a", "kind": "forward", "inputs": [], "outputs": [0]},
                   {"id": 1, "name": "b", "kind": "forward", "inputs": [0], "outputs": [1]}],
           "tensors": [{"id": 0, "size_bytes": 3}, {"id": 1, "size_bytes": 2**33 + 1}]}
    g = load_graph(doc)
    assert device_graph(g).info()["k1_variant"] == 1
    peak, arg, val = evaluate_orders(g, np.array([[0, 1]]))
    assert bool(val[0]) and (int(peak[0]), int(arg[0])) == O.peak_memory(g, (0, 1))
    doc["tensors"][1]["size_bytes"] = 5 * MB + 1
    g = load_graph(doc)
    assert device_graph(g).info()["k1_variant"] == 5
    peak, arg, val = evaluate_orders(g, np.array([[0, 1], [1, 0]]))
    assert val.tolist() == [True, False]
    assert (int(peak[0]), int(arg[0])) == O.peak_memory(g, (0, 1))


def test_packed_key_selection_matches_first_strict_min():
    import torch
    from paper_2310_19295_b200.evaluator import select_key_device
    from paper_2310_19295_b200.sharding import decode_key, key_bits
    g = load_graph(gg.config_doc("gpt2-small"))
    orders = generate_orders(g, 3, 0, 700)
    host = orders.cpu().numpy()
    host[::7] = host[::7][:, ::-1]                       # invalid rows
    dev = torch.from_numpy(host).cuda()
    peak, _, val = evaluate_orders(g, dev)
    bits = key_bits(1 << 20)
    key = int(select_key_device(g, peak, val, 1000, bits).item())
    want = O.first_strict_min(peak.cpu().tolist(), val.cpu().tolist())
    assert decode_key(key, bits) == (want[0], want[1] + 1000)
    none = int(select_key_device(g, peak, torch.zeros_like(val), 0, bits).item())
    assert decode_key(none, bits) == (2**63 - 1, -1)


@pytest.mark.parametrize("variant", [0, 1, 4, 5, 6])
def test_uint16_rows_match_int32(variant):
    """uint16 rows (RM_ORDERS_U16) give exactly the int32 results on every
    evaluator, host-staged and device-resident."""
    import torch
    from paper_2310_19295_b200.evaluator import evaluate_and_select, set_k1_variant
    g = load_graph(gg.config_doc("gpt2-small"))
    orders = generate_orders(g, 11, 0, 999)
    host = orders.cpu().numpy()
    host[::9] = host[::9][:, ::-1]
    want = coracle.eval_orders(coracle.CGraph(g), host)
    set_k1_variant(variant)
    try:
        for rows in (host.astype(np.uint16), torch.from_numpy(host).cuda().to(torch.uint16)):
            p, a, v = evaluate_orders(g, rows)
            p, a, v = (x.cpu().numpy() if hasattr(x, "cpu") else x for x in (p, a, v))
            assert np.array_equal(v, want[2])
            assert np.array_equal(p[want[2]], want[0][want[2]]) and np.array_equal(a[want[2]], want[1][want[2]])
        *_, best = evaluate_and_select(g, host.astype(np.uint16), id_base=5)
        b = O.first_strict_min(want[0].tolist(), want[2].tolist())
        assert best == (b[0], b[1] + 5)
    finally:
        set_k1_variant(0)


def _random_doc(rng, n_ops, max_in=3):
    """Random DAG document with the parity hazards mixed in: duplicate inputs
    (h1), self-consuming ops (h2), zero-consumer tensors (h3), sizes 0..8 MB."""
    MB = 1 << 20
    ops, tensors = [], []
    for v in range(n_ops):
        ins = []
        if tensors:
            for _ in range(rng.randint(0, max_in)):
                ins.append(rng.randrange(len(tensors)))
            if ins and rng.random() < 0.15:
                ins.append(ins[0])                       # duplicate input
        outs = []
        for _ in range(rng.randint(0, 2)):
            outs.append(len(tensors))
            tensors.append({"id": len(tensors), "size_bytes": rng.choice([0, 1, 3, 8]) * MB // rng.choice([1, 2])})
        if outs and rng.random() < 0.1:
            ins.append(outs[0])                          # self-consuming op
        ops.append({"id": v, "name": f"op{v}", "kind": "forward", "inputs": ins, "outputs": outs})
    return {"ops": ops, "tensors": tensors}


@pytest.mark.parametrize("seed", range(6))
def test_random_hazard_graphs_vs_oracle(seed):
    import random
    rng = random.Random(seed)
    for trial in range(25):
        g = load_graph(_random_doc(rng, rng.randint(1, 60)))
        n = len(g.ops)
        preds, succs = O.direct_preds(g), O.direct_succs(g)
        rows = [O.kahn_candidate(n, preds, succs, seed, c) for c in range(20)]
        for r in range(5):                               # random permutations: mostly invalid
            perm = list(range(n))
            rng.shuffle(perm)
            rows.append(perm)
        orders = np.array(rows, np.int64).reshape(len(rows), n)
        for variant in (0, 1, 4, 5):
            from paper_2310_19295_b200.evaluator import set_k1_variant
            set_k1_variant(variant)
            try:
                peak, arg, val = evaluate_orders(g, orders)
            finally:
                set_k1_variant(0)
            for k, row in enumerate(rows):
                want = O.evaluate_order(g, row, preds)
                assert bool(val[k]) == want[2], (seed, trial, variant, row)
                if want[2]:
                    assert (int(peak[k]), int(arg[k])) == want[:2], (seed, trial, variant, row)


@pytest.mark.parametrize("variant", [0, 1, 4, 6])
@pytest.mark.parametrize("name", ["layered", "gpt2-small", "bert-large", "gpt2-xl"])
def test_fused_key_selection(name, variant):
    """K1 with the packed-key selection fused into the launch (v4) or chained
    (other variants) equals evaluate_orders + select_key_device, including
    invalid rows, an id base, and a batch with no valid row."""
    import torch
    from paper_2310_19295_b200.evaluator import evaluate_select_key, select_key_device, set_k1_variant
    from paper_2310_19295_b200.sharding import decode_key, key_bits
    g = load_graph(gg.config_doc(name))
    orders = generate_orders(g, 5, 0, 2500)
    host = orders.cpu().numpy()
    host[::3] = host[::3][:, ::-1]
    dev = torch.from_numpy(host).cuda()
    bits = key_bits(1 << 22)
    set_k1_variant(variant)
    try:
        for base in (0, 123_456):
            p, a, v, key = evaluate_select_key(g, dev, base, bits)
            p2, a2, v2 = evaluate_orders(g, dev)
            want = int(select_key_device(g, p2, v2, base, bits).item())
            assert int(key.item()) == want
            assert torch.equal(v, v2) and torch.equal(p[v], p2[v2]) and torch.equal(a[v], a2[v2])
            b = O.first_strict_min(p2.cpu().tolist(), v2.cpu().tolist())
            assert decode_key(int(key.item()), bits) == (b[0], b[1] + base)
        bad = torch.flip(orders[1::3], dims=[1]).contiguous()   # every row reversed: none valid
        *_, key = evaluate_select_key(g, bad, 0, bits)
        assert int(key.item()) == 2**63 - 1
    finally:
        set_k1_variant(0)


def test_fused_selection_on_two_streams_from_one_thread():
    """Fused K1 selections issued from one thread on two streams with no sync
    in between keep separate partials and counters (one set per stream): each
    key equals its own batch's first strict minimum, and a third round on the
    same streams still elects the last group correctly."""
    import torch
    from paper_2310_19295_b200.evaluator import evaluate_select_key
    from paper_2310_19295_b200.sharding import decode_key, key_bits
    g = load_graph(gg.config_doc("gpt2-small"))
    a = generate_orders(g, 11, 0, 20000)
    b = generate_orders(g, 12, 0, 9000)
    bits = key_bits(1 << 20)
    want = []
    for rows in (a, b):
        p, _, v = evaluate_orders(g, rows)
        want.append(O.first_strict_min(p.cpu().tolist(), v.cpu().tolist()))
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        _, _, _, k1 = evaluate_select_key(g, a, 0, bits, stream=s1)
        _, _, _, k2 = evaluate_select_key(g, b, 0, bits, stream=s2)
        torch.cuda.synchronize()
        assert decode_key(int(k1.item()), bits) == tuple(want[0])
        assert decode_key(int(k2.item()), bits) == tuple(want[1])


def test_host_staged_calls_from_two_threads():
    """libroam is re-entrant: host-buffer calls of different batch sizes (so
    different K1 launch geometries and shared-memory sizes) from two threads on
    their own streams return what the same calls return one at a time."""
    import threading

    import torch
    from paper_2310_19295_b200.evaluator import evaluate_and_select
    g = load_graph(gg.config_doc("gpt2-small"))
    orders = generate_orders(g, 5, 0, 6000).cpu().numpy().astype(np.uint16)
    sizes = [6000, 37, 1500, 129, 4096, 5]
    want = [evaluate_and_select(g, orders[:b], id_base=b) for b in sizes]
    got = [None] * len(sizes)
    errors = []

    def worker(j):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            for _ in range(3):
                for k in range(j, len(sizes), 2):
                    got[k] = evaluate_and_select(g, orders[:sizes[k]], id_base=sizes[k], stream=st)
        except Exception as e:  # surfaced below
            errors.append(e)

    ts = [threading.Thread(target=worker, args=(j,)) for j in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for w, r in zip(want, got):
        assert np.array_equal(w[0], r[0]) and np.array_equal(w[1], r[1])
        assert np.array_equal(w[2], r[2]) and w[3] == r[3]


def test_nccl_select_key_single_rank():
    """rm_nccl_select_key through a one-rank NCCL communicator made by
    libroam itself (rm_nccl_unique_id / rm_nccl_comm_init): the fused K1 key
    survives the 8-byte all-reduce(MIN) unchanged and decodes to the oracle's
    first strict minimum; a rank with no valid candidate (INT64_MAX) loses."""
    import torch

    from paper_2310_19295_b200.evaluator import evaluate_select_key
    from paper_2310_19295_b200.sharding import NcclSelect
    g = load_graph(gg.config_doc("layered"))
    orders = generate_orders(g, 3, 0, 700)
    host = orders.cpu().numpy()
    host[5] = host[6]                                  # an invalid row
    orders = torch.from_numpy(host).cuda()
    id_bits = 20
    _, _, _, key = evaluate_select_key(g, orders, 0, id_bits)
    want = coracle.eval_orders(coracle.CGraph(g), host)
    best = O.first_strict_min(want[0].tolist(), want[2].tolist())
    sel = NcclSelect(1, NcclSelect.unique_id(), 0)
    try:
        k = key.clone()
        sel.select(k)
        torch.cuda.synchronize()
        assert int(k.item()) == int(key.item())
        assert (int(k.item()) >> id_bits, int(k.item()) & ((1 << id_bits) - 1)) == best
        none = torch.full((1,), 2**63 - 1, dtype=torch.int64, device="cuda")
        sel.select(none)
        torch.cuda.synchronize()
        assert int(none.item()) == 2**63 - 1
    finally:
        sel.close()


@pytest.mark.parametrize("name", ["layered", "gpt2-small", "bert-large"])
def test_batched_live_matches_reference_semantics(name):
    """rm_eval_live: per-candidate live_bytes_by_timestep (graph.py:452-458)
    equal to the Python restatement on sampled rows, its max / first argmax
    equal to K1's peak / argmax on every valid row, validity equal to K1's
    (corrupted rows included), for int32 and uint16 rows, host and device."""
    import torch

    from paper_2310_19295_b200.evaluator import evaluate_live
    g = load_graph(gg.config_doc(name))
    n = len(g.ops)
    B = 600
    host = generate_orders(g, 21, 0, B).cpu().numpy()
    rng = np.random.default_rng(1)
    for r in range(0, B, 37):
        i, j = rng.integers(0, n, 2)
        host[r, [i, j]] = host[r, [j, i]]
    host[3, 4] = host[3, 5]
    pk, ag, vl = evaluate_orders(g, host)
    live, val = evaluate_live(g, host)
    assert np.array_equal(val, vl)
    v = np.flatnonzero(vl)
    assert np.array_equal(live[v].max(axis=1), pk[v]) and np.array_equal(live[v].argmax(axis=1), ag[v])
    for k in v[:: max(1, len(v) // 6)]:
        assert live[k].tolist() == O.live_bytes_by_timestep(g, O.sequential_timesteps(n, host[k].tolist()))
    dl, dv = evaluate_live(g, torch.from_numpy(host).cuda())
    assert np.array_equal(dl.cpu().numpy()[v], live[v]) and np.array_equal(dv.cpu().numpy(), val)
    hl, hv = evaluate_live(g, host.astype(np.uint16))
    assert np.array_equal(hl[v], live[v]) and np.array_equal(hv, val)
