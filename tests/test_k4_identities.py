"""CPU check of the two identities K4 (k_greedy.cu) relies on, against the
reference's golden greedy_order vectors (tests/golden/greedy.json, including
the duplicate-input hazard h1 and the planner's real windows).

This is a plain-Python model of the kernel's bookkeeping, not of the
reference's loop (reference: pkg/src/memplan/ordering.py:78-180):
  * the bytes a pick frees equal out - score, so no per-step sum of freed
    bytes is needed;
  * each tracked tensor carries its consumer-entry count and the XOR of
    (local index + 1) over the entries of unrun ops; when the count reaches 1
    with an unrun entry left, the XOR names that op (0: none left), so no
    walk of the consumer list is needed.
The model asserts both at every step and must reproduce every golden order
and peak."""

from __future__ import annotations

import pytest

from conftest import golden
from paper_2310_19295_b200.graph import load_graph


def _k4_model(g, ops, live_in, live_out):
    ops = sorted(ops)
    loc = {v: i for i, v in enumerate(ops)}
    rel = sorted({t for v in ops for t in g.ops[v].outputs} | set(live_in))
    tloc, count, xor, size, cons = {}, [], [], [], []
    start_live = sum(g.tensors[t].size for t in live_in)
    for t in rel:
        entries = [loc[c] for c in g.tensors[t].consumers if c in loc]
        produced = g.tensors[t].producer in loc
        if t in live_out or (produced and not entries):
            continue  # held: never freed inside the window
        tloc[t] = len(count)
        count.append(len(entries))
        x = 0
        for j in entries:
            x ^= j + 1
        xor.append(x)
        size.append(g.tensors[t].size)
        cons.append(entries)
    n = len(ops)
    out = [sum(g.tensors[t].size for t in g.ops[v].outputs) for v in ops]
    ins = [sorted({tloc[t] for t in g.ops[v].inputs if t in tloc}) for v in ops]
    preds = [{loc[g.tensors[t].producer] for t in g.ops[v].inputs
              if g.tensors[t].producer in loc and g.tensors[t].producer != v} for v in ops]
    succ = [[] for _ in range(n)]
    for i in range(n):
        for p in sorted(preds[i]):
            succ[p].append(i)
    npred = [len(p) for p in preds]
    delta = [out[i] - sum(size[t] for t in ins[i] if count[t] == 1) for i in range(n)]
    ran = [False] * n
    ready = [i for i in range(n) if npred[i] == 0]
    live = peak = start_live
    order = []
    for _ in range(n):
        bi = min(ready, key=lambda i: (delta[i], i))
        ready.remove(bi)
        # identity 1: freed bytes = out - score
        freed = sum(size[t] for t in ins[bi] if count[t] == 1)
        assert freed == out[bi] - delta[bi]
        for t in ins[bi]:
            mult = cons[t].count(bi)
            count[t] -= 1
            if mult % 2:
                xor[t] ^= bi + 1
            if count[t] == 1:
                # identity 2: the XOR names the one unrun entry, if any
                unrun = [j for j in cons[t] if j != bi and not ran[j]]
                holder = xor[t] - 1 if xor[t] else None
                assert holder == (unrun[0] if unrun else None)
                if holder is not None:
                    delta[holder] -= size[t]
        ran[bi] = True
        for s in succ[bi]:
            npred[s] -= 1
            if npred[s] == 0:
                ready.append(s)
        live += out[bi]
        peak = max(peak, live)
        live -= freed
        order.append(ops[bi])
    return order, peak


def _cases():
    G = golden("greedy")
    graphs = {}
    for c in G["cases"]:
        key = c.get("graph") or id(c)
        if key not in graphs:
            graphs[key] = load_graph(c.get("doc") or G["graphs"][c["graph"]])
        yield graphs[key], c


@pytest.mark.parametrize("idx", range(0, 100, 10))
def test_k4_identities_on_golden_windows(idx):
    cases = list(_cases())[idx:idx + 10]
    assert cases
    for g, c in cases:
        order, peak = _k4_model(g, c["ops"], set(c["live_in"]), set(c["live_out"]))
        assert order == c["order"] and peak == c["peak"], c.get("graph")
