"""Window ordering problems from slot positions -- the batch
that feeds K4 -- as interval stabbing instead of the reference's per-window
scan of every tensor (ordering.py:470-542; 94 s of 279 s of ``plan()`` at
10.8k ops in the reference).

With op_pos[v] the slot of v (its window's slot for window ops, incl. placed
weight-update branches, ordering.py:489-503), b = op_pos[producer] and
L = max op_pos over consumers (the horizon ``len(slots)`` without consumers),
the reference's per-tensor rule for window w at slot p reduces to

    live_in(w)  = { t : b < p <= L }
    live_out(w) = { t : b <= p <  L }

(b == p exactly when the producer is inside w -- unless the linearisation
lists an op in two windows: every such window but the op's owner gets the
reference's rule evaluated directly, vectorised over tensors).  The windows are swept once in
slot order: between consecutive slots only the tensors born or dying in
between change membership (found by binary search in the (b, L)-sorted
tensor lists), so each window's sets are its predecessor's plus/minus a few
ids.  Host code: the output is the reference's
frozensets.  Equality with the reference is tested on every window the planner
builds (tests/test_plugin_host.py).
"""

from __future__ import annotations

import numpy as np

from .graph import graph_arrays


class LiveSet(frozenset):
    """The reference's frozenset of tensor ids, also carrying them as an
    int32 array (``arr``) so the K4/K5 marshalling (ordering._window_csr) does
    not walk the set element by element."""
    __slots__ = ("arr",)


def live_set(idx: np.ndarray) -> LiveSet:
    s = LiveSet(idx.tolist())
    s.arr = idx.astype(np.int32)
    return s


def window_intervals(g, lin, wu_plan=None):
    """(final ops per window, slot per window, b[T], L[T], horizon, shared):
    ``shared`` = the windows listing an op whose position is another
    window's slot (the reference keeps the LAST window listing an op as its
    position, ordering.py:490-503), for which the stabbing rule's premise
    "producer inside <=> b == p" does not hold."""
    a = graph_arrays(g)
    n = a.n_ops
    extra = {w.index: wu_plan.ops_for_window(w.index) for w in lin.windows} if wu_plan else {}
    op_pos = np.full(n, -1, np.int64)
    slot_of_window: dict[int, int] = {}
    for i, (kind, ref) in enumerate(lin.slots):
        if kind == "op":
            op_pos[ref] = i
        elif ref not in slot_of_window:  # _window_slot: first matching slot
            slot_of_window[ref] = i
    final_ops: dict[int, tuple[int, ...]] = {}
    owner = np.full(n, -1, np.int64)
    listed = False
    for w in lin.windows:
        ops = tuple(sorted((*w.ops, *extra.get(w.index, ()))))
        final_ops[w.index] = ops
        if w.index not in slot_of_window:
            raise ValueError(f"window {w.index} not in slot sequence")
        if ops:
            idx = np.asarray(ops, np.int64)
            listed = listed or bool((owner[idx] >= 0).any())
            owner[idx] = w.index          # the last window listing an op wins
            op_pos[idx] = slot_of_window[w.index]
    shared = set()
    if listed:   # an op in two windows: every listing window but its owner
        for w in lin.windows:
            ops = final_ops[w.index]
            if ops and (owner[np.asarray(ops, np.int64)] != w.index).any():
                shared.add(w.index)
    horizon = len(lin.slots)
    producer = a.producer.astype(np.int64)
    if (op_pos[producer] < 0).any() or (a.cons_idx.size and (op_pos[a.cons_idx] < 0).any()):
        raise KeyError("op without a slot position")
    b = op_pos[producer]
    T = a.n_tensors
    L = np.full(T, horizon, np.int64)
    counts = np.diff(a.cons_ptr)
    nz = np.flatnonzero(counts > 0)
    if nz.size:
        L[nz] = np.maximum.reduceat(op_pos[a.cons_idx], a.cons_ptr[:-1][nz].astype(np.int64))
    return final_ops, slot_of_window, b, L, horizon, shared


def _exact_sets(a, ops, p, b, L):
    """The reference's per-tensor rule (ordering.py:505-527) for one window,
    vectorised over tensors: membership of producer and consumers in the
    window's own op set, positions from op_pos."""
    inside = np.zeros(a.n_ops, bool)
    inside[np.asarray(ops, np.int64)] = True
    prod_in = inside[np.asarray(a.producer, np.int64)]
    cp = np.asarray(a.cons_ptr, np.int64)
    has = cp[1:] > cp[:-1]
    local = np.zeros(len(b), bool)
    if a.cons_idx.size:
        ent = np.append(inside[np.asarray(a.cons_idx, np.int64)], False).astype(np.int64)
        local[has] = np.add.reduceat(ent, cp[:-1][has]) > 0
    later = L > p
    live_out = (prod_in & later) | (~prod_in & (b < p) & later)
    live_in = ~prod_in & (b < p) & (local | later)
    return live_set(np.flatnonzero(live_in)), live_set(np.flatnonzero(live_out))


def build_window_problems(g, lin, wu_plan=None, ops_per_step: int = 1, time_budget: float = 60.0,
                          node_cap=None, *, window_type, problem_type):
    """ordering.py:470-542 with the reference's own Window / OrderingProblem
    types passed in; same list, same order, same sets."""
    final_ops, slot_of_window, b, L, _, shared = window_intervals(g, lin, wu_plan)
    wins = list(lin.windows)
    slots = [slot_of_window[w.index] for w in wins]
    sets = _sweep_live_sets(b, L, sorted(set(slots)))
    out = []
    for w, p in zip(wins, slots):
        ops = final_ops[w.index]
        if w.index in shared:
            live_in, live_out = _exact_sets(graph_arrays(g), ops, p, b, L)
        else:
            live_in, live_out = sets[p]
        out.append((window_type(index=w.index, leaf=w.leaf, ops=ops),
                    problem_type(graph=g, ops=ops, live_in=live_in, live_out=live_out,
                                 ops_per_step=ops_per_step, time_budget=time_budget,
                                 node_cap=node_cap)))
    return out


def _sweep_live_sets(b: np.ndarray, L: np.ndarray, slots: list[int]) -> dict:
    """{slot p: (live_in(p), live_out(p))} for ascending slots, swept once:
    between consecutive slots only the tensors born or dying in between
    change membership, so each set is the previous one minus/plus a few ids
    (set algebra on the previous frozenset, no per-id Python objects), and
    its id array comes from an updated membership mask.
      live_in(p)  = {t : b < p <= L}     live_out(p) = {t : b <= p < L}"""
    T = len(b)
    ob = np.argsort(b, kind="stable")
    oL = np.argsort(L, kind="stable")
    bs, Ls = b[ob], L[oL]
    S = np.asarray(slots, np.int64)
    Ll, Lr = Ls.searchsorted(S, "left").tolist(), Ls.searchsorted(S, "right").tolist()
    bl, br = bs.searchsorted(S, "left").tolist(), bs.searchsorted(S, "right").tolist()
    m_in = np.zeros(T, bool)
    m_out = np.zeros(T, bool)
    s_in, s_out = frozenset(), frozenset()
    out = {}
    prev = None
    for k, p in enumerate(slots):
        if prev is None:
            add_in = ((b < p) & (p <= L)).nonzero()[0]
            add_out = ((b <= p) & (p < L)).nonzero()[0]
            rem_in = rem_out = add_in[:0]
        else:
            # live_in: leave when L < p (L in [prev, p)); join when b in [prev, p) and L >= p
            c = oL[Ll[k - 1]:Ll[k]]
            rem_in = c[m_in[c]]
            c = ob[bl[k - 1]:bl[k]]
            add_in = c[L[c] >= p]
            # live_out: leave when L <= p (L in (prev, p]); join when b in (prev, p] and L > p
            c = oL[Lr[k - 1]:Lr[k]]
            rem_out = c[m_out[c]]
            c = ob[br[k - 1]:br[k]]
            add_out = c[L[c] > p]
        m_in[rem_in] = False
        m_in[add_in] = True
        m_out[rem_out] = False
        m_out[add_out] = True
        if len(rem_in) or len(add_in):
            s_in = s_in.difference(rem_in.tolist()).union(add_in.tolist())
        if len(rem_out) or len(add_out):
            s_out = s_out.difference(rem_out.tolist()).union(add_out.tolist())
        li, lo = LiveSet(s_in), LiveSet(s_out)
        li.arr = m_in.nonzero()[0].astype(np.int32)
        lo.arr = m_out.nonzero()[0].astype(np.int32)
        out[p] = (li, lo)
        prev = p
    return out
