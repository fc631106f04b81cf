"""Vectorised drop-ins for the reference planner's control-plane hot spots
("host C++ for tree, linearize and weight-update placement").

The reference keeps transitive predecessors as Python big-int masks and
tests them bit by bit inside Python loops; on large graphs those loops are
most of what remains of ``plan()`` once the hot path runs on the GPU
(reference ``transformer_block`` x600: ``_region_between`` 7.1 s,
``linearize``'s gap ranks 3.5 s, ``_format_ig_ok`` 2.8 s of 18.6 s).  Here the
closure comes from libroam's C++ (``rm_graph_ancestors``, one bit matrix per
graph) and each function is restated over numpy arrays:

  region_between(build, core, lo, hi)   segmentation.py:174-185
  format_ig_ok(build, members, boundary) segmentation.py:188-201
  linearize(g, root)                     segmentation.py:500-572

Each returns exactly what the reference returns (tests/test_plugin_host.py
compares them call by call; the GPU plan tests compare whole plan documents).
Host-only code: no device is needed.
"""

from __future__ import annotations

import bisect

import numpy as np

from ._lib import check, lib, ptr
from .graph import graph_arrays, graph_cache


def closure(g) -> dict:
    """Per-graph cache: ancestor bit matrix ``anc`` (uint8 [n, row_bytes]; bit
    v of row u = v precedes u), ancestor counts, and the tensor arrays."""
    ent = graph_cache(g)
    c = ent.get("closure")
    if c is None:
        from .evaluator import device_graph
        dg = device_graph(g)
        n = dg.n_ops
        words = (n + 63) // 64
        rows = np.zeros((n, max(words, 1)), np.uint64)
        if n:
            check(lib().rm_graph_ancestors(dg.handle, ptr(rows)), "rm_graph_ancestors")
        anc = rows.view(np.uint8).reshape(n, -1)
        a = graph_arrays(g)
        c = {"n": n, "anc": anc, "rows": rows, "count": masked_counts(rows, None),
             "producer": np.asarray(a.producer, np.int64),
             "cons_ptr": np.asarray(a.cons_ptr, np.int64), "cons_idx": np.asarray(a.cons_idx, np.int64)}
        ent["closure"] = c
    return c


def masked_counts(rows, mask_bytes, sel=None) -> np.ndarray:
    """popcount(row & mask) per row of a uint64 bit matrix (rm_popcount_rows,
    C++): mask_bytes a little-endian uint8 bitmask (None = all bits), sel an
    optional row index array."""
    r = rows if sel is None else np.ascontiguousarray(rows[sel])
    out = np.empty(r.shape[0], np.int64)
    m = None
    if mask_bytes is not None:
        mb = np.zeros(r.shape[1] * 8, np.uint8)
        mb[:len(mask_bytes)] = mask_bytes
        m = mb.view(np.uint64)
    check(lib().rm_popcount_rows(ptr(r), r.shape[0], r.shape[1], ptr(m), ptr(out)), "rm_popcount_rows")
    return out


def _bit(anc, rows, cols):
    """anc[rows] has bit cols (vectorised over either argument)."""
    return (anc[rows, cols >> 3] >> (cols & 7)) & 1


def _build_anc(build, c):
    """The ancestor bit matrix behind ``build.before`` (segmentation.py:
    167-168): the graph's C++ closure when ``build.preds`` is the full-graph
    closure (what build_subgraph_tree passes, segmentation.py:361-367; checked
    once per build object on a few ops), otherwise ``build.preds`` itself
    unpacked into the same layout -- exact either way, no reference code."""
    hit = getattr(build, "_roam_anc", None)
    if hit is not None:
        return hit
    n = c["n"]
    probe = sorted({0, n // 3, n // 2, n - 1}) if n else []
    same = len(build.preds) == n and all(bin(build.preds[v]).count("1") == int(c["count"][v]) for v in probe)
    if same:
        anc = c["anc"]
    else:
        row = c["anc"].shape[1]
        anc = np.frombuffer(b"".join(int(p).to_bytes(row, "little") for p in build.preds),
                            np.uint8).reshape(len(build.preds), row)
    try:
        build._roam_anc = anc
    except AttributeError:  # pragma: no cover - frozen build object
        pass
    return anc


def region_between_factory():
    cache: dict = {}

    def region_between(build, core, lo, hi):
        """segmentation.py:174-185: sorted core ops strictly between lo and hi."""
        c = closure(build.g)
        anc = _build_anc(build, c)
        key = id(core)
        hit = cache.get(key)
        if hit is None or hit[0] is not core or hit[1] != len(core):
            arr = np.fromiter(core, np.int64, len(core)) if not isinstance(core, np.ndarray) else core
            hit = (core, len(core), arr)
            cache.clear()
            cache[key] = hit
        v = hit[2]
        keep = np.ones(len(v), bool)
        if lo is not None:
            keep &= (v != lo) & (_bit(anc, v, np.int64(lo)) == 1)
        if hi is not None:
            keep &= (v != hi) & (_bit(anc, np.int64(hi), v) == 1)
        return np.sort(v[keep]).tolist()
    return region_between


def format_ig_ok_factory(mp):
    act_cache: dict = {}

    def format_ig_ok(build, members, boundary):
        """segmentation.py:188-201: no activation crosses the candidate's
        members except through its boundary ops."""
        g = build.g
        c = closure(g)
        n = c["n"]
        key = id(build.categories)
        hit = act_cache.get(key)
        if hit is None or hit[0] is not build.categories:
            act = np.array([build.categories[t.id] is mp.graph.TensorCategory.ACTIVATION
                            for t in g.tensors], bool)
            hit = (build.categories, act)
            act_cache.clear()
            act_cache[key] = hit
        act = hit[1]
        member = np.zeros(n + 1, bool)
        if members:
            member[np.fromiter(members, np.int64, len(members))] = True
        inside = member.copy()
        if boundary:
            inside[np.fromiter((b for b in boundary if b is not None), np.int64)] = True
        cp, ci, prod = c["cons_ptr"], c["cons_idx"], c["producer"]
        # per tensor: any consumer outside / any consumer among the members
        out_ent = np.append(~inside[ci], False).astype(np.int64)
        mem_ent = np.append(member[ci], False).astype(np.int64)
        starts = cp[:-1]
        has = cp[1:] > starts
        any_out = (np.add.reduceat(out_ent, starts) > 0) & has if len(starts) else np.zeros(0, bool)
        any_mem = (np.add.reduceat(mem_ent, starts) > 0) & has if len(starts) else np.zeros(0, bool)
        bad = act & ((member[prod] & any_out) | (any_mem & ~inside[prod]))
        return not bool(bad.any())
    return format_ig_ok


_BUILD_TYPES: dict = {}


def _fast_build_type(seg):
    """The reference's _TreeBuild with wu_load (segmentation.py:159-166) answered
    from a per-build index op -> weight-update branches whose gradients it
    produces, instead of a scan over every branch per query (the split step
    asks once per candidate run: 0.23 s on the 600-block graph)."""
    cls = _BUILD_TYPES.get(seg)
    if cls is None:
        class _Build(seg._TreeBuild):
            def wu_load(self, region):
                idx = self.__dict__.get("_roam_wu_index")
                if idx is None:
                    idx = {}
                    for k, br in enumerate(self.branches):
                        for t in br.gradients:
                            idx.setdefault(self.g.tensors[t].producer, set()).add(k)
                    self.__dict__["_roam_wu_index"] = idx
                hit = set()
                for v in region:
                    ks = idx.get(v)
                    if ks:
                        hit |= ks
                return sum(len(self.branches[k].ops) for k in hit)
        cls = _BUILD_TYPES[seg] = _Build
    return cls


def _mi_full(g, c):
    """``_mi_over(g, all ops)`` (segmentation.py:108-117) and each op's count
    of memory-insensitive ancestors: ancestors from the C++ closure, the
    descendants as n-1-alap (libroam's asap_alap), MI ops ordered by their
    ancestor count (distinct: they are totally ordered)."""
    from .evaluator import asap_alap
    n, anc = c["n"], c["anc"]
    n_anc = c["count"]
    n_desc = n - 1 - np.asarray(asap_alap(g)[1], np.int64) if n else np.zeros(0, np.int64)
    mi_mask = n_anc + n_desc == n - 1
    mi = sorted(np.nonzero(mi_mask)[0].tolist(), key=lambda v: int(n_anc[v]))
    mimask = np.zeros(anc.shape[1] * 8, bool)
    if mi:
        mimask[np.asarray(mi, np.int64)] = True
    gap = masked_counts(c["rows"], np.packbits(mimask, bitorder="little"))
    return mi, mi_mask, gap


def segment_tree_factory(mp):
    """Drop-in for segmentation.build_segment_tree (segmentation.py:451-476)
    and independent_segments (120-136), the inference-graph decomposition:
    the memory-insensitive ops and each op's number of MI ancestors come from
    the C++ closure instead of big-int masks popcounted per op; the nodes are
    the reference's own ``SubgraphNode`` with the same ids and fields."""
    seg, gr = mp.segmentation, mp.graph

    def independent_segments(g):
        c = closure(g)
        mi, mi_mask, gap = _mi_full(g, c)
        other = np.nonzero(~mi_mask)[0]
        out = []
        for k in range(len(mi) + 1):
            members = tuple(other[gap[other] == k].tolist())
            out.append(seg.Segment(lo=mi[k - 1] if k > 0 else None,
                                   hi=mi[k] if k < len(mi) else None, members=members))
        return out

    def build_segment_tree(g, node_limit):
        if node_limit < 2:
            raise gr.ConfigError("node_limit must be >= 2")
        children = []
        next_id = 1
        for s in independent_segments(g):
            if not s.members:
                continue
            children.append(seg.SubgraphNode(id=next_id, kind="independent", outer_fwd=s.lo, outer_bwd=s.hi,
                                             members=s.members, unsplittable=len(s.members) > node_limit))
            next_id += 1
        if not children:
            children.append(seg.SubgraphNode(id=next_id, kind="independent", tag="catchall"))
        mi, _, _ = _mi_full(g, closure(g))
        return seg.SubgraphNode(id=0, kind="root", children=tuple(children), pinned_ops=tuple(sorted(mi)))

    return independent_segments, build_segment_tree


def subgraph_tree_factory(mp):
    """Drop-in for segmentation.build_subgraph_tree (segmentation.py:343-448).

    The reference spends most of this function on bookkeeping, not on the
    tree: the core list tests membership in a set rebuilt for every op
    (O(n * |floating|)), ``_mi_over`` popcounts induced big-int masks, and the
    residual grouping tests ``before`` bit by bit.  Here those three come from
    the C++ ancestor bit matrix; the steps that shape the tree -- the
    inside-out independent-subgraph pairing, the residual runs and
    ``_split_if_oversized`` -- are the reference's own helpers, called in the
    same order on the reference's ``_TreeBuild`` (node ids come out the
    same).  ``_mi_over(g, core)`` uses the core's INDUCED closure; it equals
    the global closure on core rows because a relocatable branch's outputs
    are consumed only inside the branch (graph.py:541-545), so no path
    leaves the core through a floating op and comes back."""
    seg, gr = mp.segmentation, mp.graph

    def build_subgraph_tree(g, node_limit):
        if node_limit < 2:
            raise gr.ConfigError("node_limit must be >= 2")
        if not any(op.kind is gr.OpKind.BACKWARD for op in g.ops):
            raise gr.StructuralError("graph has no backward pass; segment it as an inference graph")
        branches = seg.weight_update_branches(g)
        floating = sorted(v for b in branches for v in b.ops)
        c = closure(g)
        n, anc = c["n"], c["anc"]
        is_core = np.ones(n, bool)
        if floating:
            is_core[np.asarray(floating, np.int64)] = False
        core = np.nonzero(is_core)[0].tolist()
        # the reference's predecessor masks (graph.py:335-348) as big ints
        preds = [int.from_bytes(anc[v].tobytes(), "little") for v in range(n)]
        build = _fast_build_type(seg)(g=g, node_limit=node_limit, preds=preds,
                                      categories=seg.classify_tensors(g), branches=branches)
        # _mi_over(g, core) (segmentation.py:108-117): ancestors within the core
        # + descendants within the core == |core| - 1, ordered by position
        cbytes = np.packbits(np.append(is_core, np.zeros(anc.shape[1] * 8 - n, bool)), bitorder="little")
        n_anc = masked_counts(c["rows"], cbytes)
        # descendants within the core = all descendants (n-1-alap, libroam C++)
        # minus the floating ones (column sums over the few floating rows)
        from .evaluator import asap_alap
        n_desc = n - 1 - np.asarray(asap_alap(g)[1], np.int64)
        if floating:
            blk = np.unpackbits(anc[np.asarray(floating, np.int64)], axis=1, bitorder="little")[:, :n]
            n_desc -= blk.sum(axis=0, dtype=np.int64)
        mi_mask = is_core & (n_anc + n_desc == len(core) - 1)
        mi_core = sorted(np.nonzero(mi_mask)[0].tolist(), key=lambda v: int(n_anc[v]))
        fwd_mi = [v for v in mi_core if g.ops[v].kind is gr.OpKind.FORWARD]
        bwd_mi = [v for v in mi_core if g.ops[v].kind is gr.OpKind.BACKWARD]

        # Every _region_between / _format_ig_ok call of the pairing loop
        # (segmentation.py:374-401) is bounded by memory-insensitive ops, which
        # are totally ordered and comparable with every core op: the MI
        # ancestors of a core op are a prefix m_0..m_{g-1} of that order, so
        # "strictly between m_a and m_b" is g in (a, b] for the other ops and
        # a < j < b for m_j itself.  Each call becomes a bucket lookup, and the
        # activation check only visits the tensors the members touch.
        pos_mi = {m: j for j, m in enumerate(mi_core)}
        mimask = np.zeros(anc.shape[1] * 8, bool)
        if mi_core:
            mimask[np.asarray(mi_core, np.int64)] = True
        gap = masked_counts(c["rows"], np.packbits(mimask, bitorder="little"))
        other = np.nonzero(is_core & ~mi_mask)[0]
        order = np.argsort(gap[other], kind="stable")
        bucket_ops = other[order]
        bucket_ptr = np.searchsorted(gap[other][order], np.arange(len(mi_core) + 2))
        mi_arr = np.asarray(mi_core, np.int64)

        def between(lo, hi):
            a, b = pos_mi[lo], pos_mi[hi]
            if a >= b:
                return []
            v = np.concatenate((bucket_ops[bucket_ptr[a + 1]:bucket_ptr[b + 1]], mi_arr[a + 1:b]))
            return np.sort(v).tolist()

        cats = build.categories
        tens = g.tensors
        act_out = [[t for t in op.outputs if cats[t] is gr.TensorCategory.ACTIVATION] for op in g.ops]
        act_in = [[t for t in op.inputs if cats[t] is gr.TensorCategory.ACTIVATION] for op in g.ops]

        def ig_ok(members, boundary):
            """segmentation.py:188-201 over the members' own tensors: an
            activation a member produces must have every consumer inside; one a
            member consumes must be produced inside."""
            inside = set(members) | boundary
            for v in members:
                for t in act_out[v]:
                    for u in tens[t].consumers:
                        if u not in inside:
                            return False
                for t in act_in[v]:
                    if tens[t].producer not in inside:
                        return False
            return True

        igs, used = [], []
        inner = None          # (inner_f, inner_b) of the last accepted pair
        for of, ob in zip(reversed(fwd_mi), bwd_mi):
            if inner is None:
                members = between(of, ob)
                boundary = {of, ob}
            else:
                members = sorted(between(of, inner[0]) + between(inner[1], ob))
                boundary = {of, ob, inner[0], inner[1]}
            if ig_ok(members, boundary):
                igs.append(build.new_node(kind="independent", outer_fwd=of,
                                          inner_fwd=None if inner is None else inner[0],
                                          inner_bwd=None if inner is None else inner[1],
                                          outer_bwd=ob, members=tuple(members),
                                          tag="middle" if inner is None else ""))
                used += [of, ob]
                inner = (of, ob)

        covered = np.zeros(n, bool)
        if used:
            covered[np.asarray(used, np.int64)] = True
        for node in igs:
            if node.members:
                covered[np.asarray(node.members, np.int64)] = True
        unc = np.nonzero(is_core & ~covered)[0]
        residuals = []
        if len(unc):
            # residual runs: uncovered ops grouped by how many pair boundaries
            # precede them (segmentation.py:408-418)
            sorted_used = sorted(set(used), key=lambda v: int(c["count"][v]))
            umask = np.zeros(anc.shape[1] * 8, bool)
            if sorted_used:
                umask[np.asarray(sorted_used, np.int64)] = True
            rank = masked_counts(c["rows"], np.packbits(umask, bitorder="little"), sel=unc)
            for r in sorted(set(rank.tolist())):
                lo = sorted_used[r - 1] if r > 0 else None
                hi = sorted_used[r] if r < len(sorted_used) else None
                residuals.append(build.new_node(kind="independent", outer_fwd=lo, outer_bwd=hi,
                                                members=tuple(unc[rank == r].tolist()), tag="residual"))

        for node in igs + residuals:
            seg._split_if_oversized(build, node, mi_core)
        children = igs + residuals
        if not children:
            children.append(build.new_node(kind="independent", tag="catchall"))
        children.append(build.new_node(kind="independent", tag="tail"))
        pinned = set()
        for node in children:
            pinned.update(node.boundary_ops())
            for ch in node.children:
                pinned.update(ch.boundary_ops())
        return seg.SubgraphNode(id=0, kind="root", members=(), children=tuple(children),
                                floating_ops=tuple(floating), pinned_ops=tuple(sorted(pinned)))
    return build_subgraph_tree


def weight_update_branches_factory(mp):
    """graph.py:513-557 weight_update_branches, computed once per graph (the
    planner asks seven times per plan: tree build, each linearisation, each
    weight-update placement); every call gets its own list of the
    reference's frozen WeightUpdateBranch records."""
    ref = mp.graph.weight_update_branches

    def weight_update_branches(g):
        ent = graph_cache(g)
        hit = ent.get("wu_branches")
        if hit is None:
            hit = ent["wu_branches"] = tuple(ref(g))
        return list(hit)
    return weight_update_branches


def assign_shared_tensors_factory(mp):
    """Drop-in for segmentation.assign_shared_tensors (segmentation.py:598-639).

    The reference places every floating weight-update op at the last window
    slot of its leaf by rescanning the whole slot sequence once per floating
    op (O(floating x slots): 0.4 s on the reference's 600-block graph); here
    one pass over the slots records each leaf's last window position.  The
    ownership rule itself (backward / weight-update / consumer-less tensors
    stay with their producer's leaf, the rest go to the leaf of their last
    consumer by (slot, id)) is unchanged, as is the owned_tensors side effect."""
    seg, gr = mp.segmentation, mp.graph

    def assign_shared_tensors(tree, g, leaf_of=None):
        lin = seg.linearize(g, tree)
        if leaf_of is None:
            leaf_of = lin.leaf_of_op
        slot_pos: dict[int, int] = {}
        last_win: dict[int, int] = {}
        for pos, (kind, ref) in enumerate(lin.slots):
            if kind == "op":
                slot_pos[ref] = pos
            else:
                w = lin.windows[ref]
                for v in w.ops:
                    slot_pos[v] = pos
                last_win[w.leaf] = pos
        for v in range(g.n_ops):
            if v not in slot_pos:
                slot_pos[v] = last_win.get(leaf_of[v], len(lin.slots))
        late = (gr.OpKind.BACKWARD, gr.OpKind.WEIGHT_UPDATE)
        ownership: dict[int, int] = {}
        owned: dict[int, list[int]] = {}
        for t in g.tensors:
            if not t.consumers or g.ops[t.producer].kind in late:
                leaf = leaf_of[t.producer]
            else:
                leaf = leaf_of[max(t.consumers, key=lambda c: (slot_pos[c], c))]
            ownership[t.id] = leaf
            owned.setdefault(leaf, []).append(t.id)
        for leaf in tree.leaves():
            leaf.owned_tensors = tuple(sorted(owned.get(leaf.id, [])))
        return ownership
    return assign_shared_tensors


def classify_tensors_factory(mp):
    """graph.py:471-492 classify_tensors, computed once per graph (the planner
    asks from the tree build, the weight-update cost table, plan() itself and
    validate_layout); every call gets its own dict of the reference's enums."""
    ref = mp.graph.classify_tensors

    def classify_tensors(g):
        ent = graph_cache(g)
        hit = ent.get("ref_categories")
        if hit is None:
            hit = ent["ref_categories"] = ref(g)
        return dict(hit)
    return classify_tensors


def linearize_factory(mp):
    seg = mp.segmentation
    build = _linearize_factory(mp)

    def linearize(g, root):
        """Computed once per (graph, tree): the planner linearises the same
        tree four times per plan (planner.py:198, ordering.py:404 twice,
        segmentation.py:608).  Callers get a fresh leaf_of_op dict each time."""
        ent = graph_cache(g)
        hit = ent.get("linearize")
        if hit is None or hit[0]() is not root:
            import weakref
            hit = ent["linearize"] = (weakref.ref(root), build(g, root))
        lin = hit[1]
        return seg.Linearization(slots=lin.slots, windows=lin.windows, leaf_of_op=dict(lin.leaf_of_op),
                                 tail_window=lin.tail_window)
    return linearize


def _linearize_factory(mp):
    seg, gr = mp.segmentation, mp.graph

    def linearize(g, root):
        """segmentation.py:500-572: the global slot skeleton (windows between
        boundary ops in forced order) with the gap rank of every op -- the
        number of boundary ops among its predecessors -- as one masked
        popcount over the ancestor bit matrix."""
        c = closure(g)
        n, anc, count = c["n"], c["anc"], c["count"]
        leaves = root.leaves()
        member_leaf: dict[int, int] = {}
        for leaf in leaves:
            for v in leaf.members:
                member_leaf[v] = leaf.id
        boundary_set: set[int] = set(root.pinned_ops)
        if not boundary_set:
            for node in root.walk():
                boundary_set.update(node.boundary_ops())
        boundaries = sorted(boundary_set, key=lambda v: int(count[v]))
        floating = set(root.floating_ops)

        bmask = np.zeros(anc.shape[1] * 8, bool)
        if boundaries:
            bmask[np.asarray(boundaries, np.int64)] = True
        bbytes = np.packbits(bmask, bitorder="little")
        rank = masked_counts(c["rows"], bbytes) if n else np.zeros(0, np.int64)
        skip = np.zeros(n, bool)
        for v in boundary_set | floating:
            skip[v] = True
        gap_ops: dict[int, list[int]] = {}
        for v in np.nonzero(~skip)[0].tolist():
            gap_ops.setdefault(int(rank[v]), []).append(v)

        windows: list = []
        slots: list[tuple[str, int]] = []
        gap_window: dict[int, int] = {}
        for gap in range(len(boundaries) + 1):
            ops = gap_ops.get(gap)
            if ops:
                owners = {member_leaf.get(v) for v in ops}
                if len(owners) != 1 or None in owners:
                    raise gr.StructuralError(f"window ops {ops} span leaves {owners}")
                windows.append(seg.Window(index=len(windows), leaf=owners.pop(), ops=tuple(ops)))
                gap_window[gap] = windows[-1].index
                slots.append(("win", windows[-1].index))
            if gap < len(boundaries):
                slots.append(("op", boundaries[gap]))

        tail_window = None
        for leaf in leaves:
            if leaf.tag == "tail":
                tail_window = len(windows)
                windows.append(seg.Window(index=tail_window, leaf=leaf.id, ops=()))
                slots.append(("win", tail_window))

        leaf_of_op: dict[int, int] = dict(member_leaf)
        catchall = next((leaf.id for leaf in leaves if leaf.tag == "catchall"), None)
        gaps = sorted(gap_window)
        for i, b in enumerate(boundaries):
            # the nearest non-empty window at or before the boundary's gap,
            # else the nearest after, else the catch-all leaf
            j = bisect.bisect_right(gaps, i)
            if j > 0:
                leaf_of_op[b] = windows[gap_window[gaps[j - 1]]].leaf
            elif j < len(gaps):
                leaf_of_op[b] = windows[gap_window[gaps[j]]].leaf
            elif catchall is not None:
                leaf_of_op[b] = catchall
            else:
                raise gr.StructuralError("no leaf available for boundary op assignment")

        for br in gr.weight_update_branches(g):
            if br.ops and br.ops[0] in floating:
                producer = g.tensors[br.gradients[0]].producer
                for v in br.ops:
                    leaf_of_op[v] = leaf_of_op[producer]

        return seg.Linearization(slots=tuple(slots), windows=tuple(windows), leaf_of_op=leaf_of_op,
                                 tail_window=tail_window)
    return linearize


def place_weight_updates_factory(mp):
    """Drop-in for ordering.place_weight_updates (ordering.py:387-467): the
    branch loop in libroam's host C++ (``rm_place_weight_updates``, wu_place.cpp)
    over the activation lifetimes swept once, returning the reference's own
    WeightUpdatePlan / BranchPlacement records.  The reference's callees stay
    the (rebound) module globals it would call: linearize, asap_alap,
    weight_update_branches, resolve_alpha (whose ConfigError surfaces for the
    first branch in the reference's placement order)."""
    import ctypes as C

    ordm, gr = mp.ordering, mp.graph

    def place_weight_updates(g, tree, r, alpha=None, *, force_immediate=False):
        alpha = ordm.DEFAULT_ALPHA if alpha is None else alpha
        lin = ordm.linearize(g, tree)
        bounds = ordm.asap_alap(g)
        floating = set(tree.floating_ops)
        branches = [b for b in ordm.weight_update_branches(g) if b.ops and b.ops[0] in floating]
        T = g.n_tensors
        mean_size = sum(t.size for t in g.tensors) / T if T else 0.0
        n = g.n_ops
        asap = np.asarray(bounds.asap, np.int32)
        alap = np.asarray(bounds.alap, np.int64)
        a = graph_arrays(g)
        cats = ordm.classify_tensors(g)
        act = np.fromiter((cats[t] is gr.TensorCategory.ACTIVATION for t in range(T)), bool, T)
        ids = np.flatnonzero(act)
        cp = np.asarray(a.cons_ptr, np.int64)
        # max alap over each tensor's consumers (horizon n - 1 without any)
        tend = np.full(T, n - 1, np.int64)
        nz = np.flatnonzero(cp[1:] > cp[:-1])
        if len(nz):
            tend[nz] = np.maximum.reduceat(alap[np.asarray(a.cons_idx, np.int64)], cp[nz])
        end = tend[ids]
        act_start = asap[np.asarray(a.producer, np.int64)[ids]].astype(np.int32) if len(ids) else np.zeros(0, np.int32)
        act_end = end.astype(np.int32)
        act_size = np.asarray(a.size, np.int64)[ids]
        # slot skeleton: kind 0 = op, 1 = window
        S = len(lin.slots)
        kind = np.fromiter((0 if k == "op" else 1 for k, _ in lin.slots), np.int32, S)
        ref = np.fromiter((v for _, v in lin.slots), np.int32, S)
        W = len(lin.windows)
        wlen = np.fromiter((len(w.ops) for w in lin.windows), np.int64, W)
        wptr = np.zeros(W + 1, np.int64)
        np.cumsum(wlen, out=wptr[1:])
        wops = np.fromiter((v for w in lin.windows for v in w.ops), np.int32, int(wptr[-1]))
        B = len(branches)
        alphas = []
        for b in branches:
            try:
                alphas.append(ordm.resolve_alpha(g, b, alpha))
            except gr.ConfigError:
                # the reference resolves alphas in placement order: raise for
                # the first unresolvable branch in that order
                key = lambda b: (max(bounds.asap[g.tensors[t].producer] for t in b.gradients), b.ops[0])  # noqa: E731
                for bb in sorted(branches, key=key):
                    ordm.resolve_alpha(g, bb, alpha)
                raise
        first = np.fromiter((b.ops[0] for b in branches), np.int32, B)
        glen = np.fromiter((len(b.gradients) for b in branches), np.int64, B)
        gptr = np.zeros(B + 1, np.int64)
        np.cumsum(glen, out=gptr[1:])
        gprod = np.fromiter((g.tensors[t].producer for b in branches for t in b.gradients), np.int32,
                            int(gptr[-1]))
        gbytes = np.fromiter((b.grad_bytes for b in branches), np.int64, B)
        alph = np.asarray(alphas, np.float64)
        o_b, o_t, o_r = (np.zeros(B, np.int32) for _ in range(3))
        o_d = np.zeros(B, np.uint8)
        o_ratio, o_proj = np.zeros(B), np.zeros(B)
        total, missing = C.c_int64(0), C.c_int32(-1)
        rc = lib().rm_place_weight_updates(
            n, ptr(asap), len(ids), ptr(act_start), ptr(act_end), ptr(act_size), float(mean_size), S,
            ptr(kind), ptr(ref), W, ptr(wptr), ptr(wops),
            -1 if lin.tail_window is None else int(lin.tail_window), B, ptr(first), ptr(gptr), ptr(gprod),
            ptr(gbytes), ptr(alph), float(r), 1 if force_immediate else 0, ptr(o_b), ptr(o_d), ptr(o_t),
            ptr(o_r), ptr(o_ratio), ptr(o_proj), C.byref(total), C.byref(missing))
        if missing.value >= 0:
            raise KeyError(missing.value)
        check(rc, "rm_place_weight_updates")
        placements = tuple(
            ordm.BranchPlacement(branch=branches[b], delayed=bool(d), target_window=t,
                                 target_leaf=lin.windows[t].leaf, alpha=alphas[b], size_ratio=ratio,
                                 ready_t=rt, projected_use=pu)
            for b, d, t, rt, ratio, pu in zip(o_b.tolist(), o_d.tolist(), o_t.tolist(), o_r.tolist(),
                                               o_ratio.tolist(), o_proj.tolist()))
        return ordm.WeightUpdatePlan(placements=placements, activation_total=int(total.value))
    return place_weight_updates
