"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain-Python restatement of the reference ROAM planner's hot-path algorithms
(/root/reference/pkg/src/memplan, cited per function).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm may
import this module, and only as the checker or the timed CPU baseline; the
product path (``paper_2310_19295_b200``) never routes through it.

Pinned against the real reference: ``tests/golden/make_golden.py`` imports the
reference (in the build container) and freezes its outputs into
``tests/golden/*.json``; ``tests/test_oracle_golden.py`` checks this module
against every vector.  The functions take reference-shaped graphs (``.ops``
with ``.inputs/.outputs/.kind``, ``.tensors`` with ``.size/.producer/
.consumers``) and plain tuples, never the product package's types.
"""

from __future__ import annotations

import heapq

MASK64 = (1 << 64) - 1


class OracleScheduleError(Exception):
    pass


class OracleConfigError(Exception):
    pass


# ------------------------------------------------------------ graph.py

def direct_preds(g) -> list[tuple[int, ...]]:
    """graph.py:97-104."""
    out = []
    for op in g.ops:
        p = {g.tensors[t].producer for t in op.inputs}
        p.discard(op.id)
        out.append(tuple(sorted(p)))
    return out


def direct_succs(g) -> list[tuple[int, ...]]:
    """graph.py:106-116."""
    out = []
    for op in g.ops:
        s: set[int] = set()
        for t in op.outputs:
            s.update(g.tensors[t].consumers)
        s.discard(op.id)
        out.append(tuple(sorted(s)))
    return out


def validate_schedule(g, order, timesteps, ops_per_step: int = 1, preds=None) -> None:
    """graph.py:375-398, same check order and messages."""
    n = len(g.ops)
    if sorted(order) != list(range(n)):
        raise OracleScheduleError("schedule must contain every op exactly once")
    if len(timesteps) != n:
        raise OracleScheduleError("timesteps must cover every op")
    if ops_per_step < 1:
        raise OracleConfigError("ops_per_step must be >= 1")
    pos = {op: i for i, op in enumerate(order)}
    last = -1
    for op in order:
        t = timesteps[op]
        if t < last:
            raise OracleScheduleError("timesteps must be non-decreasing along the order")
        last = t
    counts: dict[int, int] = {}
    for t in timesteps:
        counts[t] = counts.get(t, 0) + 1
        if counts[t] > ops_per_step:
            raise OracleScheduleError(f"timestep {t} holds more than {ops_per_step} ops")
    preds = preds if preds is not None else direct_preds(g)
    for v in range(n):
        for p in preds[v]:
            if pos[p] > pos[v] or timesteps[p] > timesteps[v]:
                raise OracleScheduleError(f"op {v} scheduled before its predecessor {p}")


def tensor_lifetimes(g, timesteps) -> list[tuple[int, int]]:
    """graph.py:440-449 (horizon = n_steps - 1, n_steps = max + 1)."""
    horizon = (max(timesteps) + 1 if timesteps else 0) - 1
    spans = []
    for t in g.tensors:
        b = timesteps[t.producer]
        d = max((timesteps[c] for c in t.consumers), default=horizon)
        spans.append((b, max(b, d)))
    return spans


def live_bytes_by_timestep(g, timesteps) -> list[int]:
    """graph.py:452-458: the O(sum of lifetimes) add loop."""
    steps = max(timesteps) + 1 if timesteps else 0
    live = [0] * steps
    for tensor, (b, d) in zip(g.tensors, tensor_lifetimes(g, timesteps)):
        for t in range(b, d + 1):
            live[t] += tensor.size
    return live


def sequential_timesteps(n: int, order) -> list[int]:
    """graph.py:401-409 timestep = position."""
    ts = [0] * n
    for i, op in enumerate(order):
        ts[op] = i
    return ts


def peak_memory(g, order, timesteps=None, ops_per_step: int = 1, preds=None) -> tuple[int, int]:
    """graph.py:461-468 (validates first; (0, 0) for an empty graph)."""
    n = len(g.ops)
    if timesteps is None:
        if sorted(order) != list(range(n)):
            raise OracleScheduleError("schedule must contain every op exactly once")
        timesteps = sequential_timesteps(n, order)
    validate_schedule(g, order, timesteps, ops_per_step, preds)
    if n == 0:
        return 0, 0
    live = live_bytes_by_timestep(g, timesteps)
    peak = max(live)
    return peak, live.index(peak)


def evaluate_order(g, order, preds=None) -> tuple[int, int, bool]:
    """Batch-element semantics of K1: (peak, argmax, valid) of a sequential
    schedule; invalid rows report (0, 0, False) (the reference raises)."""
    try:
        p, a = peak_memory(g, order, preds=preds)
        return p, a, True
    except (OracleScheduleError, OracleConfigError):
        return 0, 0, False


def first_strict_min(peaks, valids) -> tuple[int | None, int]:
    """tests/oracles.py:46-56 / planner.py:209-216: keep a candidate only if
    strictly better."""
    best, best_i = None, -1
    for i, (p, v) in enumerate(zip(peaks, valids)):
        if v and (best is None or p < best):
            best, best_i = p, i
    return best, best_i


# ----------------------------------------------------- candidate generator

def mix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def kahn_candidate(n: int, preds, succs, seed: int, cand_id: int) -> list[int]:
    """Counter-RNG Kahn order: pop the ready op with the smallest
    (mix(h ^ op), op), h = mix(seed ^ mix(cand_id)).  Restated by the device
    generator (csrc/k_gen.cu)."""
    h = mix64((seed & MASK64) ^ mix64(cand_id & MASK64))
    indeg = [len(p) for p in preds]
    ready = [(mix64(h ^ v), v) for v in range(n) if indeg[v] == 0]
    heapq.heapify(ready)
    order = []
    while ready:
        _, v = heapq.heappop(ready)
        order.append(v)
        for w in succs[v]:
            indeg[w] -= 1
            if indeg[w] == 0:
                heapq.heappush(ready, (mix64(h ^ w), w))
    return order + [-1] * (n - len(order))


# ------------------------------------------------------------ layout.py
# items are tuples (tensor, size, start, end, is_activation)

def overlaps(a, b) -> bool:
    """LayoutItem.overlaps, layout.py:28-29 (inclusive)."""
    return a[2] <= b[3] and b[2] <= a[3]


def layout_violations(items, offsets: dict, capacity: int) -> list[str]:
    """layout.py:305-329, same message order."""
    out: list[str] = []
    have = []
    for it in items:
        t = it[0]
        if t not in offsets:
            out.append(f"tensor {t} has no offset")
            continue
        off = offsets[t]
        if off < 0:
            out.append(f"tensor {t} has negative offset {off}")
        if off + it[1] > capacity:
            out.append(f"tensor {t} extent {off + it[1]} exceeds capacity {capacity}")
        have.append((it, off))
    for i, (a, ao) in enumerate(have):
        for b, bo in have[i + 1:]:
            if overlaps(a, b) and ao < bo + b[1] and bo < ao + a[1]:
                out.append(f"tensors {a[0]} and {b[0]} overlap in time and address")
    return out


def replay_static_extent(items, offsets: dict) -> int:
    """simulator.py:137-145: max over steps of max(off + size) over live items."""
    steps = max((it[3] for it in items), default=-1) + 1
    actual = 0
    for t in range(steps):
        ext = 0
        for it in items:
            if it[2] <= t <= it[3] and it[0] in offsets:
                ext = max(ext, offsets[it[0]] + it[1])
        actual = max(actual, ext)
    return actual


def lowest_fit(item, placed, floor: int = 0) -> int:
    """layout.py:71-78."""
    spans = sorted((off, off + it[1]) for it, off in placed if overlaps(it, item))
    cand = floor
    for lo, hi in spans:
        if cand + item[1] <= lo:
            break
        cand = max(cand, hi)
    return cand


def llfb_layout(items) -> tuple[dict, int]:
    """layout.py:100-118: sort by (-(end-start), -size, tensor), lowest fit."""
    order = sorted(items, key=lambda i: (-(i[3] - i[2]), -i[1], i[0]))
    placed, cap = [], 0
    for it in order:
        off = lowest_fit(it, placed)
        placed.append((it, off))
        cap = max(cap, off + it[1])
    return {it[0]: off for it, off in placed}, cap


def activation_floors(items):
    """layout.py:81-97."""
    atvs = sorted((i for i in items if i[4]), key=lambda i: (-(i[3] - i[2]), i[0]))
    placed, off = [], 0
    for a in atvs:
        placed.append((a, off))
        off += a[1]
    floors = {}
    for i in items:
        if i[4]:
            continue
        floors[i[0]] = off if any(overlaps(i, a) for a in atvs) else 0
    return placed, floors, off


def constrained_llfb_layout(items) -> tuple[dict, int]:
    """layout.py:121-146."""
    placed, floors, _ = activation_floors(items)
    rest = sorted((i for i in items if not i[4]), key=lambda i: (-(i[3] - i[2]), -i[1], i[0]))
    cap = sum(a[1] for a, _ in placed)
    for it in rest:
        off = lowest_fit(it, placed, floors[it[0]])
        placed.append((it, off))
        cap = max(cap, off + it[1])
    return {it[0]: off for it, off in placed}, cap


def component_incumbents(items):
    """exact_layout's pre-search part with activations_at_bottom
    (layout.py:165-225): union-find components of non-activation items,
    per-component bound and lowest-fit incumbent.  Returns
    (offsets, capacity, all_bounds_met, {root: (bound, incumbent_cap)})."""
    pre, floors, block_top = activation_floors(items)
    rest = [i for i in items if not i[4]]
    parent = {i[0]: i[0] for i in rest}

    def find(t):
        while parent[t] != t:
            parent[t] = parent[parent[t]]
            t = parent[t]
        return t

    for k, a in enumerate(rest):
        for b in rest[k + 1:]:
            if overlaps(a, b):
                ra, rb = find(a[0]), find(b[0])
                if ra != rb:
                    parent[max(ra, rb)] = min(ra, rb)
    groups: dict[int, list] = {}
    for it in rest:
        groups.setdefault(find(it[0]), []).append(it)
    offsets = {it[0]: off for it, off in pre}
    capacity = block_top
    met = True
    comps = {}
    for root in sorted(groups):
        comp = sorted(groups[root], key=lambda i: (-(i[3] - i[2]), -i[1], i[0]))
        bound = 0
        for probe in comp:
            t = probe[2]
            live = [i for i in comp if i[2] <= t <= i[3]]
            total = sum(i[1] for i in live)
            above = sum(i[1] for i in live if floors[i[0]])
            bound = max(bound, total, (block_top + above) if above else 0)
        placed, best = [], 0
        for it in comp:
            off = lowest_fit(it, placed, floors[it[0]])
            placed.append((it, off))
            best = max(best, off + it[1])
        comps[root] = (bound, best)
        if best > bound:
            met = False
        offsets.update({it[0]: off for it, off in placed})
        capacity = max(capacity, best)
    return offsets, capacity, met, comps


# ----------------------------------------------------------- ordering.py

def greedy_order(g, ops, live_in=(), live_out=()) -> tuple[tuple[int, ...], int]:
    """ordering.py:78-123 (_Local) + 126-180 (greedy_order)."""
    ops = tuple(sorted(ops))
    inside = set(ops)
    index = {v: i for i, v in enumerate(ops)}
    live_in, live_out = set(live_in), set(live_out)
    produced = {t for v in ops for t in g.ops[v].outputs}
    tracked, held, sizes = {}, set(), {}
    for t in sorted(produced | live_in):
        info = g.tensors[t]
        local = sum(1 for c in info.consumers if c in inside)
        sizes[t] = info.size
        tracked[t] = local
        if t in live_out or (t in produced and local == 0):
            held.add(t)
        elif t in live_in and local == 0:
            raise OracleConfigError(f"live-in tensor {t} has no consumer in the window and is not live-out")
    live = sum(sizes[t] for t in sorted(live_in))
    out_bytes = [sum(g.tensors[t].size for t in g.ops[v].outputs) for v in ops]
    pred_mask = []
    for v in ops:
        m = 0
        for t in g.ops[v].inputs:
            p = g.tensors[t].producer
            if p in inside and p != v:
                m |= 1 << index[p]
        pred_mask.append(m)
    n = len(ops)
    counts = dict(tracked)
    peak = live
    sched = 0
    order = []
    while len(order) < n:
        best = None
        for i in range(n):
            if sched >> i & 1 or (pred_mask[i] & ~sched):
                continue
            freed, seen = 0, set()
            for t in g.ops[ops[i]].inputs:
                if t in seen or t not in counts or t in held:
                    continue
                seen.add(t)
                if counts[t] == 1:
                    freed += sizes[t]
            delta = out_bytes[i] - freed
            if best is None or delta < best[0]:
                best = (delta, i)
        if best is None:
            raise OracleConfigError("window precedence contains a cycle")
        i = best[1]
        v = ops[i]
        live += out_bytes[i]
        peak = max(peak, live)
        seen = set()
        for t in g.ops[v].inputs:
            if t in seen or t not in counts:
                continue
            seen.add(t)
            counts[t] -= 1
            if counts[t] == 0 and t not in held:
                live -= sizes[t]
        sched |= 1 << i
        order.append(v)
    return tuple(order), peak


def _window_local(g, ops, live_in, live_out):
    """ordering.py:78-123 (_Local) reduced to what the exact DP needs:
    local op order, pred masks, out bytes, start_live, and the freeable
    tensors as (consumer mask, size).  A tensor frees when its count of local
    consumer ENTRIES reaches 0 with one decrement per distinct consuming op, so
    an op listing an input twice keeps it live (hazard h1)."""
    ops = tuple(sorted(ops))
    inside = set(ops)
    index = {v: i for i, v in enumerate(ops)}
    live_in, live_out = set(live_in), set(live_out)
    produced = {t for v in ops for t in g.ops[v].outputs}
    freeable = []
    for t in sorted(produced | live_in):
        info = g.tensors[t]
        local = sum(1 for c in info.consumers if c in inside)
        if t in live_out or (t in produced and local == 0):
            continue                                   # held
        if t in live_in and local == 0:
            raise OracleConfigError(f"live-in tensor {t} has no consumer in the window and is not live-out")
        cons = {c for c in info.consumers if c in inside}
        if len(cons) == local:                        # else never reaches 0 (duplicate entries)
            m = 0
            for c in cons:
                m |= 1 << index[c]
            freeable.append((m, info.size))
    start = sum(g.tensors[t].size for t in sorted(live_in))
    out_bytes = [sum(g.tensors[t].size for t in g.ops[v].outputs) for v in ops]
    pred_mask = []
    for v in ops:
        m = 0
        for t in g.ops[v].inputs:
            p = g.tensors[t].producer
            if p in inside and p != v:
                m |= 1 << index[p]
        pred_mask.append(m)
    return ops, pred_mask, out_bytes, start, freeable


def exact_order_dp(g, ops, live_in=(), live_out=(), node_cap=None):
    """ordering.py:183-286 (exact_order) restated as a DP over the window's
    order ideals (SURVEY §8 hazard h10):

      V[full] = 0,  V[mask] = min over ready i of max(live(mask) + out[i], V[mask | i])

    then the walk from mask 0 takes the smallest local index i (= ascending op
    id) with max(live + out[i], V[mask | i]) <= V[mask]; peak = max(V[0],
    start_live).  The reference's memoised DFS expands each order ideal at
    most once, so when (#ideals - 1) <= node_cap it never hits its cap and
    returns exactly this; otherwise its answer depends on how far its pruned
    DFS gets, and this function returns None.  Returns (order, peak, #ideals)."""
    ops, pred, out, start, freeable = _window_local(g, ops, live_in, live_out)
    n = len(ops)
    if n == 0:
        return (), start, 1
    full = (1 << n) - 1
    down = [m for m in range(1 << n) if all(not (m >> i & 1) or not (pred[i] & ~m) for i in range(n))]
    if node_cap is not None and len(down) - 1 > node_cap:
        return None

    def live(m):
        s = start + sum(out[i] for i in range(n) if m >> i & 1)
        return s - sum(sz for cm, sz in freeable if cm & m == cm)

    V = {full: 0}
    for m in sorted(down, key=lambda x: -bin(x).count("1")):
        if m == full:
            continue
        lv = live(m)
        V[m] = min(max(lv + out[i], V[m | 1 << i]) for i in range(n)
                   if not (m >> i & 1) and not (pred[i] & ~m))
    order, m = [], 0
    while m != full:
        lv = live(m)
        for i in range(n):
            if m >> i & 1 or pred[i] & ~m:
                continue
            if max(lv + out[i], V[m | 1 << i]) <= V[m]:
                break
        order.append(ops[i])
        m |= 1 << i
    return tuple(order), max(V[0], start), len(down)
