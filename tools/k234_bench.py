"""K2 / K3 / K4 on the planner's real subtasks (not HBM-bound;
reported as pairs/s, problems/s and items/s next to the reference's own
functions on the host CPU).

  python tools/k234_bench.py [--configs bert-large gpt2-xl] [--out f.json]

For each config graph the reference planner runs once with its batch dispatch
(_pool_map) wrapped to capture every window and leaf problem it solves.  Then:
  K3: all leaf layout problems in ONE rm_llfb_batch launch (constrained LLFB
      for leaves over layout_limit, exact-layout incumbent+bound for the rest)
      vs the reference's constrained_llfb_layout / exact_layout per leaf;
  K4: all greedy windows (over node_limit) in one rm_greedy_windows launch vs
      the reference's greedy_order per window;
  K2: layout_violations over the final plan's items (N = n_tensors) vs the
      reference's layout_violations.
Results are compared for equality before timing."""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2310_19295_b200 import graphgen as gg  # noqa: E402
from paper_2310_19295_b200 import layout as L  # noqa: E402
from paper_2310_19295_b200 import memplan_plugin as plug  # noqa: E402
from paper_2310_19295_b200 import ordering as Ord  # noqa: E402


def best_of(fn, reps=3):
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t0
        best = dt if best is None or dt < best else best
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["bert-large", "gpt2-xl"])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    mp = plug.load_memplan()
    rows = []
    for name in a.configs:
        g = mp.graph.load_graph(gg.config_doc(name))
        captured = {"win": [], "lay": []}
        orig = mp.planner._pool_map

        def capture(fn, jobs, workers):
            jobs = list(jobs)
            if fn is mp.planner._solve_window:
                captured["win"].extend(jobs)
            elif fn is mp.planner._solve_layout:
                captured["lay"].extend(jobs)
            return orig(fn, jobs, workers)

        mp.planner._pool_map = capture
        try:
            plan = mp.planner.plan(g)
        finally:
            mp.planner._pool_map = orig
        row = {"config": name, "n_ops": len(g.ops), "n_tensors": len(g.tensors)}

        # ---- K3: every leaf of the plan
        big = [p for p, lim in captured["lay"] if len(p.items) > lim]
        small = [p for p, lim in captured["lay"] if len(p.items) <= lim]
        items = sum(len(p.items) for p in big + small)
        t_ref, ref_big = best_of(lambda: [mp.layout.constrained_llfb_layout(p) for p in big], 2)
        t_ref2, ref_small = best_of(lambda: [mp.layout.exact_layout(p) for p in small], 2)
        L.pack_batch([p.items for p in big], L.CONSTRAINED)   # warm
        t_k3, got_big = best_of(lambda: L.pack_batch([p.items for p in big], L.CONSTRAINED))
        t_k3b, got_small = best_of(lambda: L.exact_layout_batch(small))
        assert all(r.offsets == m.offsets and r.capacity == m.capacity for r, m in zip(got_big, ref_big))
        assert all(r is None or (r.offsets == m.offsets and r.capacity == m.capacity)
                   for r, m in zip(got_small, ref_small))
        row["k3"] = {"leaves": len(big) + len(small), "items": items,
                     "big_leaf_items": [len(p.items) for p in big],
                     "reference_s": t_ref + t_ref2, "b200_s": t_k3 + t_k3b,
                     "items_per_s": items / (t_k3 + t_k3b),
                     "speedup": (t_ref + t_ref2) / (t_k3 + t_k3b)}

        # ---- K4: every greedy window
        gw = [p for p, lim in captured["win"] if len(p.ops) > lim]
        if gw:
            t_ref, ref_w = best_of(lambda: [mp.ordering.greedy_order(p) for p in gw], 2)
            Ord.greedy_windows(gw)
            t_k4, got_w = best_of(lambda: Ord.greedy_windows(gw))
            assert all(o == (s.order, s.peak) for o, s in zip(got_w, ref_w))
            ops = sum(len(p.ops) for p in gw)
            row["k4"] = {"windows": len(gw), "ops": ops, "window_ops": [len(p.ops) for p in gw],
                         "reference_s": t_ref, "b200_s": t_k4, "ops_per_s": ops / t_k4,
                         "speedup": t_ref / t_k4}

        # ---- K2: the final plan's full item set
        its = mp.layout.items_from_schedule(g, plan.schedule)
        offs, cap = plan.layout.offsets, plan.layout.capacity
        N = len(its)
        t_ref, ref_v = best_of(lambda: mp.layout.layout_violations(its, offs, cap), 1)
        L.layout_violations(its, offs, cap)
        t_k2, got_v = best_of(lambda: L.layout_violations(its, offs, cap))
        assert got_v == ref_v
        pairs = N * (N - 1) // 2
        row["k2"] = {"items": N, "pair_tests": pairs, "reference_s": t_ref, "b200_s": t_k2,
                     "pairs_per_s": pairs / t_k2, "speedup": t_ref / t_k2}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(rows, indent=1) + "\n")


if __name__ == "__main__":
    main()
