"""One small pass over every libroam kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck) -- see tools/gpu_sanitize.sh.

Covers K1 (default variant and the generic v1, int32 and uint16 rows,
corrupted rows, the fused packed-key selection launched back to back so
programmatic dependent launch overlaps the launches), the generator, the
argmin kernels, the single-schedule kernels, K2, K3 (plain, constrained,
components), K4, K5, the thread- and warp-form generators, the
repair_conflicts rounds and the whole plug-in path through the reference's own
plan() on small graphs.  Sizes are small: racecheck slows shared-memory
kernels by two to three orders of magnitude."""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2310_19295_b200 import evaluator as ev  # noqa: E402
from paper_2310_19295_b200 import graphgen as gg  # noqa: E402
from paper_2310_19295_b200 import layout as lay  # noqa: E402
from paper_2310_19295_b200 import memplan_plugin as plug  # noqa: E402
from paper_2310_19295_b200.graph import load_graph  # noqa: E402


def main(which: str = "all") -> None:
    torch.cuda.set_device(0)
    g = load_graph(gg.config_doc("gpt2-small"))
    B = 96
    orders = ev.generate_orders(g, 0, 0, B)
    bad = orders.clone()
    bad[1, 5] = bad[1, 6]           # duplicate
    bad[2, [10, 400]] = bad[2, [400, 10]]  # precedence violation
    bad[3, 7] = 999999              # out of range
    u16 = orders.to(torch.int32).clamp(0, 65535).to(torch.uint16)
    for rows in (orders, bad, u16):
        pk, am, vl = ev.evaluate_orders(g, rows)
        ev.select_device(pk, vl)
    if which in ("all", "k1"):
        for _ in range(3):   # back to back: PDL overlap + fused selection counter reuse
            ev.evaluate_select_key(g, orders, 0, 20)
        ev.set_k1_variant(1)
        ev.evaluate_orders(g, bad)
        ev.set_k1_variant(0)
        ev.evaluate_live(g, bad)      # batched live bytes, corrupted rows included
        torch.cuda.synchronize()
    if which in ("all", "gen"):
        # the thread-per-candidate generator, and the warp form it hands the
        # rows over to (layered: ready sets above the heap's capacity)
        ev.generate_orders(g, 3, 0, 64)
        ev.generate_orders(load_graph(gg.layered_dag_doc(layers=12, width=20)), 3, 0, 40)
        torch.cuda.synchronize()
    if which in ("all", "plan"):
        mp = plug.load_memplan()
        small = [mp.graph.load_graph(gg.layered_dag_doc(layers=6, width=8)),
                 importlib.import_module("memplan.graphgen").gen_training_graph("transformer_block", 2)]
        plug.install(mp)
        try:
            for gr in small:
                p = mp.planner.plan(gr)
                mp.simulator.replay_static(gr, p.schedule, p.layout)
        finally:
            plug.uninstall()
        items = [lay.LayoutItem(t, 1 + (7 * t) % 5, t % 9, t % 9 + 3, t % 4 == 0) for t in range(300)]
        for mode in (lay.PLAIN, lay.CONSTRAINED):
            lay.pack_batch([items, items[:40]], mode)
        # K3's DAG rounds (every problem) and their fallback on a dense one
        lay.set_pack_form(2)
        try:
            for mode in (lay.PLAIN, lay.CONSTRAINED, lay.COMPONENTS):
                lay.pack_batch([items, items[:40]], mode)
            dense = [lay.LayoutItem(t, 1 + t % 3, 0, 5, False) for t in range(80)]
            lay.pack_batch([dense], lay.PLAIN)
        finally:
            lay.set_pack_form(0)
        offs = {i.tensor: (13 * i.tensor) % 50 for i in items}
        lay.layout_violations(items, offs, 40)
        # repair_conflicts: device pair test + mover election over several rounds
        lay.repair_conflicts(mp.layout.MemoryLayout(offsets=offs, capacity=60),
                             mp.layout.LayoutProblem(items=tuple(items)))
    torch.cuda.synchronize()
    print(f"sanitize_run {which} ok; libroam launches={ev.launch_count()}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
