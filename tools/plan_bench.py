"""End-to-end planning time (BASELINE config 1 and 4): the reference's own
``plan(g)`` on the host CPU vs the same planner with the B200 hot path
installed (memplan_plugin), plan documents checked byte-identical.

  python tools/plan_bench.py [--configs layered gpt2-small bert-large gpt2-xl] [--out f.json]

Each planner runs once per config after warm-up plans of two small graphs (the
reference is deterministic; wall clock, single process).  For the GPU run the
top functions by cumulative time are recorded (cProfile) to show what stays on
the host."""

from __future__ import annotations

import argparse
import cProfile
import io
import json
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2310_19295_b200 import graphgen as gg  # noqa: E402
from paper_2310_19295_b200 import memplan_plugin as plug  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["layered", "gpt2-small", "bert-large", "gpt2-xl"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--skip-ref", action="store_true")
    a = ap.parse_args()
    mp = plug.load_memplan()
    import memplan.graphgen as rgen
    # warm-up: an inference graph and a small training graph, so both planner
    # paths have loaded their modules and the CUDA context exists
    warm = mp.graph.load_graph(gg.config_doc("layered"))
    warm_train = rgen.gen_training_graph("transformer_block", 2)
    plug.install(mp)
    mp.planner.plan(warm)       # CUDA context, module loads
    mp.planner.plan(warm_train)
    plug.uninstall()
    rows = []
    for name in a.configs:
        if name.startswith("ref-"):   # the reference's own generator, e.g. ref-transformer_block-600
            import memplan.graphgen as rgen
            _, arch, blocks = name.split("-")
            g = rgen.gen_training_graph(arch, int(blocks))
        else:
            g = mp.graph.load_graph(gg.config_doc(name))
        row = {"config": name, "n_ops": len(g.ops), "n_tensors": len(g.tensors)}
        if not a.skip_ref:
            t0 = time.perf_counter()
            ref = mp.planner.plan_doc_bytes(mp.planner.plan(g))
            row["reference_s"] = time.perf_counter() - t0
        plug.install(mp)
        try:
            prof = cProfile.Profile()
            t0 = time.perf_counter()
            prof.enable()
            got = mp.planner.plan_doc_bytes(mp.planner.plan(g))
            prof.disable()
            row["b200_s"] = time.perf_counter() - t0
            row["dispatch"] = dict(plug.STATS)
        finally:
            plug.uninstall()
        if not a.skip_ref:
            row["identical"] = got == ref
            row["speedup"] = row["reference_s"] / row["b200_s"]
        s = io.StringIO()
        pstats.Stats(prof, stream=s).sort_stats("cumulative").print_stats(30)
        row["b200_top_cumulative"] = [l.strip() for l in s.getvalue().splitlines()
                                      if l.strip() and l.strip()[0].isdigit()][:14]
        doc = json.loads(got)
        row["theoretical_peak"] = doc["stats"]["theoretical_peak"]
        row["capacity"] = doc["capacity"]
        rows.append(row)
        print(json.dumps({k: v for k, v in row.items() if k != "b200_top_cumulative"}), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(rows, indent=1) + "\n")


if __name__ == "__main__":
    main()
