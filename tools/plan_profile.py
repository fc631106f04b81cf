"""cProfile of one planner run with the B200 path installed (host-side
hot spots): python tools/plan_profile.py [config] [--sort tottime|cumulative]"""
from __future__ import annotations

import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_19295_b200 import graphgen as gg  # noqa: E402
from paper_2310_19295_b200 import memplan_plugin as plug  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gpt2-xl"
sort = sys.argv[3] if len(sys.argv) > 3 and sys.argv[2] == "--sort" else "tottime"
mp = plug.load_memplan()
plug.install(mp)
mp.planner.plan(mp.graph.load_graph(gg.config_doc("layered")))
import memplan.graphgen as rgen  # noqa: E402
mp.planner.plan(rgen.gen_training_graph("transformer_block", 2))
if name.startswith("ref-"):
    import memplan.graphgen as rgen
    _, arch, blocks = name.split("-")
    g = rgen.gen_training_graph(arch, int(blocks))
else:
    g = mp.graph.load_graph(gg.config_doc(name))
pr = cProfile.Profile()
pr.enable()
mp.planner.plan(g)
pr.disable()
pstats.Stats(pr).sort_stats(sort).print_stats(35)
