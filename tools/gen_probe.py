"""Generator probe: time the candidate generator (both forms) on a config
graph; with --once, a single launch (for ncu)."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_19295_b200 import evaluator as ev  # noqa: E402
from paper_2310_19295_b200 import graphgen as gg  # noqa: E402
from paper_2310_19295_b200.graph import load_graph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--graphs", nargs="+", default=["gpt2-small", "gpt2-xl"])
ap.add_argument("--B", type=int, default=65536)
ap.add_argument("--once", action="store_true")
ap.add_argument("--forms", type=int, nargs="+", default=[0, 1], help="0 auto, 1 warp form, 40/64 heap caps")
a = ap.parse_args()
for name in a.graphs:
    g = load_graph(gg.config_doc(name))
    if a.once:
        ev.generate_orders(g, 0, 0, a.B)
        torch.cuda.synchronize()
        continue
    for form in a.forms:
        ev.set_gen_form(form)
        B = a.B if form != 1 else 8192
        del_ = ev.generate_orders(g, 1, 0, B)   # warm-up; its memory is reused below
        del del_
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ev.generate_orders(g, 0, 0, B)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(name, "form", form, "B", B, "ms", round(ms, 3), "cand/s", round(B / ms * 1e3), flush=True)
    ev.set_gen_form(0)
