"""Back-to-back K1 launches (fused selection, rotating 3 batch copies) timed as
one CUDA-event interval, with and without per-launch events in between --
shows whether consecutive launches overlap (programmatic dependent launch)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_19295_b200 import evaluator as ev, graphgen as gg  # noqa: E402
from paper_2310_19295_b200.graph import load_graph  # noqa: E402
from paper_2310_19295_b200.sharding import key_bits  # noqa: E402

g = load_graph(gg.config_doc("gpt2-small"))
B, K = 16384, 50
o = ev.generate_orders(g, 0, 0, B)
bufs = [o] + [o.clone() for _ in range(2)]
bits = key_bits(B)
for mode in ("back_to_back", "events_between"):
    for i in range(5):
        ev.evaluate_select_key(g, bufs[i % 3], 0, bits)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    inner = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    e0.record()
    for i in range(K):
        ev.evaluate_select_key(g, bufs[i % 3], 0, bits)
        if mode == "events_between":
            inner[i].record()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"mode": mode, "ms_per_launch": e0.elapsed_time(e1) / K}))
