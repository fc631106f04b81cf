"""A/B timing of the K1 evaluator variants (1 generic, 4 v4, 5 v5) on the
config graphs: device-resident counter-RNG candidates, CUDA events on the
launching stream, L2 flushed between launches.  Prints one JSON line per
(graph, variant) with ms per launch and GB/s of algorithmic traffic."""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2310_19295_b200 import evaluator as ev
    from paper_2310_19295_b200 import graphgen as gg
    from paper_2310_19295_b200.graph import load_graph
    graphs = sys.argv[1:] or ["layered", "gpt2-small", "bert-large", "gpt2-xl"]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for name in graphs:
        g = load_graph(gg.config_doc(name))
        n = len(g.ops)
        B = 16384 if n < 4000 else 8192
        orders = ev.generate_orders(g, 0, 0, B)
        ref = None
        for variant in (1, 4, 5):
            ev.set_k1_variant(variant)
            out = ev.evaluate_orders(g, orders)
            torch.cuda.synchronize()
            got = [x.cpu() for x in out]
            if ref is None:
                ref = got
            same = all(torch.equal(a, b) for a, b in zip(got, ref))
            ts = []
            for _ in range(10):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ev.evaluate_orders(g, orders)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[len(ts) // 2]
            print(json.dumps({"graph": name, "n": n, "B": B, "variant": variant, "ms": ms,
                              "gbs": B * (4 * n + 16) / ms / 1e6, "same_as_v1": same}), flush=True)
        ev.set_k1_variant(0)
        ev.generate_orders(g, 1, 0, 1024)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ev.generate_orders(g, 2, 0, B)
        e1.record()
        torch.cuda.synchronize()
        gms = e0.elapsed_time(e1)
        print(json.dumps({"graph": name, "n": n, "B": B, "generator_ms": gms,
                          "generated_per_s": B / gms * 1e3}), flush=True)


if __name__ == "__main__":
    main()
