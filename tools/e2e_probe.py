"""Host-staged evaluate_and_select timing vs a plain pinned H2D copy of the
same rows (GPT-2 small, 16,384 uint16 rows), for choosing the staging chunk.
Run with ROAM_STAGE_CHUNK_KB set to compare chunk sizes."""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2310_19295_b200 import evaluator as ev
    from paper_2310_19295_b200 import graphgen as gg
    from paper_2310_19295_b200.graph import load_graph
    g = load_graph(gg.config_doc("gpt2-small"))
    B = 16384
    orders = ev.generate_orders(g, 0, 0, B)
    host = torch.empty(orders.shape, dtype=torch.uint16, pin_memory=True)
    host.copy_(orders.to(torch.uint16).cpu())
    hn = host.numpy()
    for _ in range(3):
        ev.evaluate_and_select(g, hn)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        ev.evaluate_and_select(g, hn)
        ts.append(time.perf_counter() - t0)
    dst = torch.empty(host.shape, dtype=host.dtype, device="cuda")
    dst.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    cs = []
    for _ in range(10):
        t0 = time.perf_counter()
        dst.copy_(host, non_blocking=True)
        torch.cuda.synchronize()
        cs.append(time.perf_counter() - t0)
    small = hn[:64]
    for _ in range(3):
        ev.evaluate_and_select(g, small)
    tsm = []
    for _ in range(20):
        t0 = time.perf_counter()
        ev.evaluate_and_select(g, small)
        tsm.append(time.perf_counter() - t0)
    print(json.dumps({"fixed_ms_64rows": sorted(tsm)[10] * 1e3}))
    print(json.dumps({"chunk_kb": os.environ.get("ROAM_STAGE_CHUNK_KB", "default"),
                      "e2e_ms_median": sorted(ts)[5] * 1e3, "e2e_ms_min": min(ts) * 1e3,
                      "copy_ms_median": sorted(cs)[5] * 1e3, "copy_ms_min": min(cs) * 1e3}), flush=True)


if __name__ == "__main__":
    main()
