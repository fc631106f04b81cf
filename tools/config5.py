"""BASELINE config 5: the candidate-order throughput sweep -- 1,048,576
counter-RNG Kahn orders on the GPT2-XL graph, sharded over N GPUs (contiguous
id ranges, one 16-byte all_gather of {peak, id}).  Prints one JSON line (rank
0) with the device time of generation and of evaluation+selection, max over
ranks, and the candidates/s of each.

  python tools/config5.py [--total 1048576] [--chunk 65536]
  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/config5.py
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--total", type=int, default=1 << 20)
    ap.add_argument("--chunk", type=int, default=1 << 18)
    ap.add_argument("--graph", default="gpt2-xl")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2310_19295_b200 import evaluator as ev
    from paper_2310_19295_b200 import graphgen as gg
    from paper_2310_19295_b200.graph import load_graph
    from paper_2310_19295_b200.sharding import NONE_PEAK, allgather_best, shard_range
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    g = load_graph(gg.config_doc(a.graph))
    lo, hi = shard_range(a.total, world, rank)
    # warm-up: graph handle, libroam and torch kernels of the loop (lazy module loading)
    best = torch.tensor([NONE_PEAK, -1], dtype=torch.int64, device=dev)
    for _ in range(2):
        wp, _, wv = ev.evaluate_orders(g, ev.generate_orders(g, 1, 0, 256))
        cb = ev.select_device(wp, wv)
        best = torch.where((cb[1] >= 0) & ((best[1] < 0) | (cb[0] < best[0])), cb, best)
        int(wv.sum().item())
    torch.cuda.synchronize()
    gen_ms = eval_ms = 0.0
    best = torch.tensor([NONE_PEAK, -1], dtype=torch.int64, device=dev)
    valid_total = 0
    events = []
    if world > 1:
        dist.barrier()
    for c0 in range(lo, hi, a.chunk):
        nb = min(a.chunk, hi - c0)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        orders = ev.generate_orders(g, 0, c0, nb, device=dev)
        e[1].record()
        peak, _, valid = ev.evaluate_orders(g, orders)
        cb = ev.select_device(peak, valid, id_base=c0)
        take = (cb[1] >= 0) & ((best[1] < 0) | (cb[0] < best[0]))
        best = torch.where(take, cb, best)
        e[2].record()
        events.append(e)
        valid_total = valid_total + valid.sum()   # on the device: no host sync per chunk
    torch.cuda.synchronize()
    for e in events:
        gen_ms += e[0].elapsed_time(e[1])
        eval_ms += e[1].elapsed_time(e[2])
    valid_total = int(valid_total)
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record()
    if world > 1:
        best = allgather_best(best)
    x1.record()
    torch.cuda.synchronize()
    xch_ms = x0.elapsed_time(x1)
    t = torch.tensor([gen_ms, eval_ms + xch_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    gen_max, eval_max = t.tolist()
    b = best.cpu().tolist()
    if rank == 0:
        n = len(g.ops)
        print(json.dumps({
            "config": f"BASELINE config 5: {a.total} Kahn candidate orders on {a.graph} ({n} ops)",
            "n_gpus": world, "chunk": a.chunk, "best": {"peak": b[0], "id": b[1]},
            "valid_on_rank0": valid_total,
            "generation_ms": gen_max, "generated_per_s": a.total / (gen_max / 1e3),
            "eval_select_exchange_ms": eval_max, "evaluated_per_s": a.total / (eval_max / 1e3),
            "eval_hbm_gbs": a.total * (4 * n + 16) / (eval_max / 1e3) / 1e9,
            "exchange_ms": xch_ms, "timing": "CUDA events, max over ranks"}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
