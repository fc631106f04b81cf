"""Summarise ncu output brought back from gpurun into profiles/ (tracked).

  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.json
  python tools/ncu_summary.py full gpurun_out/k1_full.ncu-rep profiles/r01_k1_full.json \
      [--config gpt2-small --batch 16384]

`launches`: per-kernel launch count, total and average device time, and each
kernel's share of the captured device time (ncu's per-launch times are
cold-cache and serialised: compare shares, not absolutes).
`full`: the headline metrics of one `ncu --set full` capture (DRAM bytes,
duration, throughput, occupancy, stall breakdown, shared-memory wavefronts and
bank conflicts).  With --config/--batch it also records the per-launch DRAM
traffic in profiles/k1_ncu_summary.json, which bench.py reports as
roofline.traffic.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict
from pathlib import Path

KEYS = (
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__shared_mem_per_block",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
)
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}


def launches(src: str, dst: str) -> dict:
    rows = list(csv.reader(open(src)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    agg: dict[str, list] = defaultdict(lambda: [0, 0.0])
    for r in rows[i + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * SCALE.get(d.get("Metric Unit", "ns"), 1)
    total = sum(t for _, t in agg.values()) or 1.0
    out = {"source": Path(src).name, "note": "ncu --metrics gpu__time_duration.sum --clock-control none; "
           "cold-cache serialised launches: compare shares",
           "kernels": {k: {"launches": c, "total_us": t / 1e3, "avg_us": t / c / 1e3,
                           "share": t / total} for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])}}
    Path(dst).write_text(json.dumps(out, indent=1) + "\n")
    return out


def full(src: str, dst: str, config: str | None, batch: int | None) -> dict:
    raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        ent = {"kernel": d.get("Kernel Name", "").split("(")[0].replace("void ", "")}
        for k in KEYS:
            if k in d and d[k] != "":
                v = float(d[k].replace(",", ""))
                unit = u.get(k, "")
                if unit in SCALE:
                    v *= SCALE[unit]
                    k = k + (" [B]" if "byte" in unit.lower() or unit.endswith("B") else " [ns]")
                ent[k] = v
        kernels.append(ent)
    out = {"source": Path(src).name, "note": "ncu --set full --clock-control none --import-source on",
           "launches": kernels}
    Path(dst).write_text(json.dumps(out, indent=1) + "\n")
    if config and batch and kernels:
        k = kernels[-1]
        summ = Path(dst).parent / "k1_ncu_summary.json"
        s = json.loads(summ.read_text()) if summ.exists() else {}
        s[config] = {"batch": batch, "dram_bytes_read": int(k["dram__bytes_read.sum [B]"]),
                     "dram_bytes_write": int(k["dram__bytes_write.sum [B]"]),
                     "duration_ns": k["gpu__time_duration.sum [ns]"], "from": Path(dst).name}
        summ.write_text(json.dumps(s, indent=1) + "\n")
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "full"])
    ap.add_argument("src")
    ap.add_argument("dst")
    ap.add_argument("--config")
    ap.add_argument("--batch", type=int)
    a = ap.parse_args()
    Path(a.dst).parent.mkdir(parents=True, exist_ok=True)
    res = launches(a.src, a.dst) if a.mode == "launches" else full(a.src, a.dst, a.config, a.batch)
    print(json.dumps(res, indent=1)[:3000])
