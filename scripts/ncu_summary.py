#!/usr/bin/env python3
"""Summarise ncu reports / launch lists for profiles/ (run here, no GPU).

  python scripts/ncu_summary.py full  <report.ncu-rep> <out.json>
  python scripts/ncu_summary.py launches <launches.csv> <out.json>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sectors.sum", "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second", "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def unit_scale(val: str, unit: str) -> float:
    v = float(val.replace(",", ""))
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "usecond": 1e-6, "msecond": 1e-3,
             "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
             "nsecond": 1e-9, "second": 1.0, "byte": 1.0}.get(unit, 1.0)
    return v * scale


def full(rep: str, out: str) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, launches = rows[0], rows[1], rows[2:]
    res = []
    for r in launches:
        d = {"kernel": r[hdr.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                try:
                    d[k] = unit_scale(r[i], units[i])
                except ValueError:
                    d[k] = r[i]
        d["dram_bytes"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        res.append(d)
    summary = {"report": rep, "launches": res,
               "dram_bytes_per_launch_all_modes": [d["dram_bytes"] for d in res]}
    json.dump(summary, open(out, "w"), indent=1)
    for d in res:
        print(f"{d['kernel'][:60]:60s} t={d.get('gpu__time_duration.sum', 0)*1e3:8.3f} ms "
              f"dram={d['dram_bytes']/1e9:7.3f} GB l1pipe={d.get('l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed')} "
              f"l2={d.get('lts__throughput.avg.pct_of_peak_sustained_elapsed')}")


def launches(path: str, out: str) -> None:
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(unit_scale(r[vi], r[ui]))
    total = sum(sum(v) for v in agg.values())
    res = [{"kernel": k[:140], "launches": len(v), "total_ms": sum(v) * 1e3, "avg_us": sum(v) / len(v) * 1e6,
            "share": sum(v) / total} for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]
    json.dump({"source": path, "kernels": res}, open(out, "w"), indent=1)
    for d in res:
        print(f"{d['launches']:5d} {d['total_ms']:10.3f} ms {d['share']*100:5.1f}%  {d['kernel'][:90]}")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
