#!/usr/bin/env python
"""Summarise ncu captures for profiles/: per-kernel duration, DRAM bytes,
throughputs, occupancy, top stall reasons; and the launch-list CSV of a
`--metrics gpu__time_duration.sum` pass as per-kernel shares.

    python tools/ncu_summary.py rep  <file.ncu-rep> [...]      -> JSON lines
    python tools/ncu_summary.py launches <launches.csv>        -> JSON
"""
from __future__ import annotations

import collections
import csv
import json
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
       "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
       "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def _csv(args):
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def rep(path):
    r = _csv([path, "--page", "raw"])
    if len(r) < 3:
        return []
    h, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        k = {"kernel": d.get("Kernel Name", "")[:120], "capture": path}
        for m in RAW:
            if m in d:
                k[m] = f"{d[m]} {u.get(m, '')}".strip()
        res.append(k)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = ""
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        unit = d["Metric Unit"]
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values()) or 1.0
    return {"source": path, "unit": unit, "kernels": [
        {"kernel": k, "launches": v[0], "total": v[1], "avg": v[1] / v[0], "share": v[1] / tot}
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1])]}


if __name__ == "__main__":
    mode, *files = sys.argv[1:]
    if mode == "rep":
        for f in files:
            for k in rep(f):
                print(json.dumps(k))
    else:
        for f in files:
            print(json.dumps(launches(f), indent=1))
