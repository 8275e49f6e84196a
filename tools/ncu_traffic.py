#!/usr/bin/env python
"""Per-launch DRAM traffic of the bench's kernels from an `ncu --set full`
capture of the bench command -> profiles/ncu_traffic.json (read by bench.py
for the roofline `traffic` field).

    python tools/ncu_traffic.py <capture.ncu-rep> [workload=C2]

Entries are keyed "<workload>:<kernel>" (bench.py looks up its own workload).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

KEYS = {"cg_solve": ("k_cg_persistent", "k_cg1_persistent"), "tet_map": ("k_tet_map_seg",), "edge_matvec": ("k_spmv",)}


def main():
    path = sys.argv[1]
    workload = sys.argv[2] if len(sys.argv) > 2 else "C2"
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    acc = collections.defaultdict(list)
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "")
        for key, pat in KEYS.items():
            if any(p_ in name for p_ in pat):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                b = 0.0
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    u = units[h.index(m)]
                    b += float(d[m].replace(",", "")) * scale.get(u, 1)
                extra = {}
                for m, k in (("lts__t_sector_hit_rate.pct", "l2_hit_rate_pct"),
                             ("lts__t_sectors_op_red.sum", "l2_red_sectors"),
                             ("lts__t_sectors_op_atom.sum", "l2_atom_sectors"),
                             ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
                             ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_inst_pct")):
                    if m in d and d[m] not in ("", "n/a"):
                        try:
                            extra[k] = float(d[m].replace(",", ""))
                        except ValueError:
                            pass
                acc[key].append((b, name, float(d["gpu__time_duration.sum"].replace(",", "")), extra))
    res = {}
    for key, v in acc.items():
        if key == "edge_matvec":
            v = [x for x in v if "k_cg" not in x[1]]
            if not v:
                continue
        res[f"{workload}:{key}"] = {"workload": workload, "dram_bytes_per_launch": sum(x[0] for x in v) / len(v),
                    "launches_captured": len(v), "ncu_kernel": v[0][1][:100], "capture": os.path.basename(path),
                    "ncu_duration_each": [x[2] for x in v],
                    **{k: sum(x[3].get(k, 0.0) for x in v) / len(v) for k in v[0][3]},
                    "note": "ncu --set full --clock-control none (replayed, cold cache per pass)"}
    dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    old = {}
    if os.path.exists(dst):
        old = json.load(open(dst))
    old.update(res)
    json.dump(old, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
