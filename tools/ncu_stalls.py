#!/usr/bin/env python
"""Top warp-stall reasons (pc-sampling counts) of every kernel in an ncu report."""
import csv
import subprocess
import sys

for path in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    for row in r[2:]:
        d = dict(zip(h, row))
        st = []
        for k in h:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(d[k].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1.0
        print(path, d.get("Kernel Name", "")[:60])
        for v, k in sorted(st, reverse=True)[:8]:
            print(f"   {k:24s} {100 * v / tot:5.1f}%")
