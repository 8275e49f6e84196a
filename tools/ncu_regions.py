#!/usr/bin/env python
"""Per-region stall breakdown of one kernel in an ncu report (regions = code
between consecutive BAR.SYNC instructions), plus the hottest basic blocks.

    python tools/ncu_regions.py <file.ncu-rep> [min_block_pct]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, data = rows[1], rows[2:]
    ia, isrc = h.index("Address"), h.index("Source")
    iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    f = lambda r, i: float(r[i] or 0)
    tot = sum(f(r, iss) for r in data) or 1.0
    bars = [k for k, r in enumerate(data) if "BAR.SYNC" in r[isrc]]
    prev = 0
    for k in bars + [len(data)]:
        seg = data[prev:k]
        if seg:
            s = sum(f(r, iss) for r in seg)
            if s / tot > 0.005:
                st = collections.Counter()
                for r in seg:
                    for c in stalls:
                        st[c[6:]] += f(r, h.index(c))
                print(f"region {seg[0][ia][-5:]}..{seg[-1][ia][-5:]}  {100 * s / tot:5.1f}% samples  "
                      f"{int(sum(f(r, iex) for r in seg))} warp-inst  top: "
                      + ", ".join(f"{n} {100 * v / tot:.1f}" for n, v in st.most_common(4)))
        prev = k
    blk, cur = [], []
    for k, r in enumerate(data):
        cur.append(k)
        if any(x in r[isrc] for x in ("BRA", "BSYNC", "EXIT", "BAR.SYNC")):
            blk.append(cur)
            cur = []
    blk.append(cur)
    print("hot blocks:")
    for b in blk:
        if not b:
            continue
        s = sum(f(data[k], iss) for k in b)
        if 100 * s / tot >= thr:
            ops = collections.Counter(data[k][isrc].split()[1 if data[k][isrc].strip().startswith("@") else 0]
                                      for k in b)
            print(f"  {data[b[0]][ia][-5:]} n={len(b):4d} {100 * s / tot:5.1f}%  ex={int(max(f(data[k], iex) for k in b))}"
                  f"  {dict(ops.most_common(5))}")


if __name__ == "__main__":
    main()
