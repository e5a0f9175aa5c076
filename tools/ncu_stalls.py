#!/usr/bin/env python
"""Source lines of one .ncu-rep ranked by warp-stall samples, with their top stall reasons."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = fname = None
rows = []
for line in out.splitlines():
    r = next(csv.reader(io.StringIO(line)))
    if r and r[0] in ("File Path", "File Name"):
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit() or r[2] != "-":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    if s:
        st = {k[6:]: int(v) for k, v in d.items()
              if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
        rows.append((s, fname, r[0], r[1].strip()[:70], sorted(st.items(), key=lambda x: -x[1])[:3]))
ts = sum(x[0] for x in rows) or 1
for s, f, l, src, st in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/ts:5.1f}% {f}:{l} {src} | " + " ".join(f"{k}={100*v/s:.0f}%" for k, v in st))
