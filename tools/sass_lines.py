#!/usr/bin/env python
"""Warp-stall samples of one kernel per source line, from an ncu SASS source page.

  ncu -i rep --page source --csv --print-source sass > k.csv        (on the GPU box)
  python tools/sass_lines.py k.csv paper_1603_08390_b200/lib/obj/genie_query.o \
      _ZN5genie6k_scanILi4EEEvNS_11BatchParamsEj [top]

The .o is disassembled here with `nvdisasm -g` (the build uses -lineinfo), SASS
offsets are matched to the CSV's addresses relative to the kernel's first
instruction, and samples / executed instructions are summed per innermost
source line (inlined code is charged to the line it was written on).
"""
from __future__ import annotations

import collections
import csv
import gzip
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def line_map(obj: str, fn: str) -> dict[int, tuple[str, int]]:
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=d, check=True,
                       capture_output=True)
        cub = next(Path(d).glob("*.cubin"))
        txt = subprocess.run(["nvdisasm", "-g", str(cub)], capture_output=True, text=True).stdout
    out, cur, inside = {}, None, False
    for ln in txt.splitlines():
        if ln.startswith(".text."):
            inside = ln[len(".text."):].rstrip(":") == fn
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (Path(m.group(1)).name, int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            out[int(m.group(1), 16)] = cur
    return out


def main() -> None:
    path, obj, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt") as f:
        rows = list(csv.reader(f))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    cols = rows[hdr]
    data = [r for r in rows[hdr + 1:] if r and r[0].startswith("0x")]
    base = int(data[0][0], 16)
    lm = line_map(obj, fn)
    ci = {c: i for i, c in enumerate(cols)}
    stall_cols = [c for c in cols if c.startswith("stall_")]
    per = collections.defaultdict(lambda: collections.Counter())
    total = 0
    for r in data:
        off = int(r[0], 16) - base
        key = lm.get(off, ("?", 0))
        s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
        total += s
        c = per[key]
        c["samples"] += s
        c["inst"] += int(r[ci["Instructions Executed"]] or 0)
        for sc in stall_cols:
            v = r[ci[sc]]
            if v and v != "-":
                c[sc] += int(float(v))
    src = {}
    for (fname, _l) in per:
        p = Path(__file__).resolve().parent.parent / "paper_1603_08390_b200" / "csrc" / fname
        if p.exists() and fname not in src:
            src[fname] = p.read_text().splitlines()
    print(f"total samples {total}")
    for key, c in sorted(per.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        fname, ln = key
        text = src.get(fname, [])[ln - 1].strip()[:70] if fname in src and 0 < ln <= len(src[fname]) else ""
        stalls = sorted(((v, k[6:]) for k, v in c.items() if k.startswith("stall_") and v), reverse=True)[:3]
        st = " ".join(f"{k}={v}" for v, k in stalls)
        print(f"{100 * c['samples'] / max(total, 1):5.1f}% {fname}:{ln:<5} inst={c['inst']:>9}  {st:<48} | {text}")


if __name__ == "__main__":
    main()
