#!/usr/bin/env python
"""ncu counters of k_scan, stamped with the kernel-source digest, for bench.py's
roofline block (profiles/scan_counters.json).

  on the GPU box:  python tools/scan_counters.py capture tweets [minhash ...]
                   (ncu --set full --clock-control none on the 4th k_scan launch of
                    `bench.py --workload W`, reports under gpurun_out/counters/)
  here:            python tools/scan_counters.py ingest gpurun_out/counters/*.ncu-rep

bench.py uses an entry only if its `source_sha` equals the digest of the
current csrc/ sources (kernel_source_sha), so a stale capture is reported as
stale instead of being attributed to a different kernel.
"""
from __future__ import annotations

import csv
import hashlib
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "profiles" / "scan_counters.json"

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg",
    "sm__cycles_active.avg",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_sectors_op_atom.sum",
    "lts__t_sectors_op_red.sum",
    "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "smsp__inst_executed_op_shared_atom.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "device__attribute_multiprocessor_count",
]


def kernel_source_sha() -> str:
    """Digest of everything that shapes the device code (csrc + the C header)."""
    h = hashlib.sha256()
    csrc = ROOT / "paper_1603_08390_b200" / "csrc"
    files = sorted(list(csrc.glob("*.cu")) + list(csrc.glob("*.cuh")) + [csrc / "Makefile",
                                                                         ROOT / "include" / "genie" / "genie.h"])
    for f in files:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()[:16]


def capture(workloads):
    outdir = ROOT / "gpurun_out" / "counters"
    outdir.mkdir(parents=True, exist_ok=True)
    for w in workloads:
        rep = outdir / f"scan_{w}"
        # the batch's width class: W = 4 (tweets, adult) or 8 (sift, ocr, minhash); the other
        # classes' k_scan launches exit at once
        wcls = 4 if w in ("tweets", "adult") else 8
        cmd = ["ncu", "--set", "full", "--metrics", ",".join(METRICS), "--clock-control", "none",
               "--import-source", "on", "--kernel-name-base", "demangled", "-k", f"regex:k_scan<\\(int\\){wcls},",
               "--launch-skip", "3", "--launch-count", "1",
               "-f", "-o", str(rep), sys.executable, str(ROOT / "bench.py"), "--workload", w, "--steps", "1",
               "--warmup", "3", "--no-cpu-baseline"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        (outdir / f"scan_{w}.log").write_text(r.stdout[-20000:] + "\n---\n" + r.stderr[-20000:])
        print(w, "rc", r.returncode, flush=True)
    (outdir / "source_sha.txt").write_text(kernel_source_sha() + "\n")


def read_rep(rep: Path) -> dict:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def num(d, k):
    v, u = d[k]
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}.get(u, 1)
    return x * scale


def ingest(reps):
    res = json.loads(OUT.read_text()) if OUT.exists() else {}
    sha_file = ROOT / "gpurun_out" / "counters" / "source_sha.txt"
    src_sha = sha_file.read_text().strip() if sha_file.exists() else kernel_source_sha()
    for rep in reps:
        rep = Path(rep)
        w = rep.stem.replace("scan_", "")
        d = read_rep(rep)
        sms = num(d, "device__attribute_multiprocessor_count")
        cyc = num(d, "sm__cycles_elapsed.avg")
        inst = num(d, "smsp__inst_executed.sum")
        e = {
            "workload": w, "n_gpus": 1, "kernel": "k_scan", "source_sha": src_sha,
            "capture": "ncu --set full --clock-control none, 4th k_scan launch of bench.py (cold caches)",
            "ncu_duration_ms": round(num(d, "gpu__time_duration.sum") * 1e3, 4),
            "dram_bytes_per_launch": int(num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum")),
            "dram_read": int(num(d, "dram__bytes_read.sum")), "dram_write": int(num(d, "dram__bytes_write.sum")),
            "warp_inst_per_launch": int(inst),
            "issue_frac_under_ncu": round(inst / (cyc * 4 * sms), 4),
            "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
            "ipc_per_sm": float(d["sm__inst_executed.avg.per_cycle_active"][0]),
            "occupancy_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"][0]),
            "l2_atom_sectors": int(num(d, "lts__t_sectors_op_atom.sum")),
            "l2_red_sectors": int(num(d, "lts__t_sectors_op_red.sum")),
            "l2_hit_pct": float(d["lts__t_sector_hit_rate.pct"][0]),
            "l2_throughput_pct": float(d["lts__throughput.avg.pct_of_peak_sustained_elapsed"][0]),
            "l2_to_l1_bytes": int(num(d, "l1tex__m_xbar2l1tex_read_bytes.sum")),
            "smem_atom_wavefronts": int(num(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum")),
            "smem_atom_warp_inst": int(num(d, "smsp__inst_executed_op_shared_atom.sum")),
            "dram_pct_of_peak": float(d["dram__throughput.avg.pct_of_peak_sustained_elapsed"][0]),
            "registers": int(num(d, "launch__registers_per_thread")),
        }
        res[w] = e
        print(json.dumps(e))
    OUT.write_text(json.dumps(res, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "capture":
        capture(sys.argv[2:] or ["tweets"])
    elif sys.argv[1] == "ingest":
        ingest(sys.argv[2:])
    elif sys.argv[1] == "sha":
        print(kernel_source_sha())
