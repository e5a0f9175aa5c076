#!/usr/bin/env python
"""Benchmark of the GENIE match-count hot path on B200 (BASELINE.json metric).

Default line (N=1): C2 Tweets-shaped bag-of-words match count -- 7M docs,
vocab 1M, 10 distinct Zipf(1) words per doc, 1024 fresh-document queries,
top-k = 100 (BASELINE.json configs[1], the config the north star targets).
--workload {adult,sift,minhash,ocr} measures the other configs the same way.

A "step" is one full query batch through the hot path: (LSH / minHash encode
of the query batch for C3-C5) -> lookup -> scan + c-PQ + tile select -> merge
(+ NCCL all-gather and device merge for N > 1).

value : queries/s with the index and the query batch resident in HBM
        (device API, CUDA events around each step on the launching stream,
        256 MiB L2 flush between steps, untimed)
e2e   : queries/s through the public API with host (pinned) buffers: the
        C-ABI call genie_query_batch (plus genie_lsh_encode for C3-C5); H2D of
        the queries and D2H of the results are inside the timed region.

--impl reference times the reference's CPU implementation of the path on
the box's host cores: the unmodified mcx engine (oracle/_ref) for C1/C2, the
plain-C port of it (oracle/) for C3-C5, whose reference index build
(~10^9 (keyword, id) pairs) does not fit a bench run.

Launch: python bench.py [--gpus N --steps K --warmup W]; for N > 1 under
torch.distributed.run (one process per GPU; object-id shards + one NCCL
all-gather of per-shard top-k, merged on the device).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "queries/sec (top-k=100 match-count)"
UNIT = "queries/s"
WORKLOADS = {
    "tweets": "C2 tweets-shaped bag-of-words: 7M docs, vocab 1M, 10 distinct Zipf(1) words/doc, "
              "1024 fresh-doc queries, k=100",
    "adult": "C1 adult-shaped relational range match: 48842 x 14 attrs (+-50 windows), 1024 queries, k=100",
    "sift": "C3 SIFT-shaped 128-d E2LSH: 4M points, p-stable m=237 (w=4, 67 buckets), 1024 queries, k=100",
    "minhash": "C4 document minHash Jaccard: 2M sets (32-256 u64), 128 functions, D=8192, 4096 queries, k=100",
    "ocr": "C5 OCR-shaped kernel-space LSH: 1M x 784-d, random binning m=237, D=8192, 2048 queries, k=1 (1-NN)",
}
QUERIES = {"tweets": 1024, "adult": 1024, "sift": 1024, "minhash": 4096, "ocr": 2048}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="genie", choices=["genie", "reference"])
    ap.add_argument("--workload", default="tweets", choices=list(WORKLOADS))
    ap.add_argument("--n", type=int, default=None, help="override object count (debug only)")
    ap.add_argument("--queries", type=int, default=None)
    ap.add_argument("--selector", type=int, default=0, help="0 cpq, 1 bucket/histogram ablation")
    ap.add_argument("--tile-bytes", type=int, default=0)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--span-chunk", type=int, default=None, help="postings per warp work unit (result-invariant)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the kernels one by one (no CUDA graph)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 exchange: NCCL over NVLink (default) or gloo through host memory (plumbing tests)")
    ap.add_argument("--ref-sample", type=int, default=0, help="queries per reference step (0: auto)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML
    polled every ~2 ms from a thread (a C2 timed region is only ~25 ms long);
    nvidia-smi -lms 50 when NVML is unavailable."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, reasons bitmask)
        self.max_mhz = None
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            idx = self.gpu
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis and vis.split(",")[0].strip().isdigit():
                idx = int(vis.split(",")[self.gpu].strip())
            self.h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.nvml = nv
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        nv = self.nvml
        while not self.stop.is_set():
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)),
                                     int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml:
            self.t.join(timeout=2)
            if not self.samples:  # region shorter than one poll: take one now
                self.stop.clear()
                try:
                    nv = self.nvml
                    self.samples.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)),
                                         int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))))
                except Exception:
                    pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        if self.nvml:
            bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4}
            for mhz, r in self.samples:
                sm.append(mhz)
                for nm, b in bits.items():
                    if r & b:
                        reasons.add(nm)
            mx = self.max_mhz or 0.0
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml (2 ms poll)" if self.nvml else "nvidia-smi -lms 50"}


# --------------------------------------------------------------- workloads

class Workload:
    """One BASELINE config: the host data, this rank's device index and the
    device-resident query batch.  `encode()` re-encodes the device query
    points into the batch's items (C3-C5) and is part of every step."""

    lsh = None  # engine.Encoder for C3-C5

    def __init__(self, args, rank, world, dev, local):
        import torch

        from paper_1603_08390_b200 import DeviceIndex, engine as E, synth

        self.name = args.workload
        self.torch = torch
        self.dev = dev
        Q = args.queries or QUERIES[self.name]
        t0 = time.perf_counter()
        self.qpoints = self.qsets = None
        self.encode_index = None
        if self.name in ("tweets", "adult"):
            ds = (synth.tweets(n=args.n or 7_000_000, vocab=1_000_000, words=10, queries=Q, k=100)
                  if self.name == "tweets" else synth.adult(n=args.n or 48842, queries=Q, k=100))
            self.gen_s = time.perf_counter() - t0
            self.csr, self.batch = ds.csr, ds.queries
            self.n = self.csr.n
            t0 = time.perf_counter()
            if world > 1:
                lo, hi = self.n * rank // world, self.n * (rank + 1) // world
                self.ix = DeviceIndex.shard(self.csr, lo, hi, device=local)
            else:
                self.ix = DeviceIndex.from_csr(self.csr, device=local)
            self.build_s = time.perf_counter() - t0
            self.k = 100
            self.m = None
        else:
            if self.name == "sift":
                ds = synth.sift(n=args.n or 4_000_000, dims=128, queries=Q)
                cfg = E.lsh_config(E.PSTABLE, 237, 128, 3, w=4.0)
                domain, self.k = 67, 100
            elif self.name == "ocr":
                ds = synth.ocr(n=args.n or 1_000_000, dims=784, queries=Q)
                sigma = E.kernel_width_heuristic(ds.points[:10_000])
                cfg = E.lsh_config(E.RBH, 237, 784, 7, sigma=sigma, rehash_domain=8192)
                domain, self.k = 8192, 1
                self.sigma = sigma
            else:
                ds = synth.sets(n=args.n or 2_000_000, queries=Q)
                cfg = E.lsh_config(E.MINHASH, 128, 0, 5, rehash_domain=8192)
                domain, self.k = 8192, 100
            self.gen_s = time.perf_counter() - t0
            self.ds = ds
            self.m = cfg.m
            self.lsh = E.Encoder(cfg, local)
            t0 = time.perf_counter()
            n_all = ds.points.shape[0] if ds.points is not None else ds.set_off.shape[0] - 1
            lo, hi = n_all * rank // world, n_all * (rank + 1) // world
            self.n = n_all
            tok = torch.zeros((hi - lo, self.m), dtype=torch.int32, device=dev)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if self.name != "minhash":
                d_pts = torch.from_numpy(ds.points[lo:hi]).to(dev)
            else:
                off = ds.set_off[lo:hi + 1]
                d_off = torch.from_numpy((off - off[0]).astype(np.int64)).to(dev)
                d_el = torch.from_numpy(ds.elems[off[0]:off[-1]].view(np.int64)).to(dev)
            torch.cuda.synchronize(dev)
            ev0.record()  # the index-side transform alone (inputs resident)
            if self.name == "minhash":
                self.lsh.encode_sets_device(d_off, d_el, tok)
                del d_off, d_el
            else:
                self.lsh.encode_device(d_pts, tok)
                del d_pts
            ev1.record()
            torch.cuda.synchronize(dev)
            self.encode_index = {"points": hi - lo, "ms": round(ev0.elapsed_time(ev1), 3)}
            self.ix = DeviceIndex.from_tokens_device(tok.data_ptr(), hi - lo, self.m, domain, device=local,
                                                     id_offset=lo)
            del tok
            self.build_s = time.perf_counter() - t0
            # query batch skeleton: items (i, token_i) for every function i
            qtok = self.lsh.encode_sets(ds.query_set_off, ds.query_elems) if self.name == "minhash" else \
                self.lsh.encode(ds.query_points)
            self.batch = E.point_queries(qtok, self.k)
            if self.name == "minhash":
                self.qsets = (torch.from_numpy(ds.query_set_off.astype(np.int64)).to(dev),
                              torch.from_numpy(ds.query_elems.view(np.int64)).to(dev))
            else:
                self.qpoints = torch.from_numpy(ds.query_points).to(dev)
        qb = self.batch
        self.Q = len(qb)
        self.stride = max(1, min(int(qb.max_k), self.ix.num_objects or 1))
        self.d = {
            "qid": torch.from_numpy(qb.qid.astype(np.int32)).to(dev),
            "k": torch.from_numpy(qb.k.astype(np.int32)).to(dev),
            "item_off": torch.from_numpy(qb.item_off.astype(np.int64)).to(dev),
            "dim": torch.from_numpy(qb.dim.astype(np.int16)).to(dev),
            "lo": torch.from_numpy(qb.lo.astype(np.int32)).to(dev),
            "hi": torch.from_numpy(qb.hi.astype(np.int32)).to(dev),
            "out": torch.zeros((self.Q, self.stride, 2), dtype=torch.int32, device=dev),
            "out_len": torch.zeros(self.Q, dtype=torch.int32, device=dev),
            "out_thr": torch.zeros(self.Q, dtype=torch.int32, device=dev),
            "max_k": int(qb.max_k), "total_items": qb.num_items, "stride": self.stride,
        }
        if self.m:
            self.qtok = torch.zeros((self.Q, self.m), dtype=torch.int32, device=dev)

    def encode(self, stream_ptr):
        """Query-side transform on the device (part of each C3-C5 step)."""
        if not self.m:
            return 0
        if self.qsets is not None:
            self.lsh.encode_sets_device(self.qsets[0], self.qsets[1], self.qtok, stream=stream_ptr)
        else:
            self.lsh.encode_device(self.qpoints, self.qtok, stream=stream_ptr)
        flat = self.qtok.view(-1)
        self.d["lo"].copy_(flat)
        self.d["hi"].copy_(flat)
        return 1

    def cpu_csr(self):
        if self.m is None:
            return self.csr
        return self.ix.export()  # the device CSR (equal to the host build, tests/test_gpu_lsh.py)


# --------------------------------------------------------------- reference

def reference_qps(w: Workload, sample: int, steps: int, warmup: int, budget_s: float = 0.0):
    """The reference CPU engine on the box's cores over `sample` queries of
    the same index per step (the whole batch for C1/C2): mcx::execute_batch
    (Selector::cpq, ExecMode::parallel, workers = hardware threads;
    oracle/_ref) for C1/C2, the plain-C port (oracle/, all threads) for C3-C5.
    Returns (qps per timed step, cores, kind, build seconds, StageTimings per
    timed step or None)."""
    from oracle.pyoracle import Oracle, RefLib, threads

    csr = w.cpu_csr()
    t0 = time.perf_counter()
    stages = []
    if w.m is None:
        ref = RefLib()
        rix = ref.index(csr)
        cores, kind = ref.hardware_threads(), "reference"

        def run(b):
            rc, r = rix.execute(b, selector=0, sequential=False, workers=0)
            if rc:
                raise RuntimeError(r)
            return r.timings
    else:
        o = Oracle()
        oix = o.index(csr)
        cores, kind = threads(), "port"

        def run(b):
            oix.execute(b, nthreads=cores)
            return None
    build_s = time.perf_counter() - t0
    per_step = []
    Q = len(w.batch)
    sample = min(sample, Q)
    # budget_s > 0: the whole batch stays the step, but the timed steps are
    # capped so the run fits the budget (a C2 batch is ~7 s on 16 threads)
    t_start = time.perf_counter()
    for s in range(warmup + steps):
        a = (s * sample) % max(1, Q - sample + 1)
        b = w.batch.slice(a, a + sample)
        t = time.perf_counter()
        tm = run(b)
        dt = time.perf_counter() - t
        if s >= warmup:
            per_step.append(sample / dt)
            stages.append(tm)
        if budget_s and len(per_step) >= 3 and time.perf_counter() - t_start > budget_s:
            break
    return per_step, cores, kind, build_s, (stages if stages and stages[0] else None)


def stage_summary(stages):
    """Median StageTimings (engine.hpp:44-50) of the timed reference runs, ms."""
    if not stages:
        return None
    return {k.replace("_ns", "_ms"): round(float(np.median([s[k] for s in stages])) / 1e6, 2)
            for k in ("lookup_ns", "match_ns", "select_ns", "total_ns")}


def default_sample(name: str) -> int:
    # C1/C2: the whole batch; C3-C5: a bounded prefix
    return {"tweets": 1024, "adult": 1024, "sift": 16, "minhash": 512, "ocr": 16}[name]


def run_reference_arm(args):
    import torch

    rank, local, world = dist_env()
    if rank != 0:
        return 0
    dev = torch.device("cuda", local) if torch.cuda.is_available() else None
    if args.workload in ("tweets", "adult"):
        # no GPU involvement at all: generate the inputs on the host
        class _W:  # minimal stand-in with the fields reference_qps uses
            pass
        from paper_1603_08390_b200 import synth
        Q = args.queries or QUERIES[args.workload]
        ds = (synth.tweets(n=args.n or 7_000_000, vocab=1_000_000, words=10, queries=Q, k=100)
              if args.workload == "tweets" else synth.adult(n=args.n or 48842, queries=Q, k=100))
        w = _W()
        w.m, w.csr, w.batch = None, ds.csr, ds.queries
        w.cpu_csr = lambda: ds.csr
    else:
        w = Workload(args, 0, 1, dev, local)  # tokens via the GPU encoder (inputs only)
    sample = min(args.ref_sample or default_sample(args.workload), len(w.batch))
    # at most ~2 minutes of timed CPU work: warm-up capped at 1 step, timed steps
    # stop after the budget once 3 have run (the line reports the steps run)
    qps, cores, kind, build_s, stages = reference_qps(w, sample, args.steps, min(args.warmup, 1), budget_s=120.0)
    value = float(len(qps) * sample / np.sum([sample / v for v in qps]))  # queries / total time
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(qps), "warmup": min(args.warmup, 1), "ms_per_step": round(1000.0 * sample / value, 3),
        "steps_requested": args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded generator, SURVEY.md 8d)",
        "config": {"workload": WORKLOADS[args.workload], "queries_per_step": sample,
                   "same_batch_as_genie_arm": sample == len(w.batch), "stage_ms_median": stage_summary(stages),
                   "engine": ("mcx::execute_batch Selector::cpq ExecMode::parallel (unmodified reference headers)"
                              if kind == "reference" else "plain-C port of mcx::execute_batch (oracle/)")},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": (f"the whole {sample}-query batch per step" if sample == len(w.batch) else
                                    f"{sample} queries per step of the {len(w.batch)}-query batch")
                                   + f"; CPU index build {build_s:.1f}s untimed"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- roofline

def scan_roofline(workload, world, postings, scan_ms, clocks, sms):
    """Roofline of k_scan, the dominant kernel.

    The bound is the one ncu shows (profiles/scan_counters.json, captured for
    the CURRENT kernel sources -- an entry whose source_sha differs is stale
    and not used): SM instruction issue.  achieved = warp instructions per
    launch (ncu smsp__inst_executed.sum) / the live k_scan time (CUDA events
    on the launching stream); peak = SMs x 4 schedulers x 1 warp-inst/cycle x
    the SM clock sampled during the timed region.  HBM is reported beside it:
    DRAM bytes per launch (ncu) / live time vs the measured copy bandwidth,
    and the algorithmic bytes (4 B x sum_q P_q) as a diagnostic --
    the latter exceed what the kernel moves because dense lists are read as
    bitmaps and hot lists stay in L2 across the tile-major sweep."""
    from tools.scan_counters import kernel_source_sha

    peaks_path = ROOT / "MEASURED_PEAKS.json"
    if peaks_path.exists():
        hbm_peak = float(json.loads(peaks_path.read_text())["hbm_gbs"])
        hbm_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        hbm_peak, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    alg_bytes = 4 * postings
    entry, stale = None, None
    cpath = ROOT / "profiles" / "scan_counters.json"
    if cpath.exists():
        e = json.loads(cpath.read_text()).get(workload)
        if e and e.get("n_gpus", 1) == world:
            if e.get("source_sha") == kernel_source_sha():
                entry = e
            else:
                stale = e.get("source_sha")
    mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    issue_peak = sms * 4 * mhz * 1e6 / 1e9  # G warp-instructions / s
    out = {"bound": "issue", "unit": "Gwarp-inst/s", "peak": round(issue_peak, 1),
           "peak_source": f"{sms} SMs x 4 schedulers x 1 warp-inst/cycle x {mhz:.0f} MHz (sampled)",
           "kernel": "k_scan (fused posting scan + c-PQ gate/table + tile top-k)", "kernel_ms": round(scan_ms, 4),
           "achieved": None, "frac": None, "traffic": None}
    if entry:
        ach = entry["warp_inst_per_launch"] / (scan_ms / 1e3) / 1e9
        out.update({"achieved": round(ach, 1), "frac": round(ach / issue_peak, 4),
                    "traffic": entry["dram_bytes_per_launch"],
                    "warp_inst_per_launch": entry["warp_inst_per_launch"],
                    "counters": {k: entry[k] for k in ("source_sha", "ncu_duration_ms", "issue_active_pct",
                                                       "ipc_per_sm", "occupancy_pct", "l2_atom_sectors",
                                                       "l2_red_sectors", "smem_atom_wavefronts", "l2_hit_pct",
                                                       "l2_throughput_pct", "registers") if k in entry}})
    else:
        out["note"] = ("no ncu counters for these kernel sources" +
                       (f" (profiles/scan_counters.json entry is stale: {stale})" if stale else ""))
    dram_gbs = (entry["dram_bytes_per_launch"] / (scan_ms / 1e3) / 1e9) if entry else None
    out["hbm"] = {"peak": hbm_peak, "peak_source": hbm_src, "unit": "GB/s",
                  "dram_achieved": round(dram_gbs, 1) if dram_gbs else None,
                  "dram_frac": round(dram_gbs / hbm_peak, 4) if dram_gbs else None,
                  "algorithmic_bytes_per_launch": alg_bytes,
                  "algorithmic_gbs": round(alg_bytes / (scan_ms / 1e3) / 1e9, 1),
                  "note": "algorithmic = 4 B x sum_q P_q (SURVEY 8d); a diagnostic, not a roofline fraction"}
    return out


GOLDEN_NAME = {"adult": "c1", "tweets": "c2", "sift": "c3", "minhash": "c4", "ocr": "c5"}


def result_parity(args, w, Q, stride, out, out_len, out_thr):
    """hash_results (engine.hpp:141-153) of the last timed batch against the
    reference-pinned digest of the same config (tests/golden/full_configs.json),
    when the workload runs at its BASELINE size."""
    from paper_1603_08390_b200.engine import hash_results

    g = json.loads((ROOT / "tests" / "golden" / "full_configs.json").read_text()).get(GOLDEN_NAME[args.workload])
    if not g or args.n or args.queries:
        return {"checked": False, "why": "no golden digest for this size"}
    ent = out.cpu().numpy().view(np.uint32).reshape(Q, stride, 2)
    h = hash_results(w.batch.qid, out_thr.cpu().numpy().astype(np.uint32), out_len.cpu().numpy().astype(np.uint32),
                     ent[:, :, 0], ent[:, :, 1])
    return {"checked": True, "hash": f"{h:#018x}", "golden": g["hash"], "equal": f"{h:#018x}" == g["hash"],
            "golden_source": g["source"]}


def encode_roofline(workload, w):
    """The index-side LSH / minHash transform, timed on its own (CUDA events,
    inputs resident): SURVEY 8d bounds it by FP64 issue (p-stable: one DMUL +
    one DADD per (point, function, dim); RBH: DSUB + DMUL per coordinate, plus
    an exact DDIV near bucket boundaries and a mix64 fold) against the B200
    FP64 peak the Blackwell guide states (45 TFLOP/s).  minHash is INT64 only
    (one mix64 per (element, function)): reported as hashes/s."""
    e = dict(w.encode_index)
    n, m, dims = e["points"], w.m, (w.ds.points.shape[1] if w.ds.points is not None else 0)
    s = e["ms"] / 1e3
    if workload in ("sift", "ocr"):
        flops = 2.0 * n * m * dims
        e.update({"fp64_gflop": round(flops / 1e9, 1), "fp64_tflops": round(flops / s / 1e12, 2),
                  "fp64_peak_tflops": 45.0, "peak_source": "blackwell_cuda_programming.md (B200 FP64)",
                  "frac": round(flops / s / 45e12, 3), "points_per_s": round(n / s, 1)})
    else:
        elems = int(w.ds.set_off[-1]) if w.ds.set_off is not None else 0
        e.update({"mix64_hashes": elems * m, "ghash_per_s": round(elems * m / s / 1e9, 2), "sets_per_s": round(n / s, 1)})
    return e


# ------------------------------------------------------------------- genie

def main_genie(args):
    import torch
    import torch.distributed as dist

    from paper_1603_08390_b200 import config
    from paper_1603_08390_b200.engine import QueryBatch

    rank, local, world = dist_env()
    assert world == args.gpus or world == 1, "launch N>1 under torch.distributed.run"
    # ranks beyond the box's GPUs share devices (gloo plumbing tests on a 1-GPU box)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    gloo = args.dist_backend == "gloo"
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def all_gather(dst, src):
        """[world, ...] <- every rank's src: NCCL over NVLink, or through host memory for gloo."""
        if not gloo:
            dist.all_gather_into_tensor(dst, src)
            return
        parts = [torch.zeros_like(src, device="cpu") for _ in range(world)]
        dist.all_gather(parts, src.cpu())
        dst.copy_(torch.stack(parts))

    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], device="cpu" if gloo else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    # a dedicated stream: torch's default stream has handle 0, which the C ABI
    # reads as "the index's own stream"
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream

    w = Workload(args, rank, world, dev, local)
    ix, d, Q, stride = w.ix, w.d, w.Q, w.stride
    # the device-resident step replays the batch pipeline as one CUDA graph
    cfg = config(selector=args.selector, tile_bytes=args.tile_bytes, ctas_per_sm=args.ctas_per_sm,
                 span_chunk=args.span_chunk, stage_events=True, graph=not args.no_graph)
    if world > 1:
        gath = torch.zeros((world, Q, stride, 2), dtype=torch.int32, device=dev)
        gath_len = torch.zeros((world, Q), dtype=torch.int32, device=dev)
        fin = torch.zeros((Q, stride, 2), dtype=torch.int32, device=dev)
        fin_len = torch.zeros(Q, dtype=torch.int32, device=dev)
        fin_thr = torch.zeros(Q, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    launches_per_step = 0

    def step(check=False):
        """One batch; with check, the shard batch's status (workspace growth,
        errors) is read before the merge reuses the status block."""
        nonlocal launches_per_step
        launches_per_step = w.encode(sptr)
        launches_per_step += ix.query_device(d, cfg, stream=sptr)
        st = None
        if check:
            torch.cuda.synchronize(dev)
            st = ix.status()
            retry = float(bool(st.get("retry")))
            if world > 1:
                retry = max_over_ranks(retry)
            if retry:
                return {"retry": True}
        if world > 1:
            # all-gather the per-shard top-k (global ids), merge on the device
            all_gather(gath, d["out"])
            all_gather(gath_len, d["out_len"])
            # rank-major rows merged in place (list-major layout, no transpose)
            ix.merge_device(Q, world, gath, gath_len, stride, d["k"], stride, fin, fin_len, fin_thr, stream=sptr,
                            list_major=True)
            launches_per_step += 3
            if check:
                torch.cuda.synchronize(dev)
                ix.status()  # merge errors (duplicate ids) surface here
        return st

    def run_checked():
        for _ in range(3):
            st = step(check=True)
            if not st.get("retry"):
                return st
        raise RuntimeError("workspace did not converge")

    for _ in range(max(args.warmup, 3)):
        stats = run_checked()

    # ---- timed region (device): per-step CUDA events, L2 flushed between steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    scan_ms, look_ms, merge_ms = [], [], []
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            torch.cuda.synchronize(dev)
            sn = ix.stage_ns()
            scan_ms.append(sn["match_ns"] / 1e6)
            look_ms.append(sn["lookup_ns"] / 1e6)
            merge_ms.append(sn["merge_ns"] / 1e6)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    st = ix.status()
    if os.environ.get("GENIE_PHASE_REPORT"):  # instrumented library (tools/phase_timers.py)
        from tools.phase_timers import report
        print(report(ix, int(stats["work_items"])), file=sys.stderr)
    total_ms = float(np.sum(step_ms))
    if world > 1:
        total_ms = max_over_ranks(total_ms)
    parity = result_parity(args, w, Q, stride, *((fin, fin_len, fin_thr) if world > 1 else
                                                 (d["out"], d["out_len"], d["out_thr"])))
    ms_per_step = total_ms / args.steps
    value = Q * args.steps / (total_ms / 1000.0)

    # ---- e2e through the public C-ABI calls with host (pinned) buffers
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    hout = (pin(np.zeros((Q, stride, 2), np.uint32)), pin(np.zeros(Q, np.uint32)), pin(np.zeros(Q, np.uint32)))
    # the public host-buffer call; with pinned buffers it replays as one CUDA graph
    e2e_cfg = config(selector=args.selector, tile_bytes=args.tile_bytes, ctas_per_sm=args.ctas_per_sm,
                     span_chunk=args.span_chunk, graph=not args.no_graph)
    qb = w.batch
    hb = QueryBatch(pin(qb.qid), pin(qb.k), pin(qb.item_off), pin(qb.dim), pin(qb.lo), pin(qb.hi))

    if w.m:  # host query points / sets, pinned
        e2e_src = (dict(set_off=pin(w.ds.query_set_off.astype(np.uint64)), elems=pin(w.ds.query_elems.astype(np.uint64)))
                   if w.name == "minhash" else dict(points=pin(w.ds.query_points)))

    def e2e_step():
        if w.m:
            # LshEncoder::encode_query_point + execute_batch fused on the GPU
            # (genie_lsh_query_batch): the tokens never leave the device
            w.lsh.query(ix, w.k, cfg=e2e_cfg, stride=stride, out=hout, copy=False, **e2e_src)
            h2d, d2h = sum(a.nbytes for a in e2e_src.values()), 0
        else:
            h2d, d2h = hb.nbytes(), 0
            ix.query(hb, e2e_cfg, stride=stride, out=hout, copy=False)
        if world > 1:
            lists = torch.from_numpy(hout[0]).to(dev)
            lens = torch.from_numpy(hout[1].astype(np.int32)).to(dev)
            all_gather(gath, lists.view(torch.int32))
            all_gather(gath_len, lens)
            ix.merge_device(Q, world, gath, gath_len, stride, d["k"], stride, fin, fin_len, fin_thr, stream=sptr,
                            list_major=True)
            fin.cpu(), fin_len.cpu(), fin_thr.cpu()
        return h2d, d2h + hout[0].nbytes + hout[1].nbytes + hout[2].nbytes

    for _ in range(2):
        e2e_step()
    e2e_times = []
    for _ in range(max(3, args.steps)):  # as many steps as the device-resident timing
        flush.zero_()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        h2d_bytes, d2h_bytes = e2e_step()
        e2e_times.append(time.perf_counter() - t)
    e2e_s = float(np.mean(e2e_times))
    if world > 1:
        e2e_s = max_over_ranks(e2e_s)
    e2e_value = Q / e2e_s

    # ---- roofline of the dominant kernel (k_scan: fused scan + c-PQ + tile select)
    roof = scan_roofline(args.workload, world, int(stats["postings"]), float(np.mean(scan_ms)), clocks.summary(),
                         torch.cuda.get_device_properties(dev).multi_processor_count)
    postings = int(stats["postings"])

    # ---- CPU baseline (reference engine on the host cores; rank 0, N = 1):
    # the whole C1/C2 batch, median of 3 runs
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sample = min(args.ref_sample or default_sample(args.workload), Q)
            qps, cores, kind, build_ref_s, stages = reference_qps(w, sample, steps=3, warmup=0)
            cpu = {"value": round(float(np.median(qps)), 3), "unit": UNIT, "cores": cores, "kind": kind,
                   "sample": (f"the whole {Q}-query batch" if sample == Q else f"first {sample} of the {Q} queries")
                             + f", median of 3 runs on the same index ({cores} threads; CPU index build "
                               f"{build_ref_s:.1f}s untimed)",
                   "stage_ms_median": stage_summary(stages)}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded generator, SURVEY.md 8d)",
            "config": {"workload": WORKLOADS[args.workload], "n_objects": w.n, "queries": Q, "k": int(qb.max_k),
                       "selector": ["cpq", "bucket"][min(args.selector, 1)],
                       "parallelism": (f"object-id shards x{world} + {args.dist_backend.upper()} all-gather merge" if world > 1 else "single GPU"),
                       "l2": "flushed between timed steps (256 MiB write)",
                       "postings_per_query_mean": round(postings / Q, 1),
                       "generate_s": round(w.gen_s, 2), "index_build_s": round(w.build_s, 2)},
            "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d_bytes),
                    "d2h_bytes_per_step": int(d2h_bytes),
                    "path": ("genie_lsh_query_batch (C ABI: host points/sets -> device encode -> batch)" if w.m else
                     "genie_query_batch (C ABI)") + ", pinned host buffers"
                            + (" + all-gather + genie_merge_topk_device" if world > 1 else "")},
            "roofline": roof,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clocks.summary(),
            "stage_ms": {"step_mean": round(float(np.mean(step_ms)), 4), "scan_mean": round(float(np.mean(scan_ms)), 4),
                         "lookup_mean": round(float(np.mean(look_ms)), 4),
                         "merge_mean": round(float(np.mean(merge_ms)), 4)},
            "fallback_tiles": int(stats.get("fallback_tiles", 0)), "work_items": int(stats.get("work_items", 0)),
            "parity": parity,
        }
        if getattr(w, "sigma", None):
            line["config"]["sigma"] = round(w.sigma, 6)
        if w.encode_index:
            line["encode"] = encode_roofline(args.workload, w)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)
    return main_genie(args)


if __name__ == "__main__":
    sys.exit(main())
