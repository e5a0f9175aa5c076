#!/usr/bin/env python
"""Benchmark of the GENIE match-count hot path on B200 (BASELINE.json metric).

Workload (N=1 line): C2 Tweets-shaped bag-of-words match count -- 7M docs,
vocab 1M, 10 distinct Zipf(1) words per doc, 1024 fresh-document queries,
top-k = 100 (BASELINE.json configs[1], the config the north star targets).
A "step" is one full batch of 1024 queries through the hot path: lookup ->
scan + c-PQ + tile select -> merge (+ all-gather and merge for N > 1).

value : queries/s with the index and the query batch resident in HBM
        (device API, CUDA events around each step, L2 flushed between steps)
e2e   : queries/s through the public C-ABI call (genie_query_batch) with host
        (pinned) query buffers and host result buffers; H2D of the queries
        and D2H of the results are inside the timed region.

--impl reference times the reference CPU implementation (mcx built from the
unmodified headers, oracle/_ref) on the box's host cores on the same workload.

Launch: python bench.py [--gpus N --steps K --warmup W]; for N > 1 under
torch.distributed.run (one process per GPU; object-id shards + NCCL
all-gather of per-shard top-k, merged on the device).
"""
from __future__ import annotations

import argparse
import json
import math
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
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="genie", choices=["genie", "reference"])
    ap.add_argument("--workload", default="tweets", choices=list(WORKLOADS))
    ap.add_argument("--n", type=int, default=None, help="override object count (debug)")
    ap.add_argument("--queries", type=int, default=1024)
    ap.add_argument("--selector", type=int, default=0, help="0 cpq, 1 bucket/histogram ablation")
    ap.add_argument("--tile-bytes", type=int, default=0)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--span-chunk", type=int, default=None, help="postings per warp work unit (result-invariant)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=0, help="queries per reference step (0: auto)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def make_dataset(args):
    from paper_1603_08390_b200 import synth

    if args.workload == "tweets":
        n = args.n or 7_000_000
        return synth.tweets(n=n, vocab=1_000_000, words=10, queries=args.queries, k=100)
    return synth.adult(n=args.n or 48842, queries=args.queries, k=100)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- reference

def reference_qps(csr, queries, sample: int, steps: int, warmup: int):
    """The reference CPU engine (mcx::execute_batch, Selector::cpq, all host
    threads) on a bounded sample of the workload.  Returns (qps list, cores,
    build seconds)."""
    from oracle.pyoracle import RefLib

    ref = RefLib()
    t0 = time.perf_counter()
    rix = ref.index(csr)
    build_s = time.perf_counter() - t0
    cores = ref.hardware_threads()
    per_step = []
    for s in range(warmup + steps):
        a = (s * sample) % max(1, len(queries) - sample + 1)
        b = queries.slice(a, a + sample)
        t = time.perf_counter()
        rc, r = rix.execute(b, selector=0, sequential=False, workers=0)
        dt = time.perf_counter() - t
        if rc:
            raise RuntimeError(r)
        if s >= warmup:
            per_step.append(sample / dt)
    return per_step, cores, build_s


def run_reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    ds = make_dataset(args)
    sample = args.ref_sample or (64 if args.workload == "tweets" else 256)
    qps, cores, build_s = reference_qps(ds.csr, ds.queries, sample, args.steps, args.warmup)
    value = float(np.mean(qps))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1000.0 * sample / value, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded generator, SURVEY.md 8d)",
        "config": {"workload": WORKLOADS[args.workload], "queries_per_step": sample,
                   "engine": "mcx::execute_batch Selector::cpq ExecMode::parallel (unmodified reference headers)"},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{sample} queries per step of the {len(ds.queries)}-query batch; "
                                   f"index build {build_s:.1f}s untimed"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- genie

def main_genie(args):
    import torch
    import torch.distributed as dist

    from paper_1603_08390_b200 import DeviceIndex, config
    from paper_1603_08390_b200 import _native as N

    rank, local, world = dist_env()
    assert world == args.gpus or world == 1, "launch N>1 under torch.distributed.run"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    t0 = time.perf_counter()
    ds = make_dataset(args)
    gen_s = time.perf_counter() - t0
    csr, qb = ds.csr, ds.queries
    n, Q = csr.n, len(qb)
    t0 = time.perf_counter()
    if world > 1:
        lo, hi = n * rank // world, n * (rank + 1) // world
        ix = DeviceIndex.shard(csr, lo, hi, device=local)
    else:
        ix = DeviceIndex.from_csr(csr, device=local)
    build_s = time.perf_counter() - t0

    K = int(qb.max_k)
    stride = K
    cfg = config(selector=args.selector, tile_bytes=args.tile_bytes, ctas_per_sm=args.ctas_per_sm,
                 span_chunk=args.span_chunk, stage_events=True)
    # device-resident query batch
    d = {
        "qid": torch.from_numpy(qb.qid.astype(np.int32)).to(dev),
        "k": torch.from_numpy(qb.k.astype(np.int32)).to(dev),
        "item_off": torch.from_numpy(qb.item_off.astype(np.int64)).to(dev),
        "dim": torch.from_numpy(qb.dim.astype(np.int16)).to(dev),
        "lo": torch.from_numpy(qb.lo.astype(np.int32)).to(dev),
        "hi": torch.from_numpy(qb.hi.astype(np.int32)).to(dev),
        "out": torch.zeros((Q, stride, 2), dtype=torch.int32, device=dev),
        "out_len": torch.zeros(Q, dtype=torch.int32, device=dev),
        "out_thr": torch.zeros(Q, dtype=torch.int32, device=dev),
        "max_k": K, "total_items": qb.num_items, "stride": stride,
    }
    if world > 1:
        gath = torch.zeros((world, Q, stride, 2), dtype=torch.int32, device=dev)
        gath_len = torch.zeros((world, Q), dtype=torch.int32, device=dev)
        m_in = torch.zeros((Q, world, stride, 2), dtype=torch.int32, device=dev)
        m_len = torch.zeros((Q, world), dtype=torch.int32, device=dev)
        fin = torch.zeros((Q, stride, 2), dtype=torch.int32, device=dev)
        fin_len = torch.zeros(Q, dtype=torch.int32, device=dev)
        fin_thr = torch.zeros(Q, dtype=torch.int32, device=dev)

    # a dedicated stream: torch's default stream has handle 0, which the C ABI
    # reads as "the index's own stream"
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    launches_per_step = 0

    def step():
        nonlocal launches_per_step
        launches_per_step = ix.query_device(d, cfg, stream=sptr)
        if world > 1:
            # all-gather the per-shard top-k (global ids), merge on the device
            dist.all_gather_into_tensor(gath, d["out"])
            dist.all_gather_into_tensor(gath_len, d["out_len"])
            m_in.copy_(gath.permute(1, 0, 2, 3))
            m_len.copy_(gath_len.t())
            ix.merge_device(Q, world, m_in, m_len, stride, d["k"], stride, fin, fin_len, fin_thr, stream=sptr)
            launches_per_step += 3

    def run_checked():
        for _ in range(3):
            step()
            torch.cuda.synchronize(dev)
            st = ix.status()
            if not st.get("retry"):
                return st
        raise RuntimeError("workspace did not converge")

    for _ in range(max(args.warmup, 3)):
        st = run_checked()
    stats = st

    # ---- timed region (device): per-step CUDA events, L2 flushed between steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    scan_ms, step_ms, look_ms, merge_ms = [], [], [], []
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
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = Q * args.steps / (total_ms / 1000.0)

    # correctness spot-check of the timed output against the host API path
    # (cheap; the oracle parity lives in tests/)
    # ---- e2e through the public C-ABI call with host buffers
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    from paper_1603_08390_b200.engine import QueryBatch
    hb = QueryBatch(pin(qb.qid), pin(qb.k), pin(qb.item_off), pin(qb.dim), pin(qb.lo), pin(qb.hi))
    hout = (pin(np.zeros((Q, stride, 2), np.uint32)), pin(np.zeros(Q, np.uint32)), pin(np.zeros(Q, np.uint32)))
    e2e_cfg = config(selector=args.selector, tile_bytes=args.tile_bytes, ctas_per_sm=args.ctas_per_sm,
                     span_chunk=args.span_chunk)
    for _ in range(2):
        res = ix.query(hb, e2e_cfg, stride=stride, out=hout, copy=False)
    e2e_times = []
    e2e_steps = max(3, min(args.steps, 10))
    for _ in range(e2e_steps):
        flush.zero_()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        res = ix.query(hb, e2e_cfg, stride=stride, out=hout, copy=False)
        if world > 1:
            lists = torch.from_numpy(hout[0]).to(dev)
            lens = torch.from_numpy(hout[1].astype(np.int32)).to(dev)
            dist.all_gather_into_tensor(gath, lists.view(torch.int32))
            dist.all_gather_into_tensor(gath_len, lens)
            m_in.copy_(gath.permute(1, 0, 2, 3))
            m_len.copy_(gath_len.t())
            ix.merge_device(Q, world, m_in, m_len, stride, d["k"], stride, fin, fin_len, fin_thr, stream=sptr)
            fin.cpu(), fin_len.cpu(), fin_thr.cpu()
        e2e_times.append(time.perf_counter() - t)
    e2e_s = float(np.mean(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = Q / e2e_s
    h2d_bytes = hb.nbytes()
    d2h_bytes = hout[0].nbytes + hout[1].nbytes + hout[2].nbytes

    # ---- roofline of the dominant kernel (k_scan: fused scan + c-PQ + tile select)
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    if peaks_path.exists():
        peak = float(json.loads(peaks_path.read_text())["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    postings = int(stats["postings"])
    alg_bytes = 4 * postings  # one u32 posting id per (query, posting)
    scan_avg_ms = float(np.mean(scan_ms))
    achieved = alg_bytes / (scan_avg_ms / 1000.0) / 1e9
    traffic = None
    tpath = ROOT / "profiles" / "scan_dram_bytes.json"
    if tpath.exists():
        try:
            tj = json.loads(tpath.read_text())
            if tj.get("workload") == args.workload and tj.get("n_gpus", 1) == world:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- CPU baseline (reference engine on the host cores; rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sample = args.ref_sample or (96 if args.workload == "tweets" else 512)
            qps, cores, build_ref_s = reference_qps(csr, qb, sample, steps=1, warmup=0)
            cpu = {"value": round(float(np.mean(qps)), 3), "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": f"first {sample} of the {Q} queries, same index (mcx::execute_batch, "
                             f"Selector::cpq, parallel, {cores} threads); ref index build {build_ref_s:.1f}s untimed"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded generator, SURVEY.md 8d)",
            "config": {"workload": WORKLOADS[args.workload], "n_objects": n, "postings": csr.num_postings,
                       "queries": Q, "k": K, "selector": ["cpq", "bucket"][min(args.selector, 1)],
                       "parallelism": f"object-id shards x{world} + NCCL all-gather merge" if world > 1 else "single GPU",
                       "l2": "flushed between timed steps (256 MiB write)",
                       "postings_per_query_mean": round(postings / Q, 1),
                       "generate_s": round(gen_s, 2), "index_upload_s": round(build_s, 2)},
            "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d_bytes),
                    "d2h_bytes_per_step": int(d2h_bytes),
                    "path": "genie_query_batch (C ABI) with pinned host buffers" + (
                        " + all-gather + genie_merge_topk_device" if world > 1 else "")},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": "k_scan (fused posting scan + c-PQ gate/table + tile top-k)",
                         "algorithmic_bytes_per_launch": alg_bytes, "kernel_ms": round(scan_avg_ms, 4),
                         "peak_source": peak_src,
                         "note": "hot lists are shared by many queries and stay L2-resident across the "
                                 "tile-major sweep, so algorithmic bytes exceed DRAM bytes"},
            "cpu_baseline": cpu,
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clocks.summary(),
            "stage_ms": {"step_mean": round(float(np.mean(step_ms)), 4), "scan_mean": round(scan_avg_ms, 4),
                         "lookup_mean": round(float(np.mean(look_ms)), 4), "merge_mean": round(float(np.mean(merge_ms)), 4)},
            "fallback_tiles": int(st.get("fallback_tiles", 0)), "work_items": int(st.get("work_items", 0)),
        }
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
