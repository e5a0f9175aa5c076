#!/usr/bin/env python
"""Per-GPU cost of the N-GPU C2 step, measured on one B200 (GPU box only).

The multi-GPU path (bench.py --gpus N) gives every rank the
object-id shard [r n/N, (r+1) n/N) and the whole query batch; each rank's
step is its shard batch, one all-gather of the [Q, k] rows, and the list-major
device merge.  With one GPU available this probe builds all N shards of the
headline workload on cuda:0 and times, with CUDA events and the L2 flushed
between steps (as bench.py does):

  * each shard's batch alone (the graph-replayed device-resident step) -- a
    rank's compute; the N-GPU step waits for the slowest shard;
  * the merge of the N shards' real rows (genie_merge_topk_device, list-major);

and reports the predicted N-GPU step as slowest shard + merge + an all-gather
ESTIMATE (not measured: N-1 rows of Q x k x 8 B received per rank at 600 GB/s
plus 10 us of NCCL latency).  The merged rows are checked against the
single-index batch's hash_results.

  python tools/shard_probe.py [--workload tweets] [--ns 1,2,4,8] [--steps 20]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    from paper_1603_08390_b200 import config
    from paper_1603_08390_b200.engine import hash_results

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="tweets", choices=["tweets", "adult"])
    ap.add_argument("--ns", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    args = argparse.Namespace(workload=a.workload, queries=0, n=0)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    cfg = config(stage_events=True, graph=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timed(fn, steps):
        ms = []
        for _ in range(3):
            fn()
        for _ in range(steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms.append(e0.elapsed_time(e1))
        return float(np.median(ms))

    out = []
    base_ms = None
    for N in [int(x) for x in a.ns.split(",")]:
        shards = [bench.Workload(args, r, N, dev, 0) for r in range(N)]
        Q, stride = shards[0].Q, shards[0].stride
        step_ms = []
        for w in shards:
            for _ in range(3):  # workspace growth (GENIE_RETRY) settles before timing, as in bench.py
                w.ix.query_device(w.d, cfg, stream=sptr)
                torch.cuda.synchronize(dev)
                if not w.ix.status().get("retry"):
                    break
            step_ms.append(timed(lambda w=w: w.ix.query_device(w.d, cfg, stream=sptr), a.steps))
            w.ix.status()
        # the all-gather's result (list-major [N][Q][stride]) and the merge
        gath = torch.stack([w.d["out"] for w in shards])
        gath_len = torch.stack([w.d["out_len"] for w in shards])
        fin = torch.zeros((Q, stride, 2), dtype=torch.int32, device=dev)
        fin_len = torch.zeros(Q, dtype=torch.int32, device=dev)
        fin_thr = torch.zeros(Q, dtype=torch.int32, device=dev)
        d0, ix0 = shards[0].d, shards[0].ix
        if N > 1:
            merge_ms = timed(lambda: ix0.merge_device(Q, N, gath, gath_len, stride, d0["k"], stride, fin, fin_len,
                                                      fin_thr, stream=sptr, list_major=True), a.steps)
            ix0.status()
            rows, lens, thr = fin, fin_len, fin_thr
        else:
            merge_ms = 0.0
            rows, lens, thr = d0["out"], d0["out_len"], d0["out_thr"]
        r = rows.cpu().numpy().view(np.uint32)
        h = hash_results(shards[0].batch.qid, thr.cpu().numpy().view(np.uint32), lens.cpu().numpy().view(np.uint32),
                         r[:, :, 0], r[:, :, 1])
        ag_est_ms = 0.0 if N == 1 else ((N - 1) * Q * stride * 8 / 600e9 + 10e-6) * 1e3
        pred = max(step_ms) + merge_ms + ag_est_ms
        base_ms = base_ms or pred
        line = {"n_gpus": N, "shard_step_ms": [round(x, 4) for x in step_ms], "slowest_shard_ms": round(max(step_ms), 4),
                "merge_ms": round(merge_ms, 4), "allgather_ms_estimate": round(ag_est_ms, 4),
                "predicted_step_ms": round(pred, 4), "predicted_qps": round(Q / pred * 1e3, 1),
                "predicted_speedup": round(base_ms / pred, 2), "hash": f"{h:#018x}"}
        out.append(line)
        print(json.dumps(line), flush=True)
        for w in shards:
            w.ix.close()
        del shards, gath, gath_len
        torch.cuda.empty_cache()
    hashes = {l["hash"] for l in out}
    print(json.dumps({"merged_hash_equal_across_n": len(hashes) == 1}))


if __name__ == "__main__":
    main()
