#!/usr/bin/env python
"""Where bench.py's e2e step spends the time beyond the device-resident batch
(GPU box only): wall time of the host-buffer call with and without the CUDA
graph and the L2 flush, against the device-resident call timed the same way.

  python tools/e2e_probe.py --workload tweets
"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1603_08390_b200 import QueryBatch, config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="tweets")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
dev = torch.device("cuda:0")
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
args = argparse.Namespace(workload=a.workload, queries=None, n=None, gpus=1)
w = bench.Workload(args, 0, 1, dev, 0)
ix, Q, stride = w.ix, w.Q, w.stride
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()  # noqa: E731
hout = (pin(np.zeros((Q, stride, 2), np.uint32)), pin(np.zeros(Q, np.uint32)), pin(np.zeros(Q, np.uint32)))
qb = w.batch
hb = QueryBatch(pin(qb.qid), pin(qb.k), pin(qb.item_off), pin(qb.dim), pin(qb.lo), pin(qb.hi))
ub = QueryBatch(*(np.ascontiguousarray(x) for x in (qb.qid, qb.k, qb.item_off, qb.dim, qb.lo, qb.hi)))
uout = (np.zeros((Q, stride, 2), np.uint32), np.zeros(Q, np.uint32), np.zeros(Q, np.uint32))


def timed(fn, do_flush):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(a.reps):
        if do_flush:
            flush.zero_()
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return 1e3 * float(np.median(ts))


g, ng = config(graph=True), config(graph=False)
sptr = stream.cuda_stream
cases = {
    "host pinned, graph, flush": (lambda: ix.query(hb, g, stride=stride, out=hout, copy=False), True),
    "host pinned, graph, warm L2": (lambda: ix.query(hb, g, stride=stride, out=hout, copy=False), False),
    "host pinned, no graph, flush": (lambda: ix.query(hb, ng, stride=stride, out=hout, copy=False), True),
    "host pageable, flush": (lambda: ix.query(ub, g, stride=stride, out=uout, copy=False), True),
    "device, graph, flush (+sync)": (lambda: (ix.query_device(w.d, g, stream=sptr), torch.cuda.synchronize(dev)), True),
    "device, graph, warm L2 (+sync)": (lambda: (ix.query_device(w.d, g, stream=sptr), torch.cuda.synchronize(dev)),
                                       False),
}
for name, (fn, fl) in cases.items():
    ms = timed(fn, fl)
    print(f"{a.workload:8s} {name:34s} {ms:7.3f} ms  ({Q / ms * 1e3:,.0f} q/s)", flush=True)
