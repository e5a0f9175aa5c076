#!/usr/bin/env python
"""Times the pieces of bench.py's e2e step (host encode, host-buffer query) for one workload. GPU box only."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1603_08390_b200 import config  # noqa: E402

ap = bench.argparse.ArgumentParser()
ap.add_argument("--workload", default="ocr")
a = ap.parse_args()
args = bench.argparse.Namespace(workload=a.workload, queries=None, n=None, gpus=1)
w = bench.Workload(args, 0, 1, torch.device("cuda:0"), 0)
Q = len(w.batch)
stride = w.stride
hout = (np.zeros((Q, stride, 2), np.uint32), np.zeros(Q, np.uint32), np.zeros(Q, np.uint32))
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b, h2d, d2h = w.host_encode() if w.m else (w.batch, 0, 0)
    t1 = time.perf_counter()
    w.ix.query(b, config(), stride=stride, out=hout, copy=False)
    t2 = time.perf_counter()
    print(f"{a.workload} iter {i}: host_encode {1e3*(t1-t0):.2f} ms, query(host) {1e3*(t2-t1):.2f} ms")
