"""Multi-process (world_size 2, gloo, CPU) test of the sharded path's
plumbing: each rank scans only its id range, the fixed-size per-shard top-k
buffers are all-gathered and merged (merge_topk) -- equal to the unsharded
answer.  The per-shard scan is the CPU oracle here (no GPU in this tier)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import Oracle
        from paper_1603_08390_b200 import synth
        from paper_1603_08390_b200.dist import gather_merge_host, shard_csr, shard_range

        ds = synth.tweets(n=40_000, vocab=3_000, words=10, queries=20, k=30)
        lo, hi = shard_range(ds.csr.n, rank, world)
        o = Oracle()
        local = o.index(shard_csr(ds.csr, lo, hi)).execute(ds.queries, stride=30)
        local.ids = local.ids + np.uint32(lo)  # global ids
        from paper_1603_08390_b200.engine import Results
        merged = gather_merge_host(Results(local.qid, local.ids, local.counts, local.length, local.threshold),
                                   ds.queries.k)
        whole = o.index(ds.csr).execute(ds.queries, stride=30)
        ok = np.array_equal(merged.length, whole.length) and np.array_equal(merged.threshold, whole.threshold)
        for q in range(len(ds.queries)):
            n = int(whole.length[q])
            ok &= np.array_equal(merged.ids[q, :n], whole.ids[q, :n])
            ok &= np.array_equal(merged.counts[q, :n], whole.counts[q, :n])
        out[rank] = int(ok)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shard_merge_equals_unsharded():
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    assert dict(out) == {0: 1, 1: 1}
