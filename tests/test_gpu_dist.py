"""The multi-process sharded path (dist.ShardedIndex, one process per shard)
on the GPU: 2 and 4 processes all on cuda:0, each holding its object-id shard
(genie_index_create_shard), all-gathering the per-shard top-k rows over a
gloo group and merging them with the device merge (list-major layout) --
exactly bench.py's N>1 step minus the NCCL transport, which cannot place two
ranks on one GPU.  The merged answer must equal the unsharded one and the
CPU oracle (acceptance.cpp:540-559)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


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
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
        from oracle.pyoracle import Oracle
        from paper_1603_08390_b200 import hash_results, synth
        from paper_1603_08390_b200.dist import ShardedIndex

        ds = synth.tweets(n=500_000, vocab=80_000, words=10, queries=64, k=100)
        sh = ShardedIndex(ds.csr, device=0)
        got = sh.query(ds.queries)
        want = Oracle().index(ds.csr).execute(ds.queries)
        ok = np.array_equal(got.length, want.length) and np.array_equal(got.threshold, want.threshold)
        for q in range(len(ds.queries)):
            ok &= got.row(q) == want.row(q)
        ok &= hash_results(got.qid, got.threshold, got.length, got.ids, got.counts) == \
            hash_results(want.qid, want.threshold, want.length, want.ids, want.counts)
        out[rank] = int(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_processes_on_one_gpu_equal_oracle(gpu, world):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    assert dict(out) == {r: 1 for r in range(world)}
