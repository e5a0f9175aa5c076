"""Multi-GPU execution: object-id shards, one process per GPU.

The object set partitions naturally: GPU g owns ids [g*n/G, (g+1)*n/G)
(partition_dataset, index.hpp:263-291, run concurrently instead of
sequentially as execute_partitioned does, engine.hpp:308-347).  Every rank
answers the whole query batch on its shard; the per-shard top-k lists
(global ids, fixed-size [Q, k] buffers) are exchanged with one all-gather
and merged by merge_topk (engine.hpp:158-177) -- on the device for the NCCL
path, on the host for CPU process groups (gloo).
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np

from . import engine as E


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Object ids owned by `rank`: [n*rank//world, n*(rank+1)//world)."""
    if world < 1 or not (0 <= rank < world):
        raise E.ContractError("bad rank / world size")
    return n * rank // world, n * (rank + 1) // world


def shard_csr(csr: E.CSR, lo: int, hi: int) -> E.CSR:
    """Host CSR of ids [lo, hi), rebased to local ids; keywords absent from the
    shard are dropped (each part is indexed over its own objects)."""
    keys, off, post = csr.keys, csr.key_off, csr.postings
    K = keys.shape[0]
    lens = np.diff(off).astype(np.int64)
    key_of = np.repeat(np.arange(K), lens)
    sel = (post >= lo) & (post < hi)
    kept_key = key_of[sel]
    cnt = np.bincount(kept_key, minlength=K) if K else np.zeros(0, np.int64)
    nz = np.nonzero(cnt)[0]
    new_off = np.zeros(nz.shape[0] + 1, np.uint64)
    new_off[1:] = np.cumsum(cnt[nz])
    return E.CSR(hi - lo, keys[nz], new_off, (post[sel] - lo).astype(np.uint32))


def merge_host(ids: np.ndarray, counts: np.ndarray, lens: np.ndarray, k: np.ndarray):
    """merge_topk (engine.hpp:158-177) of L lists per query on the host.
    ids/counts [Q, L, S], lens [Q, L] -> (ids [Q, K], counts [Q, K], len, threshold)."""
    Q, L, S = ids.shape
    K = int(k.max()) if Q else 1
    oi = np.zeros((Q, max(K, 1)), np.uint32)
    oc = np.zeros((Q, max(K, 1)), np.uint32)
    ol = np.zeros(Q, np.uint32)
    ot = np.zeros(Q, np.uint32)
    for q in range(Q):
        a = np.concatenate([ids[q, l, : lens[q, l]] for l in range(L)]) if L else np.zeros(0, np.uint32)
        c = np.concatenate([counts[q, l, : lens[q, l]] for l in range(L)]) if L else np.zeros(0, np.uint32)
        if np.unique(a).shape[0] != a.shape[0]:
            raise E.ContractError("merge_topk: an object was reported by more than one partition")
        order = np.lexsort((a, -c.astype(np.int64)))
        m = min(int(k[q]), order.shape[0])
        oi[q, :m], oc[q, :m] = a[order[:m]], c[order[:m]]
        ol[q] = m
        ot[q] = oc[q, m - 1] if m >= int(k[q]) and m > 0 else 0
    return oi, oc, ol, ot


def gather_merge_host(local: E.Results, k: np.ndarray, group=None) -> E.Results:
    """All-gather per-shard results over a CPU process group (gloo) and merge."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    Q, S = local.ids.shape
    buf = torch.from_numpy(np.stack([local.ids, local.counts], -1).astype(np.int64))
    lens = torch.from_numpy(local.length.astype(np.int64))
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    lbs = [torch.zeros_like(lens) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    dist.all_gather(lbs, lens, group=group)
    allb = torch.stack(bufs, 1).numpy()  # [Q, world, S, 2]
    alll = torch.stack(lbs, 1).numpy()  # [Q, world]
    oi, oc, ol, ot = merge_host(allb[..., 0].astype(np.uint32), allb[..., 1].astype(np.uint32),
                                alll.astype(np.uint32), np.asarray(k, np.uint32))
    return E.Results(local.qid, oi, oc, ol, ot)


class ShardedIndex:
    """This rank's shard on its GPU + the NCCL all-gather merge."""

    def __init__(self, csr: E.CSR, device: int, group=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.lo, self.hi = shard_range(csr.n, self.rank, self.world)
        self.index = E.DeviceIndex.shard(csr, self.lo, self.hi, device=device)
        self.device = device

    def query(self, batch: E.QueryBatch, cfg=None) -> E.Results:
        """Whole-batch answer on every rank (device path, NCCL all-gather)."""
        import torch
        import torch.distributed as dist

        dev = torch.device("cuda", self.device)
        Q, S = len(batch), max(batch.max_k, 1)
        stream = torch.cuda.Stream(dev)
        with torch.cuda.stream(stream):
            d = {
                "qid": torch.from_numpy(batch.qid.astype(np.int32)).to(dev),
                "k": torch.from_numpy(batch.k.astype(np.int32)).to(dev),
                "item_off": torch.from_numpy(batch.item_off.astype(np.int64)).to(dev),
                "dim": torch.from_numpy(batch.dim.astype(np.int16)).to(dev),
                "lo": torch.from_numpy(batch.lo.astype(np.int32)).to(dev),
                "hi": torch.from_numpy(batch.hi.astype(np.int32)).to(dev),
                "out": torch.zeros((Q, S, 2), dtype=torch.int32, device=dev),
                "out_len": torch.zeros(Q, dtype=torch.int32, device=dev),
                "out_thr": torch.zeros(Q, dtype=torch.int32, device=dev),
                "max_k": batch.max_k, "total_items": batch.num_items, "stride": S,
            }
            for _ in range(4):
                self.index.query_device(d, cfg, stream=stream.cuda_stream)
                if not self.index.status().get("retry"):
                    break
            st = self.index.status()
            # [world, Q, S] rows in rank order: the list-major layout the
            # device merge reads in place
            if dist.get_backend(self.group) == "nccl":  # NVLink all-gather of device buffers
                gath = torch.zeros((self.world, Q, S, 2), dtype=torch.int32, device=dev)
                glen = torch.zeros((self.world, Q), dtype=torch.int32, device=dev)
                dist.all_gather_into_tensor(gath, d["out"], group=self.group)
                dist.all_gather_into_tensor(glen, d["out_len"], group=self.group)
            else:  # CPU process groups (gloo): exchange through host memory
                rows = [torch.zeros((Q, S, 2), dtype=torch.int32) for _ in range(self.world)]
                lens = [torch.zeros(Q, dtype=torch.int32) for _ in range(self.world)]
                dist.all_gather(rows, d["out"].cpu(), group=self.group)
                dist.all_gather(lens, d["out_len"].cpu(), group=self.group)
                gath = torch.stack(rows).to(dev)
                glen = torch.stack(lens).to(dev)
            fin = torch.zeros((Q, S, 2), dtype=torch.int32, device=dev)
            flen = torch.zeros(Q, dtype=torch.int32, device=dev)
            fthr = torch.zeros(Q, dtype=torch.int32, device=dev)
            self.index.merge_device(Q, self.world, gath, glen, S, d["k"], S, fin, flen, fthr,
                                    stream=stream.cuda_stream, list_major=True)
            self.index.status()  # surfaces merge errors (duplicate ids across shards)
        stream.synchronize()
        out = fin.cpu().numpy().view(np.uint32)
        return E.Results(batch.qid.copy(), out[..., 0].copy(), out[..., 1].copy(),
                         flen.cpu().numpy().astype(np.uint32), fthr.cpu().numpy().astype(np.uint32), stats=st)
