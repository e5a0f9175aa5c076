#!/usr/bin/env python
"""Per-phase cycle split of k_scan (setup / dense / scan / extract, warp 0's
prepare vs a scan warp, admits) on the C2 workload, using the instrumented
build (make -C paper_1603_08390_b200/csrc phase).  GPU box only.  Other
workloads: GENIE_ENGINE_LIB=<phase lib> GENIE_PHASE_REPORT=1 python bench.py --workload W."""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def report(ix, items: int) -> str:
    import numpy as np

    from paper_1603_08390_b200 import _native as N

    w = np.zeros(40, np.uint64)
    err = C.create_string_buffer(256)
    N.engine().genie_debug_status(ix.handle, w.ctypes.data_as(N.u64p), 40, err, 256)
    tot = max(1, int(w[20] + w[21] + w[22] + w[23]))
    items = max(1, items)
    return (f"items={items} setup={100*w[20]/tot:.1f}% dense={100*w[23]/tot:.1f}% scan={100*w[21]/tot:.1f}% "
            f"extract={100*w[22]/tot:.1f}% | cycles/item setup={w[20]/items:.0f} dense={w[23]/items:.0f} "
            f"scan={w[21]/items:.0f} extract={w[22]/items:.0f} | admits/item calls={w[24]/items:.0f} "
            f"pass={w[25]/items:.0f} | prep={w[26]/items:.0f} warp1={w[27]/items:.0f} "
            f"tie-fill items={int(w[30])} cycles each={w[31]/max(1, w[30]):.0f} "
            f"scan warps max={w[18]/items:.0f} min={w[19]/items:.0f} | dense items={(int(w[17]) >> 32) & 0xffff} "
            f"lists={int(w[17]) & 0xffffffff} bit-sliced={int(w[17]) >> 48} | per dense item: thread-0 work "
            f"{w[28]/max(1, (int(w[17]) >> 32) & 0xffff):.0f} init+barrier {w[29]/max(1, (int(w[17]) >> 32) & 0xffff):.0f} "
            f"total {w[23]/max(1, (int(w[17]) >> 32) & 0xffff):.0f} | prepare: plan wait {w[34]/items:.0f} "
            f"issue {w[35]/items:.0f} gate start {w[36]/items:.0f} staging {w[37]/items:.0f}")


if __name__ == "__main__":
    os.environ["GENIE_ENGINE_LIB"] = str(ROOT / "paper_1603_08390_b200/lib/phase/libgenie_b200.so")
    sys.path.insert(0, str(ROOT))
    from paper_1603_08390_b200 import DeviceIndex, config, synth  # noqa: E402

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 7_000_000
    ds = synth.tweets(n=n, vocab=1_000_000, words=10, queries=1024, k=100)
    ix = DeviceIndex.from_csr(ds.csr)
    for tb in (0, 32768):
        for _ in range(2):
            r = ix.query(ds.queries, config(tile_bytes=tb), timings=True)
        print(f"tile_bytes={tb or 'auto'} match_ms={r.timings['match_ns']/1e6:.3f} "
              + report(ix, int(r.stats["work_items"])))
