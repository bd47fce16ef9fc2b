"""K9 probe: the group prefetch's row copy (rg_prefetch_rows) from a peer
GPU's shard into a local shadow, one process, 2 GPUs, CUDA-event timed — the
papers100M-shaped case (sorted union of ~5.8 M of 13.9 M peer rows, 512-B
rows) and the Products case (400-B rows) — plus the whole-shard copy-engine
form (rg_copy_bytes).  Run under ncu (single process) for the NVLink
counters of prefetch_rows_kernel.

  python tools/prefetch_probe.py [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    from paper_2505_10806_b200 import _lib
    from paper_2505_10806_b200.engine import bases_array

    torch.cuda.set_device(0)
    _lib.device()
    _lib.call("rg_enable_peer", 1)
    out = {}
    for name, n_q, d, n_union in (("papers100m", 13_900_000, 128, 5_800_000),
                                  ("products", 306_000, 100, 258_000)):
        peer = torch.randn((n_q, d), device="cuda:1")
        shadow = torch.empty((n_q, d), device="cuda:0")
        rng = np.random.default_rng(1)
        ids = np.sort(rng.choice(n_q, n_union, replace=False)).astype(np.int32)
        ids_d = torch.from_numpy(ids).cuda()
        nids = torch.tensor([n_union], dtype=torch.int32, device="cuda")
        route = torch.arange(n_q, dtype=torch.int32, device="cuda") | (1 << 28)  # kind 1
        src, dst = [0] * 16, [0] * 16
        src[1], dst[1] = peer.data_ptr(), shadow.data_ptr()
        s = _lib.stream_handle()

        def rows():
            _lib.call("rg_prefetch_rows", ids_d.data_ptr(), nids.data_ptr(), n_union,
                      route.data_ptr(), bases_array(src), bases_array(dst), d, d, s)

        def whole():
            _lib.call("rg_copy_bytes", shadow.data_ptr(), peer.data_ptr(), peer.numel() * 4, s)

        res = {}
        for label, fn, nbytes in (("row_gather", rows, n_union * d * 4),
                                  ("whole_shard_copy_engine", whole, n_q * d * 4)):
            for _ in range(2):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            res[label] = {"ms": ms, "bytes": nbytes, "gbs": nbytes / ms / 1e6}
        assert torch.equal(shadow[torch.from_numpy(ids).long().cuda()],
                           peer[torch.from_numpy(ids).long().cuda(1)].to("cuda:0"))
        out[name] = res
        del peer, shadow
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
