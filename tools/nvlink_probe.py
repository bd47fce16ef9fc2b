"""NVLink probe: remote-row gather throughput of gather_bundle_kernel vs a
contiguous peer copy (one process, 2 GPUs, peer access)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2505_10806_b200 import _lib
from paper_2505_10806_b200.engine import bases_array, gather_bundle

torch.cuda.set_device(0)
_lib.device()
_lib.call("rg_enable_peer", 1)
n, G = 2_000_000, 8
for d, src_stride in ((100, 100), (100, 104), (100, 128), (128, 128)):
    stride = d
    rows1 = torch.randn((n, src_stride), device="cuda:1")
    rows0 = torch.randn((n, src_stride), device="cuda:0")
    nrow = 400_000
    ids = torch.randint(0, n, (G, nrow), dtype=torch.int32, device="cuda:0")
    nids = torch.full((G,), nrow, dtype=torch.int32, device="cuda:0")
    for where, base, kind in (("local", rows0, 0), ("peer", rows1, 1)):
        route = (torch.arange(n, dtype=torch.int64, device="cuda:0") | (kind << 28)).to(torch.int32)
        b = [0] * 16
        b[kind] = base.data_ptr()
        bases = bases_array(b)
        out = torch.empty((G, nrow, stride), device="cuda:0")
        cnt = torch.zeros((G, 8), dtype=torch.int32, device="cuda:0")
        for _ in range(3):
            gather_bundle(ids, nids, nrow, G, route, bases, src_stride, stride, -1, out, cnt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            gather_bundle(ids, nids, nrow, G, route, bases, src_stride, stride, -1, out, cnt)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        payload = G * nrow * stride * 4
        print(f"d={d} src_stride={src_stride} {where:5s} gather: {payload/ms/1e6:8.1f} GB/s payload read ({ms:.3f} ms)")
    big1 = torch.empty(512 * 2**20 // 4, device="cuda:1")
    big0 = torch.empty_like(big1, device="cuda:0")
    for _ in range(3): big0.copy_(big1)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5): big0.copy_(big1)
    e1.record(); torch.cuda.synchronize()
    print(f"peer copy 512MiB: {5*big1.numel()*4/e0.elapsed_time(e1)/1e6:.1f} GB/s")
