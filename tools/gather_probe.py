"""Gather probe: LDG gather vs TMA bulk-copy gather on local rows, alone and
concurrently with a sampling level (two streams)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2505_10806_b200 import _lib
from paper_2505_10806_b200._lib import ptr
from paper_2505_10806_b200.engine import bases_array

_lib.device()
n, G, nrow, d = 2_000_000, 8, 600_000, 100
rows0 = torch.randn((n, d), device="cuda")
ids = torch.randint(0, n, (G, nrow), dtype=torch.int32, device="cuda")
nids = torch.full((G,), nrow, dtype=torch.int32, device="cuda")
route = torch.arange(n, dtype=torch.int32, device="cuda")
b = [0] * 16
b[0] = rows0.data_ptr()
bases = bases_array(b)
out = torch.empty((G, nrow, d), device="cuda")
cnt = torch.zeros((G, 8), dtype=torch.int32, device="cuda")
want = rows0[ids.long()]


def run(kind, per_sm=0):
    s = _lib.stream_handle()
    if kind == "ldg":
        _lib.call("rg_gather_bundle", ptr(ids), ptr(nids), nrow, G, ptr(route), bases.ctypes.data,
                  d, d, -1, 0, ptr(out), ptr(cnt), s)
    else:
        _lib.call("rg_gather_bundle_tma", ptr(ids), ptr(nids), nrow, G, ptr(route),
                  bases.ctypes.data, d, d, -1, ptr(out), ptr(cnt), per_sm, s)


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


payload = G * nrow * d * 4
for kind, per in (("ldg", 0), ("tma", 2), ("tma", 4), ("tma", 8), ("tma", 16)):
    out.zero_()
    ms = timeit(lambda: run(kind, per))
    ok = torch.equal(out, want)
    print(f"{kind} per_sm={per:2d}: {2 * payload / ms / 1e6:8.1f} GB/s (read+write) ok={ok}")
