"""HBM probe: write-only (fill) and copy (read+write) bandwidth over buffers
far larger than L2, CUDA-event timed, best of N.  The bundle gather is
~93 % writes (34.4 of 36.9 GB per G = 128 Products launch), so its ceiling
is the write-only rate, not the copy rate of MEASURED_PEAKS.json.

  python tools/hbm_probe.py [--gb 8]
"""

from __future__ import annotations

import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=8.0)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    n = int(a.gb * 2**30) // 4
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    x.fill_(1.0)

    def best(fn, nbytes):
        out = []
        for _ in range(a.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            out.append(nbytes / (s.elapsed_time(e) / 1e3) / 1e9)
        return max(out)

    res = {"bytes_per_buffer": 4 * n,
           "write_only_gbs": best(lambda: y.fill_(2.0), 4 * n),
           "copy_gbs": best(lambda: y.copy_(x), 8 * n),
           "read_only_gbs": best(lambda: x.sum(), 4 * n)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
