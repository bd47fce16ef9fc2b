#!/usr/bin/env python
"""bench.py — RapidGNN sample+fetch hot path on B200 (BASELINE.json metric).

A step = one group of G consecutive mini-batches of the plan, each put
through the reference's per-batch producer body (prefetch.py:123-125:
plan.block -> sample_block, then assemble_bundle for worker p with the
epoch's steady hot cache).  value = worker-batches/s summed over GPUs.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N

Inputs: gnnpipe.synth_powerlaw(n, m, d, C, seed=7) of the named shape,
reproduced bit-exactly by the native generator, partitioned with
partition_edgecut(k).  Rank r runs worker p = r; partition shard q lives on
GPU q mod N (peer shards read over NVLink through CUDA IPC pointers).
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
# more hardware work queues than streams in use: with the default 8, streams
# alias onto shared queues, and a cross-GPU wait kernel of shared sampling
# could then hold up an unrelated stream's work (a false dependency)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, str(ROOT))

METRIC = "sample+fetch mini-batches/s, Products-shape, 1-8 B200; remote rows/epoch"
CONFIGS = {
    # group 128: the chunk-major gather queue serves rows shared by the group's
    # batches from L2, so larger groups read less HBM (N = 1: G 32 / 64 / 96 /
    # 128 -> 9,490 / 11,133 / 11,715 / 11,877 batches/s); at N > 1 a group's
    # peer rows are prefetched once, so the NVLink cost per batch falls with G
    # too.  ~130 GB of HBM per GPU (two 55 GB bundle slots).
    "products": dict(n=2_449_029, m=13, d=100, classes=47, fanouts=[15, 10, 5], batch=1024,
                     parts=8, group=128),
    "reddit": dict(n=232_965, m=246, d=602, classes=41, fanouts=[25, 10], batch=1024, parts=8),
    "c1": dict(n=100_000, m=10, d=128, classes=8, fanouts=[10, 5], batch=1024, parts=2),
    # config X: structure / masks / partition from the bit-exact native
    # generator; feature rows generated on the device (rg_fill_features)
    "papers100m": dict(n=111_059_956, m=7, d=128, classes=172, fanouts=[15, 10, 5], batch=4096,
                       parts=8, device_features=True, group=8),
}
S0 = 7
L2_BYTES = 126 * 2**20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="products", choices=sorted(CONFIGS))
    ap.add_argument("--group", type=int, default=0, help="batches per step (0: config default)")
    ap.add_argument("--check", action="store_true",
                    help="verify one batch bit-exactly against the CPU oracle after timing")
    ap.add_argument("--cache-pct", type=float, default=15.0)
    ap.add_argument("--prng", default="splitmix",
                    choices=["splitmix", "pcg32", "sfc64", "xoshiro256pp"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--train-groups", type=int, default=4,
                    help="e2e_train leg: groups of 32 batches trained, overlapped vs serial "
                         "(0: skip)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--nvtx", action="store_true", help="NVTX range 'timed' around the timed steps")
    ap.add_argument("--serial", action="store_true",
                    help="no sample/gather overlap (one stream, per-kernel timing)")
    ap.add_argument("--timeline", action="store_true",
                    help="stderr: per-stream event timeline of the timed overlapped steps")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="N>1 group prefetch: NVLink loads through CUDA IPC (p2p) or two "
                         "NCCL all-to-alls, ids out and rows back (nccl; spans nodes)")
    ap.add_argument("--pull", action="store_true",
                    help="N>1: every batch pulls its peer rows over NVLink (no group prefetch)")
    ap.add_argument("--no-share", action="store_true",
                    help="N>1: every rank samples every batch of a group itself (default: the "
                         "ranks split each group's sampling and copy the shares over NVLink)")
    ap.add_argument("--env-sweep", default="",
                    help="diagnostic: ';'-separated K=V[,K=V] library knob settings; the timed "
                         "steps are re-run under each and logged (env_sweep key)")
    ap.add_argument("--graphs", action="store_true",
                    help="replay each group's launches from a captured CUDA graph (serial)")
    return ap.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- inputs
def build_inputs(cfg):
    from paper_2505_10806_b200.graph import synth_powerlaw
    from paper_2505_10806_b200.partition import partition_edgecut

    t = time.time()
    big = cfg.get("device_features", False)
    g = synth_powerlaw(cfg["n"], cfg["m"], cfg["d"], cfg["classes"], S0, with_features=not big,
                       with_labels=not big)
    book = partition_edgecut(g, cfg["parts"])
    log(f"[bench] inputs: n={g.num_nodes} E={g.num_edges} in {time.time() - t:.1f}s")
    return g, book


def structure_pin(args, g, book):
    """papers100M shape: the generated CSR, train mask and LDG owners
    against the content hashes the C oracle produced in the build container
    (tests/golden/papers100m.json, tests/golden/make_golden_papers100m.py);
    None for shapes pinned elsewhere (tests/test_host_native.py)."""
    import hashlib

    f = ROOT / "tests" / "golden" / f"{args.config}.json"
    if args.config != "papers100m" or not f.exists():
        return None
    want = json.loads(f.read_text())["hash"]

    def h(a):
        return hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=16).hexdigest()

    got = {"indptr": h(np.asarray(g.indptr, dtype="<i8")),
           "indices": h(np.asarray(g.indices, dtype="<i4")),
           "train_mask": h(np.asarray(g.train_mask, dtype="u1")),
           "owner": h(np.asarray(book.owner, dtype="u1"))}
    return got == want


def build_inputs_oracle(cfg):
    """The same graph and partition from the CPU oracle (oracle/oracle_graph.c,
    pinned to the reference's hashes): the reference arm never loads the
    product library."""
    from oracle import graph_oracle as go

    t = time.time()
    g = go.synth_powerlaw(cfg["n"], cfg["m"], cfg["d"], S0)
    owner = go.partition_edgecut(g, cfg["parts"])
    log(f"[bench] oracle inputs: n={g.num_nodes} E={g.num_edges} in {time.time() - t:.1f}s")
    return g, owner


def reference_hot_set(cfg, args, g, owner, part=0):
    """Worker `part`'s steady hot set for epoch 0 at --cache-pct, as the
    reference computes it (collect_access -> top_hot, plan.py:117-141;
    n_hot = int(#remote * pct / 100), train.py:165-168).  Products worker 0
    at 15 %: the set the reference itself produced (tests/golden/
    products_w0.npz, made by tests/golden/make_golden_products.py); other
    cases: the oracle over every batch of the epoch on the host cores."""
    gold = ROOT / "tests" / "golden"
    if (args.config == "products" and part == 0 and args.cache_pct == 15.0
            and args.prng == "splitmix" and (gold / "products_w0.npz").exists()):
        meta = json.loads((gold / "products.json").read_text())["workers"]["0"]["hot"]["15"]
        hot = np.cumsum(np.load(gold / "products_w0.npz")["hot15_delta"].astype(np.int64))
        assert len(hot) == meta["n_hot"]
        return hot, meta["n_hot"], "reference (tests/golden/products_w0.npz)"
    from oracle import gnn_oracle as orc

    train = np.flatnonzero(g.train_mask)
    nb = -(-len(train) // cfg["batch"])
    state = cpu_state(g, owner, cfg, None, part)
    ctx = mp.get_context("fork")
    with ctx.Pool(os.cpu_count() or 1, initializer=_cpu_init, initargs=(state,)) as pool:
        sets = pool.map(_cpu_inputs, range(nb), chunksize=4)
    ids, counts = orc.access_counts(sets, owner, part)
    n_hot = int(len(ids) * args.cache_pct / 100.0)
    return orc.hot_set(ids, counts, n_hot), n_hot, "oracle plan pass (host)"


class UnionCounter:
    """|union of a group's input sets| on the device (rg_group_union with an
    all-ones mask over the sampler's level-L bitmaps, then a popcount): the
    distinct source rows one gather launch has to read at least once."""

    def __init__(self, nwords: int):
        import torch

        self.nw = nwords
        self.mask = torch.full((nwords,), -1, dtype=torch.int32, device="cuda")
        self.out = torch.empty(nwords, dtype=torch.int32, device="cuda")
        self.lut = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64,
                                device="cuda")
        self.counts = []

    def add(self, smp, ng: int) -> None:
        from paper_2505_10806_b200 import _lib

        _lib.call("rg_group_union", smp.bm.data_ptr(), self.nw, ng, self.mask.data_ptr(),
                  self.out.data_ptr(), _lib.stream_handle())
        self.counts.append(self.lut[self.out.view(dtype=__import__("torch").uint8).long()].sum())

    def total(self) -> int:
        return int(sum(int(c.item()) for c in self.counts))


# ---------------------------------------------------------------- clocks
class Clocks:
    """SM clock + throttle reasons sampled during the run (NVML at 20 ms;
    nvidia-smi every 200 ms if NVML is unavailable)."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self.source = "nvml"
        self._nv = self._nvml()  # initialise before the thread starts sampling

    def _nvml(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            bits = (nv.nvmlClocksThrottleReasonHwSlowdown,
                    nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                    nv.nvmlClocksThrottleReasonSwThermalSlowdown,
                    nv.nvmlClocksThrottleReasonSwPowerCap)
            return nv, h, bits, float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        except Exception:
            return None

    def _run(self):
        if self._nv is not None:
            nv, h, bits, mx = self._nv
            while not self._stop.is_set():
                try:
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    self.samples.append((float(sm), mx, [bool(r & b) for b in bits]))
                except Exception:
                    pass
                self._stop.wait(0.01)
            return
        self.source = "nvidia-smi"
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                self.samples.append((float(f[0]), float(f[1]),
                                     [x.lower().startswith("active") for x in f[2:6]]))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"]}
        sm = [x[0] for x in self.samples]
        reasons = sorted({self.NAMES[i] for x in self.samples for i in range(4) if x[2][i]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(x[1] for x in self.samples),
                "reasons": reasons, "samples": len(self.samples), "source": self.source}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str, workload: str, group: int):
    """DRAM bytes per launch from the committed ncu capture of exactly this
    workload and group size (profiles/traffic.json), else None."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get(f"{workload}/G{group}", {}).get(kernel)
    return None


# ---------------------------------------------------------------- CPU oracle (port)
_CPU = {}


def _cpu_init(state):
    _CPU.update(state)


def _cpu_batch(i: int) -> int:
    """One reference mini-batch on the host: oracle sample_block + bundle
    rows + provenance accounting (the producer body, prefetch.py:123-125)."""
    from oracle import gnn_oracle as orc

    st = _CPU
    seeds = st["perm"][i * st["batch"]:(i + 1) * st["batch"]]
    fr, _ = orc.block(st["indptr"], st["indices"], seeds, st["fanouts"],
                      orc.batch_seed(S0, 0, i))
    ids = fr[-1]
    rows = st["features"][ids]
    orc.route_counts(ids, st["owner"], st["part"], st["hot"])
    return int(rows.shape[0])


def _cpu_inputs(i: int) -> np.ndarray:
    """input_nodes of batch i (oracle sample_block)."""
    from oracle import gnn_oracle as orc

    st = _CPU
    seeds = st["perm"][i * st["batch"]:(i + 1) * st["batch"]]
    fr, _ = orc.block(st["indptr"], st["indices"], seeds, st["fanouts"], orc.batch_seed(S0, 0, i))
    return fr[-1]


def cpu_state(g, owner, cfg, hot_ids, part=0):
    from oracle import gnn_oracle as orc

    train = np.flatnonzero(g.train_mask)
    return {"perm": orc.epoch_order(train, S0, 0), "batch": cfg["batch"], "indptr": g.indptr,
            "indices": g.indices, "fanouts": cfg["fanouts"], "features": g.features,
            "owner": np.asarray(owner), "part": part, "hot": hot_ids}


def cpu_baseline(state, seconds: float, nb: int):
    """Oracle port timed on the host cores: fork P = cpu_count workers, each
    takes batches i = r, r+P, ... ; bounded to ~`seconds` of wall time."""
    _cpu_init(state)
    t = time.time()
    _cpu_batch(0)
    t1 = time.time() - t
    cores = os.cpu_count() or 1
    per = max(1, int(seconds / max(t1, 1e-3) / 1.5))
    total = min(nb, cores * per)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_cpu_init, initargs=(state,)) as pool:
        pool.map(_cpu_batch, range(min(cores, total)))  # warm the workers
        t = time.time()
        pool.map(_cpu_batch, range(total), chunksize=1)
        wall = time.time() - t
    return {"value": total / wall, "unit": "batches/s", "cores": cores, "kind": "port",
            "sample": f"{total} mini-batches of epoch 0 (oracle sample_block + bundle rows + "
                      f"accounting, worker 0) over {cores} forked processes; "
                      f"1-process {1.0 / t1:.3f} batches/s"}


# ---------------------------------------------------------------- reference arm
def workload_config(args, cfg, part, n_hot) -> dict:
    """The `config` both arms print: the workload only (identical keys and
    values for the same workload, so the driver can pair the arms)."""
    return {"workload": args.config, "batch_size": cfg["batch"], "fanouts": cfg["fanouts"],
            "partitions": cfg["parts"], "worker": part, "cache_pct": args.cache_pct,
            "n_hot": int(n_hot), "prng": args.prng}


def run_reference(args, cfg):
    """The reference's own CPU implementation of the path on the host cores:
    the oracle port of the producer body (sample_block + assemble_bundle of
    worker 0 with the epoch's steady 15 % hot cache, prefetch.py:123-125) —
    the reference itself is pure Python and cannot travel to the GPU box.
    Inputs come from the C oracle generator; nothing loads the product
    library.  One step = one batch per host core (forked processes)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if cfg.get("device_features"):
        emit({"impl": "reference", "unavailable": "papers100M-shaped features are generated on "
                                                  "the device; no host feature table to read"})
        return
    g, owner = build_inputs_oracle(cfg)
    hot, n_hot, hot_src = reference_hot_set(cfg, args, g, owner, 0)
    state = cpu_state(g, owner, cfg, hot, 0)
    _cpu_init(state)
    cores = os.cpu_count() or 1
    nb = -(-int(g.train_mask.sum()) // cfg["batch"])
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_cpu_init, initargs=(state,)) as pool:
        i = 0
        for _ in range(args.warmup):
            pool.map(_cpu_batch, [(i + r) % nb for r in range(cores)], chunksize=1)
            i += cores
        t = time.time()
        for _ in range(args.steps):
            pool.map(_cpu_batch, [(i + r) % nb for r in range(cores)], chunksize=1)
            i += cores
        wall = time.time() - t
    value = args.steps * cores / wall
    line = {"metric": METRIC, "value": value, "unit": "batches/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": (f"synthetic: gnnpipe.synth_powerlaw({cfg['n']}, {cfg['m']}, {cfg['d']}, "
                     f"{cfg['classes']}, seed={S0}) + partition_edgecut(k={cfg['parts']}), "
                     f"from the C oracle (oracle/oracle_graph.c, hash-pinned)"),
            "impl": "reference",
            "config": workload_config(args, cfg, 0, n_hot),
            "batches_per_step": cores, "parallelism": f"{cores} forked host processes",
            "hot_set": hot_src,
            "cpu_baseline": {"value": value, "unit": "batches/s", "cores": cores, "kind": "port",
                             "sample": f"{args.steps} steps x {cores} mini-batches of epoch 0 "
                                       f"(oracle sample_block + bundle rows + accounting of "
                                       f"worker 0 with its {n_hot}-row steady cache), one batch "
                                       f"per process"},
            "e2e": {"value": value, "unit": "batches/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    # the reference arm must not touch the product: no module, no library
    assert not any(m.startswith("paper_2505_10806_b200") for m in sys.modules)
    with open("/proc/self/maps") as f:
        assert "librapidgnn_b200" not in f.read()
    emit(line)


# ---------------------------------------------------------------- B200 arm
_JSON_OUT = None


def _claim_stdout() -> None:
    """The driver reads ONE JSON line from stdout: keep a private handle on
    the real stdout for it and point fd 1 at stderr, so nothing a library
    prints (NCCL's version banner under NCCL_DEBUG=VERSION/INFO, CUDA or
    torch warnings) can land on stdout."""
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
        sys.stdout = sys.stderr


def emit(line: dict) -> None:
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    _claim_stdout()
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "WARN")  # stdout carries only the JSON line
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2505_10806_b200 import _lib
    from paper_2505_10806_b200.engine import DeviceGraph, FeatureStore
    from paper_2505_10806_b200.pipeline import WorkerPipeline, resolve_n_hot
    from paper_2505_10806_b200.plan import candidates, threshold_select
    from paper_2505_10806_b200.sampler import SeedSchedule
    from paper_2505_10806_b200 import multigpu

    g, book = build_inputs(cfg)
    pin = structure_pin(args, g, book) if args.check else None
    k, d = cfg["parts"], cfg["d"]
    if world > k:
        raise SystemExit(f"--gpus {world} > partitions {k}")
    part = rank
    owner = book.owner
    dg = DeviceGraph(g.indptr, g.indices, g.num_nodes)
    store = FeatureStore(owner, k, d)
    shard_ids = [np.flatnonzero(owner == q) for q in range(k)]
    for q in range(k):
        if q % world != rank:
            continue
        if cfg.get("device_features"):
            ids_q = torch.from_numpy(shard_ids[q].astype(np.int32)).cuda()
            rows = torch.empty((len(shard_ids[q]), store.src_stride), device="cuda")
            _lib.call("rg_fill_features", ids_q.data_ptr(), len(shard_ids[q]), d,
                      store.src_stride, S0, rows.data_ptr(), _lib.stream_handle())
            store.set_shard(q, rows)
        else:
            store.set_shard(q, FeatureStore.pad_rows(g.features[shard_ids[q]], store.src_stride,
                                                     dg.device))
    if world > 1 and args.transport == "p2p":
        multigpu.exchange_shards(store, rank, world)
    if args.transport == "nccl" and args.pull:
        raise SystemExit("--transport nccl needs the group prefetch (no --pull)")
    store.build_route(shard_ids)
    train = np.flatnonzero(g.train_mask)
    group = args.group or cfg.get("group", 32)
    pipe = WorkerPipeline(dg, store, part, train, cfg["fanouts"], cfg["batch"], S0, group,
                          nbuf=1 if (args.serial or args.graphs) else 2, prng=args.prng)
    nb, G = pipe.nb, pipe.G
    sched = SeedSchedule(S0, 1, nb)
    if world > 1 and not args.pull:
        pipe.enable_prefetch(args.transport, rank, world)  # before the cache fill (nccl)
    if world > 1 and not args.no_share and not args.serial and not args.graphs:
        pipe.enable_shared_sampling(rank, world)

    # per-epoch part: plan pass (access counts), hot set, cache fill
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    share_plan = world > 1 and getattr(pipe, "shared", False)
    counts_local = pipe.count_epoch(sched, 0)  # first pass loads modules / warms the allocator
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0.record()
    counts = pipe.count_epoch(sched, 0, shared=share_plan)
    ev1.record()
    torch.cuda.synchronize()
    plan_ms = ev0.elapsed_time(ev1)
    plan_shared_exact = bool(torch.equal(counts, counts_local)) if share_plan else None
    del counts_local
    _, nout, hist, bm = candidates(counts, store.owner, part, nb)
    n_remote = int(nout.item())
    n_hot = resolve_n_hot(args.cache_pct, n_remote)
    hot = threshold_select(counts, bm, hist.cpu().numpy().astype(np.int64), n_hot)
    pipe.build_cache(hot)
    pipe.start_epoch(sched, 0)
    torch.cuda.synchronize()
    log(f"[bench] rank {rank}: plan pass {plan_ms:.1f} ms, {n_remote} remote, n_hot {n_hot}")

    n_full = max(1, nb // G)
    smp = pipe.sampler

    def step(kk, timed_events=None):
        i0 = (kk % n_full) * G
        if args.graphs:
            return i0, pipe.step_graph(i0)
        if not args.serial:
            return i0, pipe.step_overlapped(i0)
        ng = min(G, nb - i0)
        pipe.plan.fill(pipe.perm, 0, i0, ng)
        smp.run(ng)
        if timed_events is not None:
            timed_events[0].record()
        pipe.gather(ng, i0)
        if timed_events is not None:
            timed_events[1].record()
        return i0, ng

    unions = UnionCounter(dg.nwords)
    clk = Clocks(local).__enter__()  # under load from warm-up to the end of the epoch pass
    pipe.enter_streams()
    for kk in range(args.warmup):
        step(kk)
    if args.graphs:  # capture every group's graph before timing
        for kk in range(min(n_full, args.warmup + args.steps)):
            pipe.step_graph(kk * G)
    pipe.sync_streams()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    # inputs smaller than 2x L2 (126 MB): flush L2 between timed steps and time
    # each step on its own (flush outside the timed spans)
    feat_bytes = g.num_nodes * d * 4
    flush = feat_bytes < 2 * L2_BYTES
    scrub = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda") if flush else None
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    timed_batches = []
    launches0 = pipe.launches
    if True:
        torch.cuda.synchronize()
        if args.nvtx:
            torch.cuda.nvtx.range_push("timed")
        start.record()
        pipe.enter_streams()
        if args.timeline:
            pipe.timeline = []
        for kk in range(args.steps):
            if flush:
                pipe.sync_streams()
                scrub.fill_(float(kk))
                sev[kk][0].record()
                pipe.enter_streams()
            i0, ng = step(args.warmup + kk, gev[kk])
            timed_batches.extend(range(i0, i0 + ng))
            if flush:
                pipe.sync_streams()
                sev[kk][1].record()
        pipe.sync_streams()
        end.record()
        torch.cuda.synchronize()
        if args.nvtx:
            torch.cuda.nvtx.range_pop()
    if world > 1:
        # shared sampling: no rank reuses its sampler buffers (below) while
        # a peer may still be copying its share of the last timed group
        dist.barrier()
    step_ms_local = (sum(a.elapsed_time(b) for a, b in sev) if flush
                     else start.elapsed_time(end))
    if pipe.timeline:
        for name, slot, e0, e1 in pipe.timeline:
            log(f"[timeline] rank {rank} {name:8s} slot {slot} "
                f"{start.elapsed_time(e0):9.3f} -> {start.elapsed_time(e1):9.3f} ms")
        pipe.timeline = None
    if args.serial and not args.graphs:
        gather_ms = sum(a.elapsed_time(b) for a, b in gev)
        for kk in range(args.steps):  # distinct rows per launch, outside the timing
            i0 = ((args.warmup + kk) % n_full) * G
            ng = min(G, nb - i0)
            pipe.plan.fill(pipe.perm, 0, i0, ng)
            smp.run(ng)
            unions.add(smp, ng)
    else:
        # overlapped run: time the gather alone on the same batches (serial),
        # and the group prefetch (NVLink) on its own
        pev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        pf0 = int(pipe.pf_rows.item()) if pipe.prefetch else 0
        for kk in range(args.steps):
            i0 = ((args.warmup + kk) % n_full) * G
            ng = min(G, nb - i0)
            pipe.plan.fill(pipe.perm, 0, i0, ng)
            smp.run(ng)
            unions.add(smp, ng)
            if flush:
                scrub.fill_(float(kk))
            if pipe.prefetch:
                pev[kk][0].record()
                pipe.prefetch_group(ng, smp, 0)
                pev[kk][1].record()
            gev[kk][0].record()
            pipe.gather(ng, i0, prefetched=pipe.prefetch)
            gev[kk][1].record()
        torch.cuda.synchronize()
        gather_ms = sum(a.elapsed_time(b) for a, b in gev)
        if pipe.prefetch:
            prefetch_ms = sum(a.elapsed_time(b) for a, b in pev)
            prefetch_rows = int(pipe.pf_rows.item()) - pf0
    t = torch.tensor([step_ms_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    n_batches = len(timed_batches)
    # our kernels per step: fill_seeds, mark_seeds, a compaction, per level
    # (node_meta, sample_level, a compaction), gather; + the group prefetch
    # (kind bits, union, a compaction, row copy) when it gathers rows (dense
    # groups copy whole shards with cudaMemcpyAsync: no kernels).  A
    # compaction is 2 launches, 3 with a separate chunk scan (large n)
    c = int(_lib.load().rg_bitmap_compact_launches(dg.nwords))
    pf_kernels = 3 + c if pipe.prefetch and getattr(pipe, "pf_mode", "rows") == "rows" else 0
    # shared sampling: two counter signals + a wait per peer for its share
    # and one for its copy of the slot's previous group (copies: copy engine)
    # (+ a compaction per peer share re-deriving its input lists when the
    # bitmaps came over)
    sh_kernels = (2 + 2 * (world - 1) + (world - 1) * c * int(pipe._window_gather(G))
                  if getattr(pipe, "shared", False) else 0)
    gpu_launches = args.steps * (3 + c + smp.L * (2 + c) + pf_kernels + sh_kernels)

    env_sweep = None
    if args.env_sweep:  # diagnostic: the same timed loop under other library knobs
        env_sweep = {}
        for setting in args.env_sweep.split(";"):
            saved = dict(os.environ)
            for kv in filter(None, setting.split(",")):
                key, val = kv.split("=", 1)
                os.environ[key] = val
            pipe.enter_streams()
            for kk in range(2):
                step(kk)
            pipe.sync_streams()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            start.record()
            pipe.enter_streams()
            for kk in range(args.steps):
                step(args.warmup + kk)
            pipe.sync_streams()
            end.record()
            torch.cuda.synchronize()
            tt = torch.tensor([start.elapsed_time(end)], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
            env_sweep[setting] = {"ms_per_step": ms / args.steps,
                                  "batches_per_s": world * args.steps * G / (ms / 1e3)}
            log(f"[bench] env {setting}: {env_sweep[setting]}")
            os.environ.clear()
            os.environ.update(saved)

    # full-epoch accounting pass (remote rows/epoch, parity metric)
    pipe.start_epoch(sched, 0)
    eev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    eev[0].record()
    for i0 in range(0, nb, G):
        ng = min(G, nb - i0)
        pipe.plan.fill(pipe.perm, 0, i0, ng)
        smp.run(ng)
        pipe.gather(ng, i0)
    eev[1].record()
    torch.cuda.synchronize()
    clk.__exit__()
    epoch_ms = eev[0].elapsed_time(eev[1])
    tot = pipe.totals()
    per_batch = tot["per_batch"]
    rows_b = per_batch[:, 0] + per_batch[:, 1] + per_batch[:, 2]
    timed_rows = int(sum(rows_b[i] for i in timed_batches))
    peer_rows = int(sum(per_batch[i, 5] for i in timed_batches))

    # roofline of the dominant kernel (bundle gather): read + write every row,
    # plus the id and route word per row
    peak, peak_src = peaks()
    # per batch: read + write every row + its id and route word
    gather_bytes = timed_rows * (2 * 4 * d + 8)
    # per launch: every bundle row written once, every distinct source row of
    # the group read once (the group's batches share rows, served from L2)
    union_rows = unions.total()
    launch_bytes = timed_rows * (4 * d + 8) + union_rows * 4 * d
    achieved = launch_bytes / (gather_ms / 1e3) / 1e9
    step_bytes = gather_bytes  # sampler bytes reported in DESIGN.md (~3% of the batch)

    # e2e: host seeds in (pinned H2D), accounting out (D2H) per group
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(pipe, g, cfg, args, world)

    result = None
    shared_check = None
    if getattr(pipe, "shared", False):
        if pipe.shared_status():
            raise SystemExit(f"rank {rank}: a shared-sampling wait timed out")
        shared_check = verify_shared(pipe, dist) if args.check else None
    check = run_check(pipe, g, cfg, S0, args.prng) if args.check else None
    if check is not None and shared_check is not None:
        check["shared_sampling_bit_exact"] = shared_check
    if check is not None and pin is not None:
        check["structure_pinned"] = pin
    if check is not None and plan_shared_exact is not None:
        # the epoch's access table from 1/N of the groups per rank + an
        # all-reduce equals the table of a full local plan pass
        check["plan_pass_shared_bit_exact"] = plan_shared_exact
    if check is not None and world > 1:
        flags = torch.tensor([int(check["blocks_bit_exact"] and check["rows_bit_exact"]
                                  and check.get("shared_sampling_bit_exact", True)
                                  and check.get("plan_pass_shared_bit_exact", True))],
                             device="cuda")
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        check["all_ranks_bit_exact"] = bool(flags.item())
    e2e_rows = run_e2e_host_rows(pipe, cfg, args, world) if not args.no_e2e else None
    hot_np = hot.cpu().numpy().astype(np.int64)
    legs = {}
    if world == 1 and not args.no_e2e and not cfg.get("device_features"):
        legs["e2e_dropin"] = run_dropin(g, book, cfg, hot_np, part)
        legs["q_bounded"] = run_group_leg(dg, store, part, train, cfg, hot, 2, 2, 256)
        if args.train_groups:
            legs["e2e_train"] = {
                "overlapped": run_train_leg(dg, store, part, train, cfg, hot, g.labels, 32,
                                            args.train_groups, True),
                "serial": run_train_leg(dg, store, part, train, cfg, hot, g.labels, 32,
                                        args.train_groups, False),
                "overlapped_eager": run_train_leg(dg, store, part, train, cfg, hot, g.labels, 32,
                                                  args.train_groups, True, graphs=False),
                "note": "sample+gather+GraphSAGE step (bit-exact aggregation, fp32 cuBLAS "
                        "GEMMs, SGD) per batch; overlapped = GroupProducer thread samples / "
                        "gathers group k+1 on side streams while group k trains; cuda_graphs "
                        "= each (slot, batch) step replayed from a captured graph"}
    if rank == 0 and world == 1 and not args.no_cpu and not cfg.get("device_features"):
        result = cpu_baseline(cpu_state(g, book.owner, cfg, hot_np, part), args.cpu_seconds, nb)

    traffic_b = ncu_traffic("gather_bundle_kernel", args.config, G)
    agg_batches = n_batches * world
    value = agg_batches / (total_ms / 1e3)
    remote_rows = tot["hit"] + tot["fallback"]
    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "batches/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": (f"synthetic: gnnpipe.synth_powerlaw({cfg['n']}, {cfg['m']}, {cfg['d']}, "
                 f"{cfg['classes']}, seed={S0}) reproduced bit-exactly + "
                 f"partition_edgecut(k={k})"),
        "config": workload_config(args, cfg, part, n_hot),
        "batches_per_step": G, "parallelism": f"worker-per-gpu x{world}",
        "l2": ("L2 flushed between timed steps (feature table %.0f MB < 2x L2); "
               "steps timed individually" if flush else
               "inputs larger than L2 (feature shards %.0f MB; bundle %.0f MB/batch)")
              % ((feat_bytes / 1e6,) if flush
                 else (feat_bytes / 1e6, float(rows_b.mean()) * d * 4 / 1e6)),
        "roofline": {"kernel": getattr(pipe, "gather_kernel", "rg_gather_bundle"), "bound": "hbm",
                     "achieved": achieved, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_b,
                     "bytes_per_launch": launch_bytes / args.steps,
                     "union_rows_per_launch": union_rows / args.steps,
                     "bundle_rows_per_launch": timed_rows / args.steps,
                     "ms_per_launch": gather_ms / args.steps,
                     "share_of_step": gather_ms / step_ms_local,
                     "dram_achieved": (traffic_b / (gather_ms / args.steps / 1e3) / 1e9
                                       if traffic_b else None),
                     "dram_frac": (traffic_b / (gather_ms / args.steps / 1e3) / 1e9 / peak
                                   if traffic_b else None),
                     "per_batch_bytes": {
                         "bytes_per_launch": gather_bytes / args.steps,
                         "gbs": gather_bytes / (gather_ms / 1e3) / 1e9,
                         "step_frac": step_bytes / (step_ms_local / 1e3) / 1e9 / peak,
                         "note": "every batch's rows counted as read from HBM (SURVEY.md §8d "
                                 "per-batch figure); the group's shared rows come from L2, so "
                                 "this exceeds the DRAM roofline by design"},
                     "note": ("achieved = the launch's algorithmic bytes / its event-timed "
                              "duration: bundle rows written + ids/routes + each distinct "
                              "source row of the group read once; dram_frac = ncu DRAM bytes "
                              "(traffic, profiles/traffic.json) / the same time")},
        "e2e": e2e,
        "e2e_host_rows": e2e_rows,
        **legs,
        "nvlink": ({"mode": (("group prefetch: the peer shards copied whole on the copy "
                              "engines (dense group, rg_copy_bytes), gather all-local"
                              if getattr(pipe, "pf_mode", "rows") != "rows" else
                              "group prefetch (rg_prefetch_rows): each group's peer rows "
                              "copied once into local shadows, gather all-local")
                             if args.transport == "p2p" else
                             "group prefetch over NCCL all-to-all (ids out, rows back, "
                             "rg_scatter_rows into local shadows), gather all-local"),
                    "transport": args.transport,
                    "prefetched_rows_per_group": prefetch_rows / args.steps,
                    "prefetched_rows_per_batch": prefetch_rows / max(1, n_batches),
                    "bytes_per_batch": prefetch_rows * 4 * d / max(1, n_batches),
                    "achieved_gbs": prefetch_rows * 4 * d / (prefetch_ms / 1e3) / 1e9,
                    "prefetch_ms_per_step": prefetch_ms / args.steps,
                    "peer_copy_ref_gbs": 770.0,
                    "note": ("peer-shard payload bytes copied over NVLink by the group "
                             "prefetch, timed alone; 770 GB/s = measured peer copy per "
                             "direction (B200_PROFILING.md)" if args.transport == "p2p" else
                             "NCCL transport: the prefetch time also contains waits for the "
                             "other ranks' matching collectives (ranks drift in the serial "
                             "re-timing loop), so achieved_gbs understates the link")}
                   if world > 1 and pipe.prefetch else
                   {"mode": "per-batch pull",
                    "peer_rows_per_batch": peer_rows / max(1, n_batches),
                    "bytes_per_batch": peer_rows * 4 * d / max(1, n_batches),
                    "achieved_gbs": peer_rows * 4 * d / (gather_ms / 1e3) / 1e9,
                    "peer_copy_ref_gbs": 770.0,
                    "note": "peer-shard payload bytes read by the gather over NVLink, timed "
                            "with the gather alone; 770 GB/s = measured peer copy per "
                            "direction (B200_PROFILING.md)"} if world > 1 else None),
        "gpu_launches": gpu_launches,
        **({"env_sweep": env_sweep} if env_sweep else {}),
        "clocks": clk.summary(),
        "remote_rows_epoch": {"worker": part, "uncached": remote_rows,
                              "fallback": tot["fallback"], "cache_hits": tot["hit"],
                              "rpcs": tot["rpcs"], "reduction": remote_rows / max(1, tot["fallback"]),
                              "bad": tot["bad"], "epoch_ms": epoch_ms, "plan_pass_ms": plan_ms},
        "cpu_baseline": result,
        "check": check,
    }
    emit(line)
    if world > 1:
        dist.destroy_process_group()


def verify_shared(pipe, dist) -> bool:
    """A group produced with shared sampling (this rank sampled its share,
    the peers' shares copied over NVLink) equals the same group sampled
    entirely on this GPU: every batch's whole block (frontiers, counts and
    ELL edges of every level, the input bitmap and its ranks) and its
    bundle rows.  The shared
    group lands in slot 1, the local one in slot 0 (no copies of the
    bundles needed)."""
    import torch

    torch.cuda.synchronize()
    dist.barrier()
    pipe.enter_streams()
    ng = pipe.step_overlapped(0)
    if pipe.last_slot != 1:
        ng = pipe.step_overlapped(0)
    pipe.sync_streams()
    torch.cuda.synchronize()
    dist.barrier()  # every peer finished copying from this rank's buffers
    sh, loc = pipe.samplers[1], pipe.samplers[0]
    pipe.step(0)  # the same group sampled locally into slot 0
    torch.cuda.synchronize()
    L = sh.L
    window = pipe._window_gather(ng)
    nf = loc.nfront[:, :ng].cpu()
    ok = torch.equal(sh.nfront[:, :ng], loc.nfront[:, :ng])
    for b in range(ng):
        n = int(nf[L, b])
        ok = ok and torch.equal(sh.bm[b], loc.bm[b])
        if window:
            ok = ok and torch.equal(sh.wpre[b], loc.wpre[b])
        for d in range(L + 1):  # every level's frontier
            ok = ok and torch.equal(sh.front[d][b, : int(nf[d, b])], loc.front[d][b, : int(nf[d, b])])
        for d in range(L):  # every level's sampled edges (ELL rows up to their counts)
            m, F = int(nf[d, b]), sh.step_fan[d]
            cs, cl = sh.cnt[d][b, :m], loc.cnt[d][b, :m]
            ok = ok and torch.equal(cs, cl)
            live = torch.arange(F, device=cs.device)[None, :] < cl[:, None].long()
            es, el = sh.ell[d][b, : m * F].view(m, F), loc.ell[d][b, : m * F].view(m, F)
            ok = ok and torch.equal(es[live], el[live])
        ok = ok and torch.equal(pipe.row_bufs[1][b, :n], pipe.row_bufs[0][b, :n])
    dist.barrier()
    return bool(ok)


def run_check(pipe, g, cfg, s0, prng="splitmix"):
    """Batch 0 of the epoch against the CPU oracle (the PRNG-variant oracle
    for --prng pcg32/sfc64/xoshiro256pp): frontiers and edges bit-exact;
    bundle rows bit-exact against the feature rows of its input nodes
    (re-generated / read independently of the gather)."""
    import torch

    from oracle import gnn_oracle as orc
    from paper_2505_10806_b200 import _lib
    from paper_2505_10806_b200.sampler import block_from_sampler

    smp = pipe.sampler
    pipe.step(0)
    perm = pipe.perm[: cfg["batch"]].cpu().numpy()
    blk = block_from_sampler(smp, 0, perm, 0, 0)
    t = time.time()
    if prng == "splitmix":
        fr, ed = orc.block(g.indptr, g.indices, perm, cfg["fanouts"], orc.batch_seed(s0, 0, 0))
    else:
        from oracle import prng_oracle

        fr, ed = prng_oracle.block(g.indptr, g.indices, perm, cfg["fanouts"],
                                   orc.batch_seed(s0, 0, 0), prng)
    ok = all(np.array_equal(a, b) for a, b in zip(blk.frontiers, fr))
    ok = ok and all(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
                    for a, b in zip(blk.edges, ed))
    ids = torch.from_numpy(fr[-1].astype(np.int32)).cuda()
    d = cfg["d"]
    if cfg.get("device_features"):
        want = torch.empty((len(ids), pipe.store.src_stride), device="cuda")
        _lib.call("rg_fill_features", ids.data_ptr(), len(ids), d, pipe.store.src_stride, s0,
                  want.data_ptr(), _lib.stream_handle())
        want = want[:, :d]
    else:
        want = torch.from_numpy(g.features[fr[-1]]).cuda()
    rows_ok = bool(torch.equal(pipe.rows[0, : len(ids), :d], want))
    return {"batch": 0, "input_nodes": int(len(fr[-1])), "blocks_bit_exact": bool(ok),
            "rows_bit_exact": rows_ok, "oracle_s": round(time.time() - t, 1)}


def run_dropin(g, book, cfg, hot_np, part, batches: int = 48, warm: int = 6):
    """The reference-facing API end to end: Prefetcher(plan, ...) with the
    worker's shard, a StoreClient over every shard and the steady cache,
    exactly as train.py:208-221 drives it; every bundle's rows are read as
    the numpy array the reference returns (FeatureBundle.rows).  One batch
    per plan.block + assemble_bundle, producer thread Q = 3 ahead."""
    import torch

    import paper_2505_10806_b200 as rg

    k, d = cfg["parts"], cfg["d"]
    owner = np.asarray(book.owner)
    train = np.flatnonzero(g.train_mask)
    shards = [rg.StoreShard(q, np.flatnonzero(owner == q), g.features[owner == q])
              for q in range(k)]
    client = rg.StoreClient(owner, [rg.InprocTransport(s) for s in shards], d)
    cache = rg.build_steady(hot_np, client, rg.TransferAccount())
    plan = rg.generate_plan(g, train, cfg["fanouts"], cfg["batch"], 1, S0, keep_inputs=False,
                            group=cfg.get("group", 32))
    acct = rg.TransferAccount()
    torch.cuda.synchronize()
    pf = rg.Prefetcher(plan, 0, owner, part, shards[part], client, cache, acct, depth=3)
    nbytes = 0
    for _ in range(warm):
        pf.next_bundle().rows
    t = time.perf_counter()
    for _ in range(batches):
        b = pf.next_bundle()
        nbytes += b.rows.nbytes
    wall = time.perf_counter() - t
    pf.drain()
    del shards, client, cache
    torch.cuda.empty_cache()
    return {"value": batches / wall, "unit": "batches/s", "batches": batches,
            "d2h_bytes_per_batch": nbytes / batches,
            "api": "Prefetcher(plan, 0, owner, p, shard, client, cache, account, depth=3): "
                   "plan.block + assemble_bundle per batch on a producer thread, "
                   "FeatureBundle.rows (numpy) read by the consumer"}


def run_group_leg(dg, store, part, train, cfg, hot, group: int, nbuf: int, steps: int):
    """Memory-bounded configuration: G batches per step x nbuf slots live
    bundles (G = 2, nbuf = 2: Q + 1 = 4 bundles, the reference's bound,
    prefetch.py:1-7), overlapped, device-timed."""
    import torch

    from paper_2505_10806_b200.pipeline import WorkerPipeline
    from paper_2505_10806_b200.sampler import SeedSchedule

    pipe = WorkerPipeline(dg, store, part, train, cfg["fanouts"], cfg["batch"], S0, group,
                          nbuf=nbuf)
    pipe.build_cache(hot)
    pipe.start_epoch(SeedSchedule(S0, 1, pipe.nb), 0)
    pipe.enter_streams()
    n_full = pipe.nb // group
    for kk in range(8):
        pipe.step_overlapped((kk % n_full) * group)
    pipe.sync_streams()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record()
    pipe.enter_streams()
    for kk in range(steps):
        pipe.step_overlapped(((8 + kk) % n_full) * group)
    pipe.sync_streams()
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    del pipe
    torch.cuda.empty_cache()
    return {"value": steps * group / (ms / 1e3), "unit": "batches/s", "batches_per_step": group,
            "slots": nbuf, "live_bundles": group * nbuf, "steps": steps}


def run_train_leg(dg, store, part, train, cfg, hot, labels_np, group: int, groups: int,
                  overlap: bool, graphs: bool = True):
    """Consumer attached: every batch sampled + gathered AND trained (the
    device GraphSAGE step of train.py: bit-exact aggregation, cuBLAS fp32
    GEMMs, SGD), `groups` groups of `group` batches.  overlap=True: the
    GroupProducer thread samples/gathers group k+1 on the side streams while
    group k trains (prefetch.py:91-164); False: produce, then train, serially.
    Wall-clock batches/s (the host enqueues the training step)."""
    import torch

    from paper_2505_10806_b200 import model
    from paper_2505_10806_b200.pipeline import GroupProducer, WorkerPipeline
    from paper_2505_10806_b200.sampler import SeedSchedule

    torch.backends.cuda.matmul.allow_tf32 = False
    d = cfg["d"]
    pipe = WorkerPipeline(dg, store, part, train, cfg["fanouts"], cfg["batch"], S0, group,
                          nbuf=2 if overlap else 1)
    pipe.build_cache(hot)
    pipe.start_epoch(SeedSchedule(S0, 1, pipe.nb), 0)
    labels = torch.from_numpy(np.asarray(labels_np)).cuda()
    params = model.init_params(d, 32, cfg["classes"], len(cfg["fanouts"]), 1234)
    loss_sum = torch.zeros((), dtype=torch.float64, device="cuda")
    trainer = model.GraphTrainer(params, labels, d, dg.n, 0.05) if graphs else None

    def train_group(smp, rows_buf, ng, nf, lock=None):
        nonlocal params
        if trainer is not None:
            for b in range(ng):
                trainer.step(smp, rows_buf, b, lock)
            return
        for b in range(ng):
            blk = model.block_from_slot(smp, b, nf[:, b])
            rows = rows_buf[b, : int(nf[smp.L, b]), :d]
            loss, grads = model.loss_and_grad(blk, rows, labels, params)
            params = model.sgd_step(params, grads, 0.05)
            loss_sum.add_(loss.double())

    def epoch_part(starts):
        if overlap:
            prod = GroupProducer(pipe, starts)
            try:
                while (item := prod.next_group()) is not None:
                    i0, ng, slot, nf = item
                    train_group(pipe.samplers[slot], pipe.row_bufs[slot], ng, nf,
                                prod.capture_lock)
                    prod.release(slot)
            finally:
                prod.close()
        else:
            for i0 in starts:
                ng = pipe.step(i0)
                train_group(pipe.sampler, pipe.rows, ng, pipe.sampler.nfront[:, :ng].cpu().numpy())

    n_full = max(1, pipe.nb // pipe.G)
    group = pipe.G
    epoch_part([0])  # warm-up: allocator, cuBLAS handles
    if graphs:  # capture every (slot, batch) graph outside the timing
        epoch_part([group % (n_full * group)] if n_full > 1 else [0])
        if trainer is not None and len(trainer.graphs) < 2 * group:
            epoch_part([0])
    torch.cuda.synchronize()
    t = time.perf_counter()
    starts = [((1 + k) % n_full) * group for k in range(groups)]
    epoch_part(starts)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    loss = float((trainer.loss_sum if trainer is not None else loss_sum).item())
    captures = trainer.captures if trainer is not None else 0
    del pipe, trainer
    torch.cuda.empty_cache()
    return {"value": groups * group / wall, "unit": "batches/s", "batches": groups * group,
            "group": group, "overlap": overlap, "cuda_graphs": graphs, "graph_captures": captures,
            "loss_sum": loss}


def run_e2e_host_rows(pipe, cfg, args, world):
    """Informational: the numpy-facing drop-in returns bundle rows on the
    host, so every batch's rows (the valid |input| x d part of its slot) are
    copied to pinned host memory on a copy stream, through a ring of two
    batch-sized host buffers (a slot is reused once the host has seen the
    copy that filled it).  PCIe-bound; bytes counted exactly."""
    import torch
    import torch.distributed as dist

    G, nb, smp = pipe.G, pipe.nb, pipe.sampler
    d = cfg["d"]
    n_full = max(1, nb // G)
    steps = max(2, min(args.steps, 6))
    host = [torch.empty((pipe.cap_in, d), dtype=torch.float32).pin_memory() for _ in range(2)]
    copy = torch.cuda.Stream()
    done = [torch.cuda.Event(), torch.cuda.Event()]
    ready = torch.cuda.Event()
    nbytes, q = 0, 0
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = time.perf_counter()
    for kk in range(steps):
        i0 = (kk % n_full) * G
        pipe.step(i0)
        nf = smp.nfront[smp.L, :G].cpu().numpy()
        ready.record()
        for b in range(G):
            slot = q % 2
            q += 1
            done[slot].synchronize()  # the host has the previous contents
            n = int(nf[b])
            with torch.cuda.stream(copy):
                copy.wait_event(ready)
                host[slot][:n].copy_(pipe.rows[b, :n, :d], non_blocking=True)
                done[slot].record(copy)
            nbytes += n * d * 4
        torch.cuda.current_stream().wait_stream(copy)  # rows buffer reused next step
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    tt = torch.tensor([wall], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return {"value": steps * G * world / float(tt.item()), "unit": "batches/s",
            "d2h_bytes_per_step": nbytes / steps, "steps": steps,
            "api": "bundle rows to pinned host memory every step (numpy drop-in layout), "
                   "2-batch pinned ring"}


def run_e2e(pipe, g, cfg, args, world):
    """Public pipeline API with host buffers: each step copies the group's
    seed ids + batch seeds from pinned host memory (H2D), samples and
    gathers, and reads the per-batch accounting back (D2H, host-visible
    before the next step).  The bundle rows stay in HBM for the on-device
    consumer (model.py's aggregation), as in a GPU training loop."""
    import torch
    import torch.distributed as dist

    from paper_2505_10806_b200.sampler import SeedSchedule, seed_for

    G, nb, smp = pipe.G, pipe.nb, pipe.sampler
    sched = SeedSchedule(S0, 1, nb)
    B = cfg["batch"]
    perm = pipe.perm.cpu().numpy()
    n_full = max(1, nb // G)
    seeds_h = torch.zeros((n_full, G, smp.caps[0]), dtype=torch.int32).pin_memory()
    nseeds_h = torch.zeros((n_full, G), dtype=torch.int32).pin_memory()
    rng_h = torch.zeros((n_full, G), dtype=torch.int64).pin_memory()
    for s in range(n_full):
        for b in range(G):
            i = s * G + b
            chunk = perm[i * B:(i + 1) * B]
            seeds_h[s, b, :len(chunk)] = torch.from_numpy(chunk.astype(np.int32))
            nseeds_h[s, b] = len(chunk)
            rng_h[s, b] = int(np.uint64(seed_for(sched, 0, i)).astype(np.int64))
    out_h = torch.zeros((G, 8), dtype=torch.int32).pin_memory()
    overlapped = not args.serial and not args.graphs
    ring = [torch.zeros((G, 8), dtype=torch.int32).pin_memory() for _ in range(2)]
    ring_ev = [torch.cuda.Event() for _ in range(2)]
    pending = []

    def one_overlapped(kk):
        """Prefetcher-style: group kk's seeds go H2D and its sample/gather
        are enqueued, then group kk-1's accounting (enqueued D2H behind its
        gather) is read on the host."""
        s = kk % n_full
        i0 = s * G
        pipe.step_overlapped(i0, (seeds_h[s], nseeds_h[s], rng_h[s]))
        r = kk % 2
        with torch.cuda.stream(pipe.s_gather):
            ring[r].copy_(pipe.counters[i0:i0 + G], non_blocking=True)
            ring_ev[r].record(pipe.s_gather)
        pending.append(r)
        got = 0
        while len(pending) > 1:
            q = pending.pop(0)
            ring_ev[q].synchronize()
            got += int(ring[q][:, 2].sum())
        return got

    def drain():
        while pending:
            q = pending.pop(0)
            ring_ev[q].synchronize()

    def one(kk):
        if overlapped:
            return one_overlapped(kk)
        s = kk % n_full
        i0 = s * G
        smp.seeds.copy_(seeds_h[s], non_blocking=True)
        smp.nseeds.copy_(nseeds_h[s], non_blocking=True)
        smp.rng.copy_(rng_h[s], non_blocking=True)
        smp.run(G)
        pipe.gather(G, i0)
        out_h.copy_(pipe.counters[i0:i0 + G], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return int(out_h[:, 2].sum())

    if overlapped:
        pipe.enter_streams()
    for kk in range(args.warmup):
        one(kk)
    drain()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = time.perf_counter()
    for kk in range(args.steps):
        one(args.warmup + kk)
    drain()  # the last group's accounting is on the host inside the timed region
    wall = time.perf_counter() - t
    if overlapped:
        pipe.sync_streams()
    tt = torch.tensor([wall], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    wall = float(tt.item())
    h2d = G * smp.caps[0] * 4 + G * 4 + G * 8
    d2h = G * 8 * 4
    return {"value": args.steps * G * world / wall, "unit": "batches/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": "WorkerPipeline: seeds from pinned host, accounting read back per step"
                   + (" (prefetcher-style: step k's read-back after step k+1 is enqueued)"
                      if overlapped else "")}


if __name__ == "__main__":
    main()
