"""End-to-end runner on the device (train.py:1-329 of the reference).

Same RunConfig fields, the same MetricsRecord CSV (train.py:34-89) and the
same per-worker epoch loop (train.py:171-264): plan (device plan pass) ->
per-worker hot set (n_hot = int(#remote * pct / 100), epoch or global
scope) -> per epoch: cache fill / swap, every batch sampled + gathered on
the GPU (G batches per launch group), trained with the device GraphSAGE
step, then full-graph evaluation.  Accounting columns are bit-exact with the
reference; loss / accuracy agree to GEMM rounding.

Workers are replicas of one data path (train.py:291-311): they run one
after the other on this GPU (or one per GPU under bench.py / torchrun).
"""

from __future__ import annotations

import csv
import threading
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import model
from .engine import DeviceGraph, FeatureStore
from .graph import load_graph, synth_powerlaw
from .partition import (halo_expand, load_partition, partition_edgecut,
                        partition_random)
from .pipeline import GroupProducer, WorkerPipeline, resolve_n_hot
from .plan import candidates, generate_plan
from .rng import mix64
from .sampler import SeedSchedule

CSV_HEADER = [
    "epoch", "mode", "t_e_ms", "rpc_calls", "nodes_pulled", "bytes_pulled",
    "cache_hits", "cache_misses", "reuse_ratio", "loss", "train_acc",
]
_PARAM_SEED_TAG = 0x70617261  # train.py:39


@dataclass
class MetricsRecord:
    epoch: int
    mode: str
    t_e_ms: float
    rpc_calls: int
    nodes_pulled: int
    bytes_pulled: int
    cache_hits: int
    cache_misses: int
    reuse_ratio: float | None
    loss: float
    train_acc: float


def write_metrics(records: list[MetricsRecord], path) -> None:
    """CSV with the fixed header; reuse_ratio empty when undefined (train.py:57-68)."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(CSV_HEADER)
        for r in records:
            w.writerow([r.epoch, r.mode, repr(r.t_e_ms), r.rpc_calls, r.nodes_pulled,
                        r.bytes_pulled, r.cache_hits, r.cache_misses,
                        "" if r.reuse_ratio is None else repr(r.reuse_ratio), repr(r.loss),
                        repr(r.train_acc)])


def read_metrics(path) -> list[MetricsRecord]:
    with open(path, newline="") as f:
        return [MetricsRecord(
            epoch=int(r["epoch"]), mode=r["mode"], t_e_ms=float(r["t_e_ms"]),
            rpc_calls=int(r["rpc_calls"]), nodes_pulled=int(r["nodes_pulled"]),
            bytes_pulled=int(r["bytes_pulled"]), cache_hits=int(r["cache_hits"]),
            cache_misses=int(r["cache_misses"]),
            reuse_ratio=None if r["reuse_ratio"] == "" else float(r["reuse_ratio"]),
            loss=float(r["loss"]), train_acc=float(r["train_acc"])) for r in csv.DictReader(f)]


@dataclass
class RunConfig:
    graph_path: str | None = None
    gen_nodes: int = 20000
    gen_edges_per_node: int = 5
    feat_dim: int = 32
    num_classes: int = 8
    partitions: int = 2
    partitioner: str = "edgecut"
    partition_path: str | None = None
    s0: int = 7
    epochs: int = 5
    batch_size: int = 512
    fanouts: list[int] = field(default_factory=lambda: [10, 25])
    n_hot: int | None = None
    n_hot_pct: float = 15.0
    hot_scope: str = "epoch"
    prefetch_depth: int = 3
    mode: str = "rapid"
    latency_ms: float = 0.0
    transport: str = "inproc"
    lr: float = 0.05
    hidden_dim: int = 32
    num_layers: int = 2
    precision: str = "f32"
    metrics_out: str | None = None
    dump_cache_keys: bool = False
    # B200 additions
    prng: str = "splitmix"
    group: int = 16
    overlap: bool = True  # sample+gather group k+1 while group k trains (GroupProducer)
    cuda_graphs: bool = True  # replay each slot/batch training step from a CUDA graph

    def validate(self) -> None:
        """train.py:121-135."""
        if self.mode not in ("baseline", "rapid"):
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.hot_scope not in ("epoch", "global"):
            raise ValueError(f"unknown hot scope {self.hot_scope!r}")
        if self.partitioner not in ("random", "edgecut"):
            raise ValueError(f"unknown partitioner {self.partitioner!r}")
        if self.transport not in ("inproc", "tcp"):
            raise ValueError(f"unknown transport {self.transport!r}")
        if self.prefetch_depth < 1:
            raise ValueError("prefetch depth must be >= 1")
        if self.precision not in ("f32", "f64"):
            raise ValueError(f"unknown precision {self.precision!r}")
        if len(self.fanouts) != self.num_layers:
            raise ValueError("fanouts must list one value per layer")


@dataclass
class WorkerResult:
    part: int
    records: list[MetricsRecord]
    params: list
    plan_digest: str
    cache_keys: np.ndarray | None = None
    cache_fill: tuple = (0, 0, 0)


def _graph_and_book(cfg: RunConfig):
    """train.py:148-162: RGF1 file or generator; RPB1 file or partitioner."""
    g = (load_graph(cfg.graph_path) if cfg.graph_path else
         synth_powerlaw(cfg.gen_nodes, cfg.gen_edges_per_node, cfg.feat_dim, cfg.num_classes,
                        cfg.s0))
    if cfg.partition_path:
        book = load_partition(cfg.partition_path)
    elif cfg.partitioner == "random":
        book = partition_random(g, cfg.partitions, cfg.s0)
    else:
        book = partition_edgecut(g, cfg.partitions)
    return g, halo_expand(g, book)


def run(cfg: RunConfig) -> list[WorkerResult]:
    """Execute every partition's worker; write the per-worker CSVs."""
    cfg.validate()
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False  # fp32 GEMMs, as numpy
    try:
        return _run(cfg)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32


def _run(cfg: RunConfig) -> list[WorkerResult]:
    g, book = _graph_and_book(cfg)
    dtype = torch.float32 if cfg.precision == "f32" else torch.float64
    owner = np.asarray(book.owner)
    k = int(book.k)
    dg = DeviceGraph.of(g)
    store = FeatureStore(owner, k, g.feat_dim)
    shard_ids = [np.flatnonzero(owner == q) for q in range(k)]
    for q in range(k):
        store.set_shard(q, FeatureStore.pad_rows(g.features[shard_ids[q]], store.src_stride,
                                                 dg.device))
    store.build_route(shard_ids)
    train = np.flatnonzero(g.train_mask)
    full = model.FullGraph(g, dtype=dtype)
    labels = full.labels
    rapid = cfg.mode == "rapid"
    results = []
    counts = None
    for p in range(k):
        pipe = WorkerPipeline(dg, store, p, train, cfg.fanouts, cfg.batch_size, cfg.s0,
                              cfg.group, nbuf=2 if cfg.overlap else 1, prng=cfg.prng)
        nb = pipe.nb
        sched = SeedSchedule(cfg.s0, cfg.epochs, nb)
        if counts is None:  # the plan pass (and its digest) is shared by all workers
            keep = nb * cfg.epochs * cfg.batch_size <= 2_000_000  # host input sets: small runs
            plan = generate_plan(g, train, cfg.fanouts, cfg.batch_size, cfg.epochs, cfg.s0,
                                 keep_inputs=keep, group=cfg.group, prng=cfg.prng)
            digest = plan.digest_hex() if keep else ""
            counts = plan.counts
            counts_all = plan.counts_all()
        max_count = max(1, nb * cfg.epochs)
        params = model.init_params(g.feat_dim, cfg.hidden_dim, g.num_classes, cfg.num_layers,
                                   mix64(cfg.s0 ^ _PARAM_SEED_TAG), dtype=dtype)
        n_hot = 0
        if rapid and cfg.epochs > 0:
            _, nout, _, _ = candidates(counts_all, store.owner, p, max_count)
            n_hot = cfg.n_hot if cfg.n_hot is not None else resolve_n_hot(cfg.n_hot_pct,
                                                                           int(nout.item()))
        fill = [0, 0, 0]
        hits_acc = misses_acc = 0
        records = []
        cache_keys = None
        secondary = None  # (thread, result dict) building epoch e+1's cache
        trainer = (model.GraphTrainer(params, labels, g.feat_dim, g.num_nodes, cfg.lr)
                   if cfg.cuda_graphs else None)
        for e in range(cfg.epochs):
            t0 = time.perf_counter()
            if rapid and (cfg.hot_scope == "epoch" or e == 0):
                if secondary is not None:  # cache.py:106-129: join, swap
                    secondary[0].join()
                    if "error" in secondary[1]:
                        raise secondary[1]["error"]
                    hot, cache = secondary[1]["hot"], secondary[1]["cache"]
                    pipe.cache = cache
                    secondary = None
                else:
                    scope = counts[e] if cfg.hot_scope == "epoch" else counts_all
                    hot = pipe.select_hot(scope, n_hot, max_count)
                    cache = pipe.build_cache(hot)
                if cache.fill[1]:
                    fill = [fill[0] + cache.fill[0], fill[1] + cache.fill[1],
                            fill[2] + 4 * g.feat_dim * cache.fill[1]]
                if e == 0 and cfg.dump_cache_keys:
                    cache_keys = hot.cpu().numpy().astype(np.int64)
            if rapid and cfg.hot_scope == "epoch" and e + 1 < cfg.epochs:
                secondary = _start_secondary(pipe, counts[e + 1], n_hot, max_count)
            pipe.start_epoch(sched, e)
            loss_sum = torch.zeros((), dtype=torch.float64, device=dg.device)
            if trainer is not None:
                loss_sum = trainer.loss_sum.clone()

            def train_group(smp, rows_buf, ng, nf, lock=None):
                nonlocal params
                if trainer is not None:
                    for b in range(ng):
                        trainer.step(smp, rows_buf, b, lock)
                    return
                for b in range(ng):
                    blk = model.block_from_slot(smp, b, nf[:, b])
                    rows = rows_buf[b, : int(nf[smp.L, b]), : g.feat_dim]
                    if dtype != torch.float32:
                        rows = rows.to(dtype)
                    loss, grads = model.loss_and_grad(blk, rows, labels, params)
                    params = model.sgd_step(params, grads, cfg.lr)
                    loss_sum.add_(loss.double())

            starts = range(0, nb, pipe.G)
            if cfg.overlap:
                # rapid: the producer thread sleeps the injected latency (hidden
                # behind training, prefetch.py:116-132); baseline pulls inline
                # in the worker (train.py:223-230), so its latency is not hidden
                prod = GroupProducer(pipe, starts, cfg.latency_ms if rapid else 0.0)
                try:
                    while (item := prod.next_group()) is not None:
                        i0, ng, slot, nf = item
                        if not rapid and cfg.latency_ms > 0:
                            _sleep_rpcs(pipe, i0, ng, cfg.latency_ms)
                        train_group(pipe.samplers[slot], pipe.row_bufs[slot], ng, nf,
                                    prod.capture_lock)
                        prod.release(slot)
                finally:
                    prod.close()
            else:
                smp = pipe.sampler
                for i0 in starts:
                    ng = pipe.step(i0)
                    nf = smp.nfront[:, :ng].cpu().numpy()
                    if cfg.latency_ms > 0:
                        _sleep_rpcs(pipe, i0, ng, cfg.latency_ms)
                    train_group(smp, pipe.rows, ng, nf)
            if trainer is not None:
                loss_sum = trainer.loss_sum - loss_sum
                params = trainer.params
            if secondary is not None:
                secondary[0].join()  # the epoch includes the wait (train.py:233)
            t = pipe.totals()
            nodes = t["fallback"]
            if rapid:
                if cfg.hot_scope == "epoch":
                    hits, misses = t["hit"], t["fallback"]
                else:
                    hits_acc += t["hit"]
                    misses_acc += t["fallback"]
                    hits, misses = hits_acc, misses_acc
                reuse = hits / (hits + misses) if hits + misses else None
            else:
                hits, misses = 0, nodes
                reuse = 0.0 if misses else None
            t_e_ms = (time.perf_counter() - t0) * 1000.0
            acc = full.evaluate(params, g.train_mask)
            records.append(MetricsRecord(
                epoch=e, mode=cfg.mode, t_e_ms=t_e_ms, rpc_calls=t["rpcs"], nodes_pulled=nodes,
                bytes_pulled=4 * g.feat_dim * nodes, cache_hits=hits, cache_misses=misses,
                reuse_ratio=reuse, loss=float(loss_sum.item()) / nb if nb else float("nan"),
                train_acc=acc if acc is not None else float("nan")))
        results.append(WorkerResult(part=p, records=records, params=params,
                                    plan_digest=digest, cache_keys=cache_keys,
                                    cache_fill=tuple(fill)))
    if cfg.metrics_out:
        for r in results:
            write_metrics(r.records, worker_metrics_path(cfg.metrics_out, r.part))
    return results


def _start_secondary(pipe: WorkerPipeline, counts: torch.Tensor, n_hot: int, max_count: int):
    """Build the next epoch's cache (top_hot of its access counts, then the
    VectorPull) on a background thread and its own stream while the current
    epoch runs (cache.py:80-104); joined and swapped at the epoch boundary."""
    out: dict = {}
    dev = torch.cuda.current_device()
    ready = torch.cuda.Event()
    ready.record()  # counts / store are complete on the caller's stream

    def build():
        try:
            torch.cuda.set_device(dev)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                stream.wait_event(ready)
                hot = pipe.select_hot(counts, n_hot, max_count)
                out["cache"] = pipe.make_cache(hot)
                out["hot"] = hot
            stream.synchronize()
        except BaseException as exc:  # re-raised by the epoch loop
            out["error"] = exc

    t = threading.Thread(target=build, daemon=True)
    t.start()
    return t, out


def _sleep_rpcs(pipe: WorkerPipeline, i0: int, ng: int, latency_ms: float) -> None:
    """Injected per-request latency (store.py:73-74) for the group's fallback
    pulls, slept on the calling thread."""
    masks = pipe.counters[i0:i0 + ng, 3].cpu().numpy().view(np.uint32)
    rpcs = sum(bin(int(m)).count("1") for m in masks)
    time.sleep(latency_ms * rpcs / 1000.0)


def worker_metrics_path(path: str, part: int) -> str:
    """out.csv -> out.w0.csv (train.py:324-329)."""
    if "." in path.rsplit("/", 1)[-1]:
        stem, ext = path.rsplit(".", 1)
        return f"{stem}.w{part}.{ext}"
    return f"{path}.w{part}"
