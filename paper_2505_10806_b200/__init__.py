"""B200-native drop-in for the RapidGNN data path (gnnpipe's sampler /
plan / cache / store / prefetch API, reference gnnpipe/__init__.py:5-19).

The module names and signatures follow the reference; the work runs in the
sm_100a kernels of librapidgnn_b200.so (C ABI: include/rapidgnn_b200.h).
Importing the package needs only the built library; device entry points
raise if no B200 is present (there is no CPU fallback).
"""

from .graph import Graph, from_edge_list, load_graph, save_graph, synth_powerlaw
from .partition import (PartitionBook, halo_expand, load_partition, partition_edgecut,
                        partition_random, save_partition)
from .sampler import ComputationBlock, SeedSchedule, epoch_batches, sample_block, seed_for
from .plan import BatchPlan, FrequencyTable, collect_access, generate_plan, top_hot
from .store import (InprocTransport, LookupError_, StoreClient, StoreShard, TransferAccount,
                    TransportError, bytes_for)
from .cache import CacheLookup, FeatureCache, build_steady
from .prefetch import FeatureBundle, PrefetchError, Prefetcher, assemble_bundle
from .train import MetricsRecord, RunConfig, read_metrics, run, write_metrics

__all__ = [
    "Graph", "from_edge_list", "load_graph", "save_graph", "synth_powerlaw",
    "PartitionBook", "halo_expand", "load_partition", "partition_edgecut", "partition_random",
    "save_partition",
    "ComputationBlock", "SeedSchedule", "epoch_batches", "sample_block", "seed_for",
    "BatchPlan", "FrequencyTable", "collect_access", "generate_plan", "top_hot",
    "InprocTransport", "LookupError_", "StoreClient", "StoreShard", "TransferAccount",
    "TransportError", "bytes_for",
    "CacheLookup", "FeatureCache", "build_steady",
    "FeatureBundle", "PrefetchError", "Prefetcher", "assemble_bundle",
    "MetricsRecord", "RunConfig", "read_metrics", "run", "write_metrics",
]
