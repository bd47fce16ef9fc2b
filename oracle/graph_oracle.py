"""CPU ORACLE — test infrastructure, not product code.

The reference's input graphs without the product library: gnnpipe's
synth_powerlaw (graph.py:133-216) and partition_edgecut (partition.py:37-77)
from the plain-C restatement oracle/oracle_graph.c (built by oracle/Makefile
into oracle/_build/liboracle_graph.so), with numpy continuing the Philox
stream for the features and the masks exactly as the reference does.  Used
by bench.py's reference arm / CPU baseline and pinned by tests to the
reference's own content hashes (tests/golden/golden.json "generator").
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

from . import gnn_oracle as orc

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle_graph.so"
_lib = None


def build() -> Path:
    src = HERE / "oracle_graph.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = ctypes.CDLL(str(LIB))
        P, I64, U64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32
        lib.oracle_synth_powerlaw_csr.argtypes = [I64, I64, U64, U64, P, P, P]
        lib.oracle_partition_edgecut.argtypes = [I64, P, P, I32, P]
        _lib = lib
    return _lib


class OracleGraph:
    """The fields of gnnpipe.graph.Graph the data path reads."""

    def __init__(self, indptr, indices, features, train_mask, val_mask, test_mask):
        self.num_nodes = len(indptr) - 1
        self.num_edges = len(indices)
        self.indptr, self.indices = indptr, indices
        self.features = features
        self.feat_dim = features.shape[1]
        self.train_mask, self.val_mask, self.test_mask = train_mask, val_mask, test_mask


def synth_powerlaw(n: int, m: int, feat_dim: int, seed: int,
                   with_features: bool = True) -> OracleGraph:
    """CSR (indices int32), features, train mask of synth_powerlaw(n, m, d, ., seed)."""
    bitgen = np.random.Philox(seed)
    key = bitgen.state["state"]["key"]
    indptr = np.empty(n + 1, dtype=np.int64)
    indices = np.empty(2 * m * (n - m), dtype=np.int32)
    st = np.zeros(13, dtype=np.uint64)
    rc = _load().oracle_synth_powerlaw_csr(n, m, int(key[0]), int(key[1]), indptr.ctypes.data,
                                           indices.ctypes.data, st.ctypes.data)
    if rc != 0:
        raise ValueError(f"oracle_synth_powerlaw_csr failed ({rc})")
    bitgen.state = {"bit_generator": "Philox",
                    "state": {"counter": st[0:4].copy(), "key": st[4:6].copy()},
                    "buffer": st[6:10].copy(), "buffer_pos": int(st[10]),
                    "has_uint32": int(st[11]), "uinteger": int(st[12])}
    rng = np.random.Generator(bitgen)
    features = (rng.standard_normal((n, feat_dim), dtype=np.float32) if with_features
                else np.zeros((n, 0), dtype=np.float32))
    # masks: shuffled(arange(n), mix64(seed ^ "mask")), first 70 % train (graph.py:201-206)
    master = orc.mix(orc.mix(seed ^ 0x6D61736B))
    perm = np.argsort(orc.counter_stream(master, n), kind="stable")
    n_train, n_val = int(0.70 * n), int(0.15 * n)
    masks = [np.zeros(n, dtype=bool) for _ in range(3)]
    masks[0][perm[:n_train]] = True
    masks[1][perm[n_train:n_train + n_val]] = True
    masks[2][perm[n_train + n_val:]] = True
    return OracleGraph(indptr, indices, features, *masks)


def partition_edgecut(g: OracleGraph, k: int) -> np.ndarray:
    """owner int64[n] of partition_edgecut(g, k)."""
    owner = np.empty(g.num_nodes, dtype=np.int64)
    rc = _load().oracle_partition_edgecut(g.num_nodes, g.indptr.ctypes.data,
                                          np.ascontiguousarray(g.indices, np.int32).ctypes.data,
                                          k, owner.ctypes.data)
    if rc != 0:
        raise ValueError(f"oracle_partition_edgecut failed ({rc})")
    return owner
