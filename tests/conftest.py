"""Shared fixtures.  GPU tests carry @pytest.mark.gpu; the CPU suite
(pytest -m "not gpu") checks the oracle against the reference's goldens,
the native host code, the ABI surface and the host-side logic."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: multi-second CPU test")


@pytest.fixture(scope="session")
def golden() -> dict:
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def small_npz():
    return np.load(GOLDEN / "small.npz")


class HostGraph:
    """Minimal graph record built from the golden arrays (no device)."""

    def __init__(self, z):
        self.indptr = z["indptr"]
        self.indices = z["indices"]
        self.features = z["features"]
        self.labels = z["labels"]
        self.train_mask = z["train_mask"]
        self.num_nodes = len(self.indptr) - 1
        self.num_edges = len(self.indices)
        self.feat_dim = self.features.shape[1]


@pytest.fixture(scope="session")
def small_graph_arrays(small_npz):
    return HostGraph(small_npz)


def case_names(golden):
    return [c["name"] for c in golden["sample_cases"]]


def load_case(z, golden, name):
    meta = next(c for c in golden["sample_cases"] if c["name"] == name)
    L = meta["layers"]
    fr = [z[f"case_{name}_front{d}"] for d in range(L + 1)]
    ed = [(z[f"case_{name}_src{d}"], z[f"case_{name}_dst{d}"]) for d in range(L)]
    return meta, z[f"case_{name}_seeds"], fr, ed


def fixture_graph(kind: str):
    """The hand-built graphs of the reference's conftest (conftest.py:31-50)."""
    from paper_2505_10806_b200.graph import from_edge_list

    if kind == "star":
        return from_edge_list(21, [(0, i) for i in range(1, 21)])
    if kind == "path":
        return from_edge_list(3, [(0, 1), (1, 2)])
    if kind == "iso":
        return from_edge_list(4, [(0, 1)])
    raise KeyError(kind)
