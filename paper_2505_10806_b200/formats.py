"""RGF1 / RPB1 containers straight to the device.

The reference's loaders (graph.py:219-290, partition.py:97-119) parse the
files into numpy arrays; the data path then needs them in HBM.  Here the
file is memory-mapped, each section streamed through one reused pinned
staging buffer into its device tensor (chunked, copies async on a side
stream, double-buffered so the host fill of chunk i+1 overlaps the H2D of
chunk i), and converted / validated on the device: u64 neighbour ids become
the int32 CSR the kernels read, u32 labels int64, u8 masks bool, and the
reference's checks (indptr endpoints and monotonicity, neighbour range,
disjoint masks) run as device reductions.  Errors are the reference's:
GraphFormatError (bad magic / version / header), OSError (truncated),
GraphValidationError (invalid contents).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .engine import DeviceGraph
from .graph import RGF1_MAGIC, RGF1_VERSION, GraphFormatError, GraphValidationError

_HEADER = struct.Struct("<4sIQQII")  # magic, version, nodes, edges, dim, classes
_RPB_HEADER = struct.Struct("<4sIQ")  # magic, k, nodes
RPB1_MAGIC = b"RPB1"
_CHUNK = 64 << 20  # bytes per staged copy


@dataclass
class DeviceGraphData:
    """An RGF1 graph resident in HBM: the CSR the kernels read, plus features,
    labels and masks as device tensors."""

    graph: DeviceGraph
    features: torch.Tensor  # float32 [n, d]
    labels: torch.Tensor  # int64 [n]
    train_mask: torch.Tensor  # bool [n]
    val_mask: torch.Tensor
    test_mask: torch.Tensor
    num_classes: int

    @property
    def num_nodes(self) -> int:
        return self.graph.n

    @property
    def feat_dim(self) -> int:
        return int(self.features.shape[1])


class _Stager:
    """Host -> device copies of byte ranges of a mapped file through two
    pinned buffers on a side stream."""

    def __init__(self, device):
        self.device = device
        self.bufs = [torch.empty(_CHUNK, dtype=torch.uint8).pin_memory() for _ in range(2)]
        self.done = [torch.cuda.Event(), torch.cuda.Event()]
        self.stream = torch.cuda.Stream(device=device)
        self.k = 0

    def copy(self, src: np.ndarray, dst: torch.Tensor) -> None:
        """dst (device, contiguous) <- the bytes of src (host, any layout)."""
        raw = src.reshape(-1).view(np.uint8)
        out = dst.view(-1).view(torch.uint8)
        if raw.size != out.numel():
            raise ValueError("staging size mismatch")
        for off in range(0, raw.size, _CHUNK):
            n = min(_CHUNK, raw.size - off)
            slot = self.k % 2
            self.k += 1
            self.done[slot].synchronize()  # the previous copy out of this buffer finished
            np.copyto(self.bufs[slot].numpy()[:n], raw[off:off + n])
            with torch.cuda.stream(self.stream):
                out[off:off + n].copy_(self.bufs[slot][:n], non_blocking=True)
                self.done[slot].record(self.stream)

    def finish(self) -> None:
        torch.cuda.current_stream(self.device).wait_stream(self.stream)


def load_graph_device(path, device=None) -> DeviceGraphData:
    """Read an RGF1 file (graph.py:219-290 layout) into HBM."""
    device = torch.device(device or "cuda")
    path = Path(path)
    size = path.stat().st_size
    if size < _HEADER.size:
        raise GraphFormatError("file too short for RGF1 header")
    with open(path, "rb") as f:
        magic, version, n, e, d, c = _HEADER.unpack(f.read(_HEADER.size))
    if magic != RGF1_MAGIC:
        raise GraphFormatError(f"bad magic {bytes(magic)!r}")
    if version != RGF1_VERSION:
        raise GraphFormatError(f"unsupported version {version}")
    need = _HEADER.size + 8 * (n + 1) + 8 * e + 4 * n * d + 4 * n + 3 * n
    if size < need:
        raise OSError("truncated RGF1 payload")
    if n >= 2**31 - 1:
        raise NotImplementedError("node ids must fit in int32")
    mm = np.memmap(path, dtype=np.uint8, mode="r", offset=0, shape=(need,))
    off = _HEADER.size

    def section(dtype, count):
        nonlocal off
        nbytes = np.dtype(dtype).itemsize * count
        a = mm[off:off + nbytes].view(dtype)
        off += nbytes
        return a

    st = _Stager(device)
    indptr = torch.empty(n + 1, dtype=torch.int64, device=device)
    st.copy(section("<u8", n + 1), indptr)  # u64 bits as int64
    idx64 = torch.empty(e, dtype=torch.int64, device=device)
    st.copy(section("<u8", e), idx64)
    features = torch.empty((n, d), dtype=torch.float32, device=device)
    st.copy(section("<f4", n * d), features)
    lab32 = torch.empty(n, dtype=torch.int32, device=device)
    st.copy(section("<u4", n), lab32)
    masks = torch.empty((3, n), dtype=torch.uint8, device=device)
    st.copy(section("<u1", 3 * n), masks)
    st.finish()
    # the reference's validation (graph.py:59-80), on the device
    if int(indptr[0]) != 0 or int(indptr[-1]) != e:
        raise GraphValidationError("indptr endpoints do not match edge count")
    if n and bool((indptr[1:] < indptr[:-1]).any()):
        raise GraphValidationError("indptr is not nondecreasing")
    if e and (bool((idx64 < 0).any()) or bool((idx64 >= n).any())):
        raise GraphValidationError("neighbor id out of range")
    mb = masks.bool()
    if bool(((mb[0] & mb[1]) | (mb[0] & mb[2]) | (mb[1] & mb[2])).any()):
        raise GraphValidationError("train/val/test masks overlap")
    indices = idx64.to(torch.int32)
    del idx64
    dg = DeviceGraph.from_device(indptr, indices, n)
    return DeviceGraphData(graph=dg, features=features, labels=lab32.to(torch.int64),
                           train_mask=mb[0], val_mask=mb[1], test_mask=mb[2], num_classes=c)


def load_partition_device(path, device=None) -> tuple[int, torch.Tensor]:
    """RPB1 (partition.py:97-119) -> (k, owner uint8 [n] in HBM)."""
    device = torch.device(device or "cuda")
    path = Path(path)
    size = path.stat().st_size
    if size < _RPB_HEADER.size:
        raise ValueError("file too short for RPB1 header")
    with open(path, "rb") as f:
        magic, k, n = _RPB_HEADER.unpack(f.read(_RPB_HEADER.size))
    if magic != RPB1_MAGIC:
        raise ValueError(f"bad magic {magic!r}")
    if size < _RPB_HEADER.size + 4 * n:
        raise OSError("truncated RPB1 payload")
    if k > 255:
        raise NotImplementedError("at most 255 partitions in the device owner map")
    mm = np.memmap(path, dtype="<u4", mode="r", offset=_RPB_HEADER.size, shape=(n,))
    st = _Stager(device)
    own = torch.empty(n, dtype=torch.int32, device=device)
    st.copy(mm, own)
    st.finish()
    if n and (bool((own < 0).any()) or bool((own >= k).any())):
        raise ValueError("owner id out of range")
    return int(k), own.to(torch.uint8)
