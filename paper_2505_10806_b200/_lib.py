"""ctypes binding of librapidgnn_b200.so (the C ABI in include/rapidgnn_b200.h).

There is no CPU fallback: if the shared library is missing or the device is
not an sm_100 GPU, every device entry point raises.  Error codes map to the
exception classes the reference raises for the same conditions.
"""

from __future__ import annotations

import ctypes
import threading
from ctypes import c_double, c_int32, c_int64, c_uint32, c_uint64, c_void_p
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "librapidgnn_b200.so"

RG_OK = 0
RG_ERR_INVALID = -1
RG_ERR_CUDA = -2
RG_ERR_UNSUPPORTED = -3
RG_ERR_NOT_OWNED = -4

RG_KIND_SHIFT = 28
RG_KIND_CACHE = 15
RG_ROW_MASK = 0x0FFFFFFF
RG_ROUTE_INVALID = 0xFFFFFFFF
RG_MAX_PARTS = 15
RG_CNT_LOCAL, RG_CNT_HIT, RG_CNT_FALLBACK, RG_CNT_OWNER_MASK, RG_CNT_BAD = 0, 1, 2, 3, 4
RG_CNT_PEER = 5
RG_NCOUNTERS = 8
PRNG_KINDS = {"splitmix": 0, "pcg32": 1, "sfc64": 2, "xoshiro256pp": 3}

P = c_void_p
# name -> (restype, argtypes); mirrors include/rapidgnn_b200.h
_SIGNATURES = {
    "rg_last_error": (ctypes.c_char_p, []),
    "rg_abi_version": (c_int32, []),
    "rg_device_ok": (c_int32, []),
    "rg_mix64": (c_int32, [P, P, c_int64, P]),
    "rg_stream_keys": (c_int32, [c_uint64, c_int64, P, P]),
    "rg_fill_seeds": (c_int32, [P, c_int64, c_int32, c_int64, c_int32, P, P, c_int32, c_uint64,
                                c_int64, P, P]),
    "rg_mark_seeds": (c_int32, [P, P, c_int32, c_int32, P, c_int64, P]),
    "rg_sample_level": (c_int32, [P, P, c_int64, c_int32, P, c_int64, P, c_int32, c_int32, P, P,
                                  P, P, c_int64, P, P, c_int32, c_int32, P]),
    "rg_bitmap_chunks": (c_int64, [c_int64]),
    "rg_bitmap_compact_launches": (c_int32, [c_int64]),
    "rg_bitmap_compact": (c_int32, [P, c_int64, c_int32, P, P, c_int64, P, P, P]),
    "rg_bitmap_set": (c_int32, [P, P, P, P]),
    "rg_scan_chunks": (c_int64, [c_int64]),
    "rg_ell_to_edges": (c_int32, [P, P, c_int64, P, P, c_int32, c_int32, P, P, P, P, c_int64, P,
                                  P]),
    "rg_count_inputs": (c_int32, [P, c_int64, c_int32, c_int64, P, P]),
    "rg_count_histogram": (c_int32, [P, P, c_int32, c_int64, P, c_int32, P, P]),
    "rg_threshold_split": (c_int32, [P, P, c_int64, c_uint32, P, P, P]),
    "rg_gather_counts": (c_int32, [P, P, P, c_int64, P, P]),
    "rg_fill_features": (c_int32, [P, c_int64, c_int32, c_int32, c_uint64, P, P]),
    "rg_route_with_cache": (c_int32, [P, c_int64, P, c_int64, P, P]),
    "rg_gather_bundle": (c_int32, [P, P, c_int64, c_int32, P, P, c_int32, c_int32, c_int32,
                                   c_uint32, P, P, P]),
    "rg_gather_window": (c_int32, [P, P, c_int64, c_int32, c_int64, P, P, c_int32, c_int32,
                                   c_int32, c_uint32, P, P, P]),
    "rg_copy_bytes": (c_int32, [P, P, c_int64, P]),
    "rg_flag_signal": (c_int32, [P, c_uint64, P]),
    "rg_flag_wait": (c_int32, [P, c_uint64, c_int32, P, P]),
    "rg_softmax_xent": (c_int32, [c_int32, P, c_int32, c_int64, P, P, P, P, P, P, P]),
    "rg_sgd_apply": (c_int32, [c_int32, c_int32, P, P, P, P, c_double, P]),
    "rg_route_kind_bits": (c_int32, [P, c_int64, c_uint32, P, P]),
    "rg_group_union": (c_int32, [P, c_int64, c_int32, P, P, P]),
    "rg_prefetch_rows": (c_int32, [P, P, c_int64, P, P, P, c_int32, c_int32, P]),
    "rg_scatter_rows": (c_int32, [P, c_int64, P, P, c_int32, P, c_int32, c_int32, P]),
    "rg_sage_positions": (c_int32, [P, c_int64, P, c_int64, P, P, c_int32, c_int64, P, P, P, P,
                                    P, P]),
    "rg_sage_mean_fwd": (c_int32, [c_int32, P, c_int32, c_int32, P, P, c_int64, P, P, c_int32,
                                   P, P, P]),
    "rg_sage_transpose_scratch": (c_int64, [c_int64, c_int64, c_int32]),
    "rg_sage_transpose": (c_int32, [P, P, c_int64, c_int32, c_int64, P, P, P, c_int64, P]),
    "rg_sage_mean_bwd": (c_int32, [c_int32, P, P, c_int64, c_int32, P, P, P, P, c_int64, P, P,
                                   P, P, P]),
    "rg_prng_raw": (c_int32, [c_int32, c_uint64, c_uint64, c_int64, P]),
    "rg_prng_select": (c_int32, [c_int32, c_uint64, c_uint64, c_int32, c_int32, P]),
    "rg_philox_raw": (c_int32, [c_uint64, c_uint64, c_int64, P]),
    "rg_synth_powerlaw_csr": (c_int32, [c_int64, c_int64, c_uint64, c_uint64, P, P, P]),
    "rg_partition_edgecut": (c_int32, [c_int64, P, P, c_int32, P]),
    "rg_ipc_handle": (c_int32, [P, P, P]),
    "rg_ipc_open": (c_int32, [P, ctypes.POINTER(c_void_p)]),
    "rg_ipc_close": (c_int32, [P]),
    "rg_enable_peer": (c_int32, [c_int32]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None
_device_checked = False


class ExtensionMissing(ImportError):
    """The CUDA extension was not built; run __graft_entry__.build()."""


class NativeNotOwned(KeyError):
    pass


def load() -> ctypes.CDLL:
    """Load the shared library (host entry points work without a GPU)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ExtensionMissing(
                    f"{LIB_PATH} not found: build it with `python -m paper_2505_10806_b200.build`")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def check(rc: int, what: str = "") -> None:
    if rc == RG_OK:
        return
    msg = load().rg_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == RG_ERR_INVALID:
        raise ValueError(text)
    if rc == RG_ERR_UNSUPPORTED:
        raise NotImplementedError(text)
    if rc == RG_ERR_NOT_OWNED:
        raise NativeNotOwned(text)
    raise RuntimeError(f"CUDA error in {text}")


def device() -> ctypes.CDLL:
    """The library, after checking once that an sm_100 device is usable.

    Every device-side caller goes through this, so a missing GPU or a wrong
    architecture is a loud error, never a silent host fallback."""
    global _device_checked
    lib = load()
    if not _device_checked:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_2505_10806_b200 needs a CUDA device (B200, sm_100a); "
                               "there is no CPU fallback")
        torch.cuda.init()
        if not lib.rg_device_ok():
            raise RuntimeError("librapidgnn_b200 cannot run on this device: "
                               + lib.rg_last_error().decode(errors="replace"))
        _device_checked = True
    return lib


def _args(args):
    """numpy arrays pass as their host address; the caller's args tuple
    keeps them alive for the duration of the call (a temporary's
    .ctypes.data taken inline would dangle once the array is freed)."""
    return [a.ctypes.data if isinstance(a, np.ndarray) else a for a in args]


def call(name: str, *args) -> None:
    check(getattr(device(), name)(*_args(args)), name)


def host_call(name: str, *args) -> None:
    check(getattr(load(), name)(*_args(args)), name)


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    """Device (or host numpy) address of a tensor/array, None for None."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data
