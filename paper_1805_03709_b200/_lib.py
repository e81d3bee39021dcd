"""ctypes binding of libvsb200.so (the C ABI declared in include/vsb200.h).

The shared library is built in-tree by ``paper_1805_03709_b200.build``.  There
is deliberately no CPU fallback: if the library or a CUDA device is missing,
every product entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import pathlib
import threading

import os

# VSB_LIB lets experiments load an alternative build of the same ABI
LIB_PATH = pathlib.Path(os.environ.get("VSB_LIB") or pathlib.Path(__file__).resolve().with_name("libvsb200.so"))
HEADER_PATH = pathlib.Path(__file__).resolve().parent.parent / "include" / "vsb200.h"

VS_OK = 0
VS_ERR_CAPACITY = 1
VS_ERR_INVALID = 2
VS_ERR_CUDA = 3
VS_ERR_OVERFLOW = 4

VS_OP_INSERT = 0
VS_OP_FIND = 1
VS_OP_ERASE = 2


class NativeUnavailable(RuntimeError):
    """libvsb200.so (or a CUDA device) is not available; no fallback exists."""


class CapacityExhausted(RuntimeError):
    """Raised when an insert needs an excess entry and the free list is empty.

    Same name and base class as the reference (concurrent_hash.py:45-46).
    """


_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_i32 = ctypes.c_int32
_pu64 = ctypes.POINTER(ctypes.c_uint64)

# name -> (restype, argtypes); mirrors include/vsb200.h one to one
SIGNATURES: dict[str, tuple] = {
    "vs_last_error": (ctypes.c_char_p, []),
    "vs_abi_version": (_i32, []),
    "vs_profile_begin": (_i32, []),
    "vs_launch_count": (ctypes.c_uint64, []),
    "vs_profile_end": (_i32, [ctypes.POINTER(ctypes.c_double * 4), ctypes.POINTER(ctypes.c_uint64 * 4), _pu64]),
    "vs_hash_keys": (_i32, [_vp, _u64, _u32, _vp, _vp]),
    "vs_table_create": (_i32, [_u64, _u64, ctypes.c_int, ctypes.POINTER(_vp)]),
    "vs_table_destroy": (_i32, [_vp]),
    "vs_table_info": (_i32, [_vp, _pu64, _pu64, _pu64]),
    "vs_table_insert": (_i32, [_vp, _vp, _u64, _vp, _vp, _vp]),
    "vs_table_insert_bounded": (_i32, [_vp, _vp, _u64, _vp, _vp, _vp, _vp]),
    "vs_table_find": (_i32, [_vp, _vp, _u64, _vp, _vp, _vp]),
    "vs_table_erase": (_i32, [_vp, _vp, _u64, _vp, _vp, _vp]),
    "vs_table_apply": (_i32, [_vp, _vp, _vp, _u64, _vp, _vp, _vp]),
    "vs_table_check": (_i32, [_vp, _vp]),
    "vs_table_single": (_i32, [_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int32 * 3),
                               ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(ctypes.c_int32), _vp]),
    "vs_table_size": (_i32, [_vp, _vp, _pu64, _vp]),
    "vs_table_free_count": (_i32, [_vp, _pu64, _vp]),
    "vs_table_clear": (_i32, [_vp, _vp]),
    "vs_table_snapshot": (_i32, [_vp, _vp, _vp, _u64, _vp, _vp]),
    "vs_table_extract": (_i32, [_vp, _u64, _u64, _vp, _vp, _vp]),
    "vs_table_audit": (_i32, [_vp, ctypes.POINTER(ctypes.c_uint64 * 6), _vp]),
    "vs_mc_encode": (_i32, [_vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp]),
    "vs_mc_encode_keys": (_i32, [_vp, _vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp]),
    "vs_mc_faces": (_i32, [_vp, _vp, _u64, _vp, _vp]),
    "vs_mc_encode_keys_ex": (_i32, [_vp, _vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _u64,
                                    _vp]),
    "vs_mc_neighbors": (_i32, [_vp, _vp, _u64, _vp, _vp]),
    "vs_mc_compact": (_i32, [_vp, _vp, _u64, _vp, _vp, _vp, _u64, _vp, _vp]),
    "vs_scan_workspace_bytes": (_u64, [_u64]),
    "vs_affected_dedup": (_i32, [_vp, _vp, _u64, _vp, _vp, _vp]),
    "vs_stream_insert_many": (_i32, [ctypes.POINTER(_vp), ctypes.c_int, _vp, _u64, _vp, _vp,
                                     ctypes.POINTER(_vp), _pu64, ctypes.POINTER(_vp), _vp, _vp]),
    "vs_stream_extract_random": (_i32, [ctypes.POINTER(_vp), ctypes.c_int, _u64, _pu64, _vp, _vp, _vp]),
    "vs_server_tick": (_i32, [_vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp, ctypes.POINTER(_vp), ctypes.c_int,
                              _vp, _vp, _vp, _vp, _vp, _vp]),
    "vs_stream_tick": (_i32, [ctypes.POINTER(_vp), ctypes.c_int, _vp, _u64, _vp, _vp, _vp, _u64, _pu64, _vp, _vp, _vp,
                              _vp, _vp, _vp]),
    "vs_stream_extract_visible": (_i32, [ctypes.POINTER(_vp), ctypes.c_int, _u64, _pu64,
                                         ctypes.POINTER(ctypes.c_double * 24), ctypes.c_double, ctypes.c_double,
                                         _vp, _vp, _vp]),
    "vs_mc_pack": (_i32, [_vp, _vp, _u64, _vp, _vp, _vp]),
    "vs_tsdf_put": (_i32, [_vp, _vp, _vp, _u64, _vp, _vp, _vp]),
    "vs_rc_params_bytes": (_u64, []),
    "vs_rc_candidates": (_i32, [_vp, _vp, _vp, _u64, _vp, _vp]),
    "vs_rc_zero_rows": (_i32, [_vp, _vp, _u64, _vp, _vp]),
    "vs_rc_integrate": (_i32, [_vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "vs_rc_integrate_table": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "vs_stream_remove_many": (_i32, [ctypes.POINTER(_vp), ctypes.c_int, _vp, _u64, _vp, _vp]),
    "vs_stream_extract_ordered": (_i32, [_vp, _vp, _u64, _pu64, _u64, _u64, _vp, _pu64, _vp, _vp]),
    "vs_table_probe_sol": (_i32, [_vp, _u64, ctypes.c_int, _vp, _vp]),
    "vs_shard_create": (_i32, [_vp, ctypes.c_int, ctypes.c_int, _u64, ctypes.POINTER(_vp)]),
    "vs_shard_destroy": (None, [_vp]),
    "vs_shard_export": (_i32, [_vp, ctypes.POINTER(ctypes.c_uint8 * 64)]),
    "vs_shard_connect": (_i32, [_vp, ctypes.c_char_p]),
    "vs_shard_apply": (_i32, [_vp, _vp, _vp, _u64, _vp, _vp]),
    "vs_shard_connect_local": (_i32, [ctypes.POINTER(_vp), ctypes.c_int]),
    "vs_shard_check": (_i32, [_vp]),
    "vs_shard_set_timeout_ms": (_i32, [_vp, _u64]),
    "vs_shard_owner": (_i32, [_vp, _u64, ctypes.c_int, _vp]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load (once) and type the native library; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeUnavailable(
                f"{LIB_PATH} is missing: run `python -m paper_1805_03709_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("VSB_LIB") and not hasattr(lib, name):
                continue  # A/B runs against an older library build (scripts/ab.py)
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().vs_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    """Map a vs_status to the reference's exception types."""
    if status == VS_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if status == VS_ERR_CAPACITY:
        raise CapacityExhausted(msg)
    if status == VS_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"libvsb200 status {status}: {msg}")


def require_cuda():
    """Import torch and insist on a CUDA device (the product path is GPU-only)."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: libvsb200 has no CPU fallback")
    load()
    return torch


def ptr(t) -> ctypes.c_void_p:
    """Raw data pointer of a torch tensor (or None for NULL)."""
    if t is None:
        return ctypes.c_void_p(None)
    return ctypes.c_void_p(t.data_ptr())


def stream_of(device) -> ctypes.c_void_p:
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class Profile:
    """Context manager around vs_profile_begin/end (bench.py)."""

    TAGS = ("hash", "mc", "stream", "other")

    def __init__(self, events: bool = True):
        # events=False: count launches only (no per-launch event records on
        # the host path of a host-paced timed region)
        self.events = events

    def __enter__(self):
        if self.events:
            check(load().vs_profile_begin())
        else:
            self._n0 = int(load().vs_launch_count())
        return self

    def __exit__(self, *exc):
        if not self.events:
            self.ms = {t: 0.0 for t in self.TAGS}
            self.count = {t: 0 for t in self.TAGS}
            self.launches = int(load().vs_launch_count()) - self._n0
            return False
        ms = (ctypes.c_double * 4)()
        cnt = (ctypes.c_uint64 * 4)()
        launches = ctypes.c_uint64()
        check(load().vs_profile_end(ctypes.byref(ms), ctypes.byref(cnt), ctypes.byref(launches)))
        self.ms = {t: float(ms[i]) for i, t in enumerate(self.TAGS)}
        self.count = {t: int(cnt[i]) for i, t in enumerate(self.TAGS)}
        self.launches = int(launches.value)
        return False
