"""Host-side logic of the stream-set fan-out that needs no GPU: the cached
ctypes argument arrays of a client group (server._group_args) must follow
the group's identity and FIFO reallocations."""
from __future__ import annotations

import gc
import types

from paper_1805_03709_b200 import server


class _Tensor:
    def __init__(self, ptr, rows=0):
        self._ptr, self.shape = ptr, (rows, 3)

    def data_ptr(self):
        return self._ptr


def _fake_set(i):
    st = object.__new__(server.StreamSet)  # bypass the CUDA constructor
    st._set = types.SimpleNamespace(handle=types.SimpleNamespace(value=0x1000 + i))
    st._fifo = _Tensor(0x2000 + i, rows=64)
    st._tail_dev = _Tensor(0x3000 + i)
    return st


def test_group_args_cached_per_group():
    server._GROUP_CACHE.clear()
    g = [_fake_set(i) for i in range(4)]
    a = server._group_args(g)
    assert list(a["handles"]) == [0x1000 + i for i in range(4)]
    assert list(a["fifos"]) == [0x2000 + i for i in range(4)]
    assert list(a["caps"]) == [64] * 4
    assert list(a["tails"]) == [0x3000 + i for i in range(4)]
    assert server._group_args(g) is a  # same group: reused
    assert server._group_args(g[:3]) is not a  # another group: its own arrays


def test_group_args_follow_fifo_growth():
    server._GROUP_CACHE.clear()
    g = [_fake_set(i) for i in range(2)]
    a = server._group_args(g)
    g[1]._fifo = _Tensor(0x9000, rows=128)
    server._FIFO_GEN[0] += 1  # what StreamSet._ensure_fifo does on reallocation
    b = server._group_args(g)
    assert b is not a
    assert list(b["fifos"]) == [0x2000, 0x9000] and list(b["caps"]) == [64, 128]


def test_group_args_never_match_a_dead_set():
    server._GROUP_CACHE.clear()
    g = [_fake_set(0)]
    server._group_args(g)
    key_ids = tuple(map(id, g))
    del g
    gc.collect()
    # whatever object reuses the id, the weak reference of the entry is dead
    for entry_key, (refs, _) in server._GROUP_CACHE.items():
        if entry_key[0] == key_ids:
            assert all(r() is None for r in refs)
    h = [_fake_set(7)]
    assert list(server._group_args(h)["handles"]) == [0x1007]
