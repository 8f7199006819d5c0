"""CPU tests of the process-wide pinned-framebuffer registry (_native._Pins)
against a fake library: least-recently-used eviction, buffers with a copy in
flight never evicted, pages unlocked when the caller drops the array, and
ranges page-locked by someone else never unregistered here."""

import gc

import numpy as np
import pytest

from paper_2305_07450_b200 import _native


class FakeLib:
    def __init__(self, already=()):
        self.locked = set()
        self.already = set(already)
        self.calls = []

    def rt_host_register(self, ctx, p, nbytes):
        addr = p.value
        self.calls.append(("reg", addr))
        if addr in self.already:
            return _native.RT_ALREADY_REGISTERED
        assert addr not in self.locked
        self.locked.add(addr)
        return _native.RT_OK

    def rt_host_unregister(self, ctx, p):
        addr = p.value
        self.calls.append(("unreg", addr))
        assert addr in self.locked, "unregistered a range this registry does not own"
        self.locked.remove(addr)
        return _native.RT_OK


@pytest.fixture
def fake(monkeypatch):
    lib = FakeLib()
    monkeypatch.setattr(_native, "load", lambda: lib)
    return lib


def addr(a):
    return a.__array_interface__["data"][0]


def test_lru_eviction_and_refresh_on_hit(fake):
    pins = _native._Pins()
    bufs = [np.zeros(1 << 16, np.uint32) for _ in range(4)]
    for b in bufs[:3]:
        assert pins.pin(b, max_pinned=3)
    assert pins.pin(bufs[0], max_pinned=3)  # a hit moves it to the back
    assert pins.pin(bufs[3], max_pinned=3)  # evicts the least recent: bufs[1]
    assert fake.locked == {addr(bufs[0]), addr(bufs[2]), addr(bufs[3])}
    # re-pinning a pinned buffer does not register it again
    n = len(fake.calls)
    assert pins.pin(bufs[3], max_pinned=3)
    assert len(fake.calls) == n


def test_held_buffers_are_never_evicted(fake):
    pins = _native._Pins()
    busy = np.zeros(1 << 16, np.uint32)
    assert pins.pin(busy, max_pinned=1)
    pins.hold(busy)
    others = [np.zeros(1 << 16, np.uint32) for _ in range(3)]
    for b in others:
        assert pins.pin(b, max_pinned=1)
    assert addr(busy) in fake.locked
    with pytest.raises(RuntimeError):
        pins.unpin(busy)
    pins.release(busy)
    assert pins.pin(others[0], max_pinned=1)
    assert addr(busy) not in fake.locked


def test_dropped_arrays_are_unlocked(fake):
    pins = _native._Pins()
    a = np.zeros(1 << 16, np.uint32)
    ad = addr(a)
    assert pins.pin(a)
    assert ad in fake.locked
    del a
    gc.collect()
    assert ad not in fake.locked
    assert pins.count() == 0


def test_foreign_registration_is_used_but_never_released(fake):
    pins = _native._Pins()
    a = np.zeros(1 << 16, np.uint32)
    fake.already.add(addr(a))
    assert pins.pin(a)
    assert pins.pinned(a)
    pins.unpin(a)  # not ours: no unregister call (FakeLib would raise)
    assert ("unreg", addr(a)) not in fake.calls
