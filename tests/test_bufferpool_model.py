"""The reference's pool-model property test (test_bufferpool.py:146-175) on
this framework's BufferPool (CPU, fake device seam): random acquire/release
sequences over three exact buckets keep the LIFO recycle model — a fresh
buffer only when the bucket is empty, otherwise a recycled one — and the
stats add up."""

from hypothesis import given, settings
from hypothesis import strategies as st

from fakes import FakeDevice
from paper_2210_06438_b200.bufferpool import BufferPool
from paper_2210_06438_b200.sched import Scheduler, SchedulerConfig


@settings(deadline=None, max_examples=60)
@given(st.lists(st.integers(-12, 11), max_size=40))
def test_random_sequences_respect_pool_model(ops):
    dev = FakeDevice(Scheduler(SchedulerConfig(worker_count=1)))
    pool = BufferPool(dev)
    keys = [("device", "f8", 4), ("device", "f8", 8), ("pinned_host", "f4", 4)]
    held, cached, expected_raw = [], {k: [] for k in keys}, 0
    for op in ops:
        if op >= 0 or not held:
            key = keys[op % 3]
            lease = pool.acquire(*key)
            if cached[key]:
                assert lease.origin == "recycled"
                # most recently returned first (LIFO)
                assert lease._buffer is cached[key].pop()
            else:
                assert lease.origin == "fresh"
                expected_raw += 1
            assert lease.array.numel() == key[2]   # storage materialises
            held.append((key, lease))
        else:
            key, lease = held.pop(abs(op) % len(held))
            pool.release(lease)
            cached[key].append(lease._buffer)
    s = pool.stats()
    assert s.raw_allocations == expected_raw
    assert s.acquisitions == s.raw_allocations + s.reuses
    assert s.outstanding == len(held)
    assert s.cached == sum(len(v) for v in cached.values())
    assert dev.raw_allocations["device"] + dev.raw_allocations["pinned_host"] \
        == expected_raw        # storage kept across recycling
