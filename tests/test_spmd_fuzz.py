"""SPMD divergence fuzzing (the reference's acceptance criterion 5,
test_acceptance.py:156-229): 1000 seeded cases, each with one team member
whose visit sequence diverges from its teammates' in one of ten ways, must
all raise OrderingViolationError for the region, and team sizes must stay
within the cap.  Host logic only (C++ formation core + Python facade on the
fake device seam)."""

import random
from fractions import Fraction

import pytest

from fakes import FakeDevice
from paper_2210_06438_b200.aggregator import AggregationRegion
from paper_2210_06438_b200.bufferpool import BufferPool
from paper_2210_06438_b200.errors import OrderingViolationError
from paper_2210_06438_b200.executorpool import ExecutorPool
from paper_2210_06438_b200.sched import Scheduler, SchedulerConfig, await_all

# the reference's mutation kinds (test_acceptance.py:156-158)
KINDS = ("alloc_space", "alloc_len", "alloc_dtype", "swap_order",
         "early_leave", "skip_copy", "copy_dir", "copy_len",
         "kernel_name", "kernel_bps")


def visit(region, length, kind):
    """One task's region visit; `kind` mutates it (None = the SPMD norm:
    alloc pinned, alloc device, h2d, launch, d2h, await, leave)."""
    def body():
        member = yield region.enter()
        member.slice_alloc("device" if kind == "alloc_space" else
                           "pinned_host", "f8", length)
        if kind == "swap_order":
            member.slice_copy("h2d", 8 * length)
            member.slice_alloc("device", "f8", length)
        else:
            member.slice_alloc("device", "f4" if kind == "alloc_dtype"
                               else "f8",
                               length + (kind == "alloc_len"))
            if kind == "early_leave":
                member.leave()
                return
            if kind != "skip_copy":
                member.slice_copy("d2h" if kind == "copy_dir" else "h2d",
                                  8 * length + 8 * (kind == "copy_len"))
        member.slice_launch("wrong" if kind == "kernel_name" else "fused",
                            3 if kind == "kernel_bps" else 2, Fraction(1))
        done = member.slice_copy("d2h", 8 * length)
        yield await_all(done)
        member.leave()
    return body


def run_case(rng):
    cap = rng.randint(2, 6)
    per_parent = rng.randint(2, min(cap, 4))
    tasks = 2 * per_parent
    mutant = rng.randrange(tasks)
    kind = rng.choice(KINDS)
    length = rng.randint(3, 9)
    sched = Scheduler(SchedulerConfig(worker_count=8))
    device = FakeDevice(sched)
    pool = ExecutorPool(sched, device, 2)
    region = AggregationRegion(sched, pool, BufferPool(device), "r", cap)
    for name in ("fused", "wrong"):
        region.register_kernel(name, lambda stream, args: None)
    for ex in pool.executors:     # both streams busy: teams form
        device.hold(ex.stream_id)
    for i in range(tasks):
        sched.spawn(visit(region, length, kind if i == mutant else None))
    with pytest.raises(OrderingViolationError) as err:
        sched.run()
    assert err.value.region == "r", kind
    hist = region.stats().size_histogram
    assert hist and max(hist) <= cap, (kind, hist, cap)
    return kind


def test_divergence_fuzzing_1000_cases():
    rng = random.Random(20260819)     # the reference's seed
    seen = {}
    for _ in range(1000):
        kind = run_case(rng)
        seen[kind] = seen.get(kind, 0) + 1
    assert sum(seen.values()) == 1000 and set(seen) == set(KINDS)


@pytest.mark.parametrize("kind", KINDS)
def test_each_divergence_kind_detected(kind):
    class Fixed(random.Random):
        def choice(self, seq):
            return kind
    assert run_case(Fixed(len(kind))) == kind
