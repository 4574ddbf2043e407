"""The device seam's semantics on real CUDA streams (CudaDevice), as the
reference's device tests pin them for the virtual device
(test_device.py:330-340 stream_busy, :389-398 body at enqueue): a stream is
busy while any enqueued op is unfinished and idle once it drains; idle
watches fire when it drains and can be cancelled; a kernel's body runs at
enqueue time; copies move real bytes; the stream limit is enforced."""

import pytest

pytestmark = pytest.mark.gpu


def _rig():
    from paper_2210_06438_b200.device import CudaDevice
    from paper_2210_06438_b200.sched import Scheduler, SchedulerConfig
    sched = Scheduler(SchedulerConfig(worker_count=1))
    return sched, CudaDevice(sched)


def test_stream_busy_until_drained_and_idle_watches(cuda):
    import torch
    from paper_2210_06438_b200.device import KernelSpec
    sched, dev = _rig()
    sid = dev.create_stream()
    assert not dev.stream_busy(sid)             # nothing enqueued
    big = torch.empty(1 << 26, dtype=torch.float64, device=cuda)
    fired, cancelled = [], []

    def launch(stream):                         # ~0.5 GB of writes
        for _ in range(4):
            big.fill_(1.0)
    body_ran = []
    tok = dev.enqueue_kernel(sid, KernelSpec("k", blocks=1),
                             launch=launch, body=lambda: body_ran.append(1))
    assert body_ran == [1]                      # body at enqueue
    assert dev.stream_busy(sid)
    dev.watch_stream_idle(sid, lambda now: fired.append(now))
    cancel = dev.watch_stream_idle(sid, lambda now: cancelled.append(now))
    cancel()
    torch.cuda.synchronize()
    assert not dev.stream_busy(sid)             # end-exclusive: done = idle
    while dev.poll():
        pass
    assert tok.is_ready and len(fired) == 1 and cancelled == []
    assert not dev.has_outstanding()


def test_copy_moves_bytes_and_counts(cuda):
    import torch
    sched, dev = _rig()
    sid = dev.create_stream()
    src = torch.arange(1000, dtype=torch.float64).pin_memory()
    dst = torch.zeros(1000, dtype=torch.float64, device=cuda)
    tok = dev.enqueue_copy(sid, "h2d", 8 * 1000, src, dst)
    torch.cuda.synchronize()
    while dev.poll():
        pass
    assert tok.is_ready and bool((dst.cpu() == src).all())
    assert dev.copies_enqueued == 1 and dev.bytes_copied == 8000


def test_stream_limit_and_bad_arguments(cuda):
    from paper_2210_06438_b200.device import MAX_STREAMS
    from paper_2210_06438_b200.errors import CapacityError, UsageError
    sched, dev = _rig()
    for _ in range(MAX_STREAMS):
        dev.create_stream()
    with pytest.raises(CapacityError):
        dev.create_stream()
    with pytest.raises(UsageError):
        dev.enqueue_copy(0, "sideways", 8)
    with pytest.raises(UsageError):
        dev.stream_busy(MAX_STREAMS + 5)
