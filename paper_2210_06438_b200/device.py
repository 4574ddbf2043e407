"""The device seam of taskfuse/device.py on a real B200.

The reference's VirtualDevice (device.py:141-433) co-simulates streams,
block slots and a launch lane on a virtual clock; here the hardware does
that, and `CudaDevice` keeps only the seam the upper layers call
(device.py:177-269), with the same names and semantics:

    create_stream()                 a real CUDA stream (non-blocking)
    stream_busy(sid)                enqueued-but-unfinished work? (the last
                                    recorded CUDA event has not completed)
    watch_stream_idle(sid, fn)      fn(t) when the stream next drains
    enqueue_kernel(sid, spec, launch=None, body=None)
                                    launch(stream) issues the real kernel
    enqueue_copy(sid, dir, nbytes, src=None, dst=None)
                                    real stream-ordered copy (tf_memcpy_async)
                                    when buffers are given
    raw_alloc(kind, nbytes)         device / pinned-host bytes
    outstanding(sid)

Completion tokens fire when the device is polled (Scheduler.run polls every
attached device while no task is runnable) and the op's event has completed,
in stream order, exactly once — so task bodies written against the
reference (`yield await_all(token)`) run unchanged.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass
from fractions import Fraction
from typing import Callable

import torch

from . import _lib
from .errors import CapacityError, UsageError, ValidationError

MAX_STREAMS = 128
THREADS_PER_BLOCK = 128


@dataclass(frozen=True)
class KernelSpec:
    """device.py:86-103 — launch shape bookkeeping (blocks, slices)."""

    kernel_id: str
    blocks: int
    work_factor: Fraction = Fraction(1)
    threads_per_block: int = THREADS_PER_BLOCK
    slice_count: int = 1

    def __post_init__(self):
        if self.blocks < 1:
            raise ValidationError(f"blocks must be >= 1, got {self.blocks}")
        if self.slice_count < 1:
            raise ValidationError("slice_count must be >= 1")
        if self.work_factor <= 0:
            raise ValidationError("work_factor must be > 0")


class _Op:
    __slots__ = ("event", "token", "kind")

    def __init__(self, event, token, kind):
        self.event = event
        self.token = token
        self.kind = kind


class _Stream:
    __slots__ = ("index", "stream", "handle", "queue", "idle_callbacks")

    def __init__(self, index, stream):
        self.index = index
        self.stream = stream
        self.handle = stream.cuda_stream
        self.queue: deque[_Op] = deque()
        self.idle_callbacks: list[Callable[[int], None]] = []


class CudaDevice:
    def __init__(self, sched, device=None, record_events: bool = False):
        self.sched = sched
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.record_events = record_events
        self.events: list[tuple] = []
        self._streams: list[_Stream] = []
        self.kernels_enqueued = 0
        self.copies_enqueued = 0
        self.bytes_copied = 0
        self.raw_allocations = {"device": 0, "pinned_host": 0}
        self.sync_count = 0
        self._index = self.device.index if self.device.index is not None \
            else torch.cuda.current_device()
        self._free_events: list = []   # retired ops' events, reused
        self._lib = _lib.load()
        sched.attach_device(self)

    # -- streams -----------------------------------------------------------
    def create_stream(self) -> int:
        if len(self._streams) >= MAX_STREAMS:
            raise CapacityError(
                f"device supports at most {MAX_STREAMS} concurrent streams")
        st = torch.cuda.Stream(device=self.device)
        self._streams.append(_Stream(len(self._streams), st))
        return len(self._streams) - 1

    def stream(self, sid: int) -> torch.cuda.Stream:
        return self._stream(sid).stream

    def _stream(self, sid: int) -> _Stream:
        try:
            return self._streams[sid]
        except (IndexError, TypeError):
            raise UsageError(f"unknown stream {sid}") from None

    def stream_busy(self, sid: int) -> bool:
        """device.py:187-194: any enqueued op not yet complete."""
        # a pure query (no callbacks fire here): stream order means the
        # newest op's event completes last
        s = self._stream(sid)
        return bool(s.queue) and not s.queue[-1].event.query()

    def watch_stream_idle(self, sid: int, fn) -> Callable[[], None]:
        s = self._stream(sid)
        s.idle_callbacks.append(fn)

        def cancel():
            if fn in s.idle_callbacks:
                s.idle_callbacks.remove(fn)
        return cancel

    def outstanding(self, sid: int) -> int:
        s = self._stream(sid)
        return sum(1 for op in s.queue if not op.event.query())

    # -- work submission ---------------------------------------------------
    def _submit(self, s: _Stream, kind: str, label: str):
        ev = self._free_events.pop() if self._free_events else \
            torch.cuda.Event()
        ev.record(s.stream)
        tok = self.sched.new_token(f"{label}@s{s.index}")
        s.queue.append(_Op(ev, tok, kind))
        return tok

    def enqueue_kernel(self, sid: int, spec: KernelSpec, launch=None,
                       body=None):
        """Issue `launch(stream)` (the batched kernel) on the stream.  A
        reference-style `body` callable runs at enqueue time, as the
        reference does (device.py:218-235)."""
        s = self._stream(sid)
        if body is not None:
            body()
        if launch is not None:
            # the stream is also made current for torch ops inside launch;
            # set/restore directly (torch.cuda.stream() re-queries the
            # device on every entry, a measurable cost per visit)
            prev = torch.cuda.current_stream(self._index)
            torch.cuda.set_stream(s.stream)
            try:
                launch(s.stream)
            finally:
                torch.cuda.set_stream(prev)
        self.kernels_enqueued += 1
        if self.record_events:
            self.events.append((self.sched.now, "kernel_enqueue", s.index,
                                spec.kernel_id, spec.blocks,
                                spec.slice_count))
        return self._submit(s, "kernel", f"kernel:{spec.kernel_id}")

    def enqueue_copy(self, sid: int, direction: str, nbytes: int, src=None,
                     dst=None):
        if direction not in ("h2d", "d2h"):
            raise UsageError(
                f"copy direction must be h2d or d2h, got {direction!r}")
        if nbytes < 0:
            raise UsageError("copy size must be >= 0")
        s = self._stream(sid)
        if src is not None and dst is not None and nbytes:
            if nbytes > min(src.numel() * src.element_size(),
                            dst.numel() * dst.element_size()):
                raise UsageError("copy larger than its buffers")
            _lib.check(self._lib.tf_memcpy_async(
                dst.data_ptr(), src.data_ptr(), nbytes, s.handle),
                "tf_memcpy_async")
        self.copies_enqueued += 1
        self.bytes_copied += nbytes
        return self._submit(s, "copy", f"copy:{direction}")

    def raw_alloc(self, kind: str, nbytes: int, dtype=torch.float64):
        """Real allocation: device memory, or page-locked host memory."""
        if kind not in ("device", "pinned_host"):
            raise UsageError(f"unknown allocation kind {kind!r}")
        if nbytes < 0:
            raise UsageError("allocation size must be >= 0")
        self.raw_allocations[kind] += 1
        itemsize = torch.empty((), dtype=dtype).element_size()
        count = max(1, nbytes // itemsize)
        if kind == "device":
            return torch.empty(count, dtype=dtype, device=self.device)
        return torch.empty(count, dtype=dtype).pin_memory()

    # -- completion ----------------------------------------------------------
    def _retire(self, s: _Stream) -> bool:
        progress = False
        while s.queue and s.queue[0].event.query():
            op = s.queue.popleft()
            self._free_events.append(op.event)
            op.token.fire()
            progress = True
        if progress and not s.queue and s.idle_callbacks:
            callbacks, s.idle_callbacks = s.idle_callbacks, []
            now = self.sched.now
            for fn in callbacks:
                fn(now)
        return progress

    def poll(self) -> bool:
        """Fire every completed op's token; drained streams fire their idle
        watches (device.py:356-373).  Returns True on any progress."""
        progress = False
        for s in self._streams:
            if s.queue:
                progress = self._retire(s) or progress
            elif s.idle_callbacks:
                callbacks, s.idle_callbacks = s.idle_callbacks, []
                now = self.sched.now
                for fn in callbacks:
                    fn(now)
                progress = True
        return progress

    def has_outstanding(self) -> bool:
        return any(s.queue or s.idle_callbacks for s in self._streams)

    def synchronize(self) -> None:
        torch.cuda.synchronize(self.device)
        self.sync_count += 1
        self.poll()
