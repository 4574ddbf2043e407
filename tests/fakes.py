"""Test double for the device seam, for CPU-only tests of the host logic
(scheduler, aggregation regions, buffer pool).  Streams are queues of
pending ops; `poll()` completes one op per stream per call, like a device
making progress while the host waits; `hold(sid)` parks a never-finishing
primer op on a stream (the reference tests' prime_stream, test_aggregator
.py:35-39) until `release(sid)`."""

from collections import deque

import torch


class _Op:
    def __init__(self, token, held=False):
        self.token = token
        self.held = held


class FakeDevice:
    def __init__(self, sched):
        self.sched = sched
        self.streams = []
        self.kernels_enqueued = 0
        self.copies_enqueued = 0
        self.bytes_copied = 0
        self.raw_allocations = {"device": 0, "pinned_host": 0}
        self.launch_log = []
        sched.attach_device(self)

    def create_stream(self):
        self.streams.append({"q": deque(), "cb": []})
        return len(self.streams) - 1

    def stream(self, sid):
        return None

    def stream_busy(self, sid):
        return bool(self.streams[sid]["q"])

    def watch_stream_idle(self, sid, fn):
        cbs = self.streams[sid]["cb"]
        cbs.append(fn)

        def cancel():
            if fn in cbs:
                cbs.remove(fn)
        return cancel

    def outstanding(self, sid):
        return len(self.streams[sid]["q"])

    def _submit(self, sid, label, held=False):
        tok = self.sched.new_token(label)
        self.streams[sid]["q"].append(_Op(tok, held))
        return tok

    def hold(self, sid):
        return self._submit(sid, "primer", held=True)

    def release(self, sid):
        for op in self.streams[sid]["q"]:
            op.held = False

    def enqueue_kernel(self, sid, spec, launch=None, body=None):
        if body is not None:
            body()
        if launch is not None:
            launch(None)
        self.kernels_enqueued += 1
        self.launch_log.append((sid, spec.kernel_id, spec.blocks,
                                spec.slice_count))
        return self._submit(sid, f"kernel:{spec.kernel_id}")

    def enqueue_copy(self, sid, direction, nbytes, src=None, dst=None):
        if src is not None and dst is not None and nbytes:
            n = nbytes // src.element_size()
            dst.view(-1)[:n].copy_(src.view(-1)[:n])
        self.copies_enqueued += 1
        self.bytes_copied += nbytes
        return self._submit(sid, f"copy:{direction}")

    def raw_alloc(self, kind, nbytes, dtype=torch.float64):
        self.raw_allocations[kind] += 1
        item = torch.empty((), dtype=dtype).element_size()
        return torch.empty(max(1, nbytes // item), dtype=dtype)

    def poll(self):
        progress = False
        for s in self.streams:
            q = s["q"]
            if q and not q[0].held:
                q.popleft().token.fire()
                progress = True
                if not q and s["cb"]:
                    cbs, s["cb"] = s["cb"], []
                    for fn in cbs:
                        fn(self.sched.now)
            elif not q and s["cb"]:
                cbs, s["cb"] = s["cb"], []
                for fn in cbs:
                    fn(self.sched.now)
                progress = True
        if not progress:
            # only held primers remain: let them go (the primer "finishes")
            for s in self.streams:
                if s["q"] and s["q"][0].held:
                    s["q"][0].held = False
                    progress = True
        return progress

    def has_outstanding(self):
        return any(s["q"] or s["cb"] for s in self.streams)
