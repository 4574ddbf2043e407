"""The C-ABI library loads, exports every entry point include/taskfuse_b200.h
declares, and its host-only formation core (no GPU needed) reproduces the
reference's team formation bit-exactly on recorded reference traces."""

import ctypes as C
import re

from conftest import ROOT

HEADER = ROOT / "include" / "taskfuse_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tf_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported(native_lib):
    from paper_2210_06438_b200 import _lib
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(native_lib, s), s
        assert s in _lib.SIGNATURES, f"{s} not bound in _lib.SIGNATURES"


def test_header_constants_match_python_mirror():
    """Every TF_* #define the Python side uses has the header's value."""
    from paper_2210_06438_b200 import _lib
    defs = dict(re.findall(r"#define\s+(TF_[A-Z0-9_]+)\s+(-?\d+)",
                           HEADER.read_text()))
    mirrored = [k for k in defs if hasattr(_lib, k)]
    for k in ("TF_LAUNCH_OVERLAP_PREV", "TF_PLAN_TEAM_BUFFERS",
              "TF_STEP_HALO_YZ", "TF_STEP_HALO_X"):
        assert k in mirrored, k
    for k in mirrored:
        assert getattr(_lib, k) == int(defs[k]), k
    # the launch / plan / halo flag bits are distinct
    bits = [int(defs[k]) for k in ("TF_LAUNCH_OVERLAP_PREV",
                                   "TF_PLAN_TEAM_BUFFERS", "TF_STEP_HALO_YZ",
                                   "TF_STEP_HALO_X")]
    assert sum(bits) == (bits[0] | bits[1] | bits[2] | bits[3])


def test_no_cpu_fallback():
    """The product path refuses host tensors instead of computing on the CPU."""
    import pytest
    import torch
    from paper_2210_06438_b200 import ops
    from paper_2210_06438_b200.errors import TaskfuseCudaError
    pool = torch.zeros((1, 14, 14, 14), dtype=torch.float64)
    faces = torch.zeros((1, 3, 10, 10, 10), dtype=torch.float64)
    with pytest.raises(TaskfuseCudaError, match="CUDA device"):
        ops.recon_flux(pool, 8, (1, 1, 1), faces, faces, faces)
    with pytest.raises(TaskfuseCudaError):
        ops.ghost_fill(pool, 8, 1)
    with pytest.raises(TaskfuseCudaError):
        ops.update(pool, 8, faces, 0.3, pool)


def test_version(native_lib):
    assert b"sm_100a" in native_lib.tf_version()


def test_region_validation(native_lib):
    h = C.c_void_p()
    assert native_lib.tf_region_create(b"r", 0, 1, 1, C.byref(h)) != 0
    assert native_lib.tf_region_create(b"r", 129, 1, 1, C.byref(h)) != 0
    assert native_lib.tf_region_create(b"r", 2, 0, 1, C.byref(h)) != 0
    assert native_lib.tf_region_create(b"r", 128, 3, 2, C.byref(h)) == 0
    lead = 1190910889  # crc32("reconstruct")
    h2 = C.c_void_p()
    assert native_lib.tf_region_create(b"reconstruct", 4, 5, 7,
                                       C.byref(h2)) == 0
    for i in range(5):
        assert native_lib.tf_region_parent_executor(h2, i) == (lead % 7 + i) % 7
    native_lib.tf_region_destroy(h)
    native_lib.tf_region_destroy(h2)


def replay_native(lib, trace):
    """Drive the C++ formation core with a recorded reference signal log."""
    from paper_2210_06438_b200 import _lib
    handles = {}
    for r in trace["regions"]:
        h = C.c_void_p()
        assert lib.tf_region_create(r["name"].encode(), r["max_team"],
                                    r["parents"], trace["executors"],
                                    C.byref(h)) == 0
        handles[r["name"]] = h
    closed = {name: [] for name in handles}

    def record(name, team, reason):
        h = handles[name]
        size = lib.tf_region_team_size(h, team)
        buf = (C.c_int64 * size)()
        lib.tf_region_team_members(h, team, buf, size)
        parent = lib.tf_region_team_parent(h, team)
        closed[name].append((parent, list(buf), reason))
        assert lib.tf_region_release_team(h, team) == 0

    reasons = {1: "cap", 2: "solo", 3: "drain"}
    for ev in trace["events"]:
        if ev[0] == "arrive":
            _, name, tag, busy = ev
            asked = []

            def answer(ctx, executor, busy=busy, asked=asked):
                asked.append(executor)
                assert busy is not None, "core queried busy; reference did not"
                return int(busy)
            cb = _lib.BUSY_FN(answer)
            res = _lib.EnterResult()
            assert lib.tf_region_enter(handles[name], tag, cb, None,
                                       C.byref(res)) == 0
            assert bool(res.queried) == (busy is not None)
            if res.closed:
                record(name, res.team, reasons[res.closed])
        else:
            stream = ev[1]
            for name, h in handles.items():
                buf = (C.c_int64 * 4096)()
                n = lib.tf_region_stream_idle(h, stream, buf, 4096)
                assert n >= 0
                for i in range(n):
                    record(name, buf[i], "drain")
    stats = {}
    for name, h in handles.items():
        tf, solo = C.c_int64(), C.c_int64()
        hist = (C.c_int64 * 129)()
        lib.tf_region_stats(h, C.byref(tf), C.byref(solo), hist)
        stats[name] = (tf.value, solo.value,
                       {str(k): hist[k] for k in range(129) if hist[k]})
        lib.tf_region_destroy(h)
    return closed, stats


def test_native_formation_replays_reference(native_lib, traces_golden):
    assert len(traces_golden) >= 10
    for tr in traces_golden:
        closed, stats = replay_native(native_lib, tr)
        for name, exp in tr["closes"].items():
            got = closed[name]
            assert [list(x) for x in got] == [list(x) for x in exp], \
                (tr["name"], name)
            st = tr["stats"][name]
            assert stats[name] == (st["teams_formed"], st["solo_fast_path"],
                                   st["histogram"]), (tr["name"], name)


def test_stream_idle_reports_every_closed_team(native_lib):
    """More forming teams than any fixed buffer (10 000 parents on one
    executor): every team the drain closes reaches the caller, and a short
    buffer leaves the rest forming instead of closing them unreported."""
    from paper_2210_06438_b200.strategy3 import FormationCore
    core = FormationCore("reconstruct", 2, 10_000, 1)
    for tag in range(10_000):
        res = core.enter(tag, lambda e: True)
        assert not res.closed
    lib = native_lib
    assert lib.tf_region_watch_count(core.handle, 0) == 10_000
    buf = (C.c_int64 * 16)()
    assert lib.tf_region_stream_idle(core.handle, 0, buf, 16) == 16
    assert lib.tf_region_watch_count(core.handle, 0) == 10_000 - 16
    assert core.stats()["teams_formed"] == 16
    rest = core.stream_idle(0)
    assert len(rest) == 10_000 - 16
    assert sorted(list(buf) + rest) == sorted(set(list(buf) + rest))
    assert core.stats()["teams_formed"] == 10_000
    assert lib.tf_region_watch_count(core.handle, 0) == 0
