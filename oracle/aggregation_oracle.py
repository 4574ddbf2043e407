"""CPU oracle for strategy-3 team formation — TEST INFRASTRUCTURE ONLY.

A pure-Python restatement of AggregationRegion's formation logic
(/root/reference/pkg/src/taskfuse/aggregator.py:247-345) driven by a
recorded signal log instead of a virtual device:

    ("arrive", region, tag, busy)   one `enter()`; busy is what the
                                    reference's device.stream_busy returned
                                    (None when it was not consulted)
    ("drain", stream)               device.py:364-370 fired the stream's
                                    idle callbacks

Replaying a log yields, per region, the closed teams in closure order as
(team_seq, parent, [tags in slice order], reason).  Pinned against traces
recorded from the reference itself (tests/golden/make_golden.py).  The
product formation core is C++ (paper_2210_06438_b200/csrc/aggregator.cpp);
tests replay the same logs through both.
"""

from __future__ import annotations

from zlib import crc32

MAX_TEAM = 128  # aggregator.py:42


class _Team:
    def __init__(self, seq, parent):
        self.seq = seq
        self.parent = parent
        self.tags = []
        self.state = "forming"


class RegionOracle:
    def __init__(self, name: str, max_team: int, parent_count: int,
                 executors: int):
        # aggregator.py:250-282
        if not 1 <= max_team <= MAX_TEAM:
            raise ValueError(f"max_team must be in 1..{MAX_TEAM}")
        self.name = name
        self.max_team = max_team
        lead = crc32(name.encode()) % executors
        self.parent_executor = [(lead + i) % executors
                                for i in range(parent_count)]
        self.forming = [None] * parent_count
        self.watch = {e: [] for e in range(executors)}
        self.arrivals = 0
        self.next_seq = 0
        self.closed = []            # (seq, parent, tags, reason)
        self.solo_fast_path = 0
        self.histogram = {}

    def _close(self, team, reason):
        # aggregator.py:334-345
        team.state = "closed"
        size = len(team.tags)
        self.histogram[size] = self.histogram.get(size, 0) + 1
        self.closed.append((team.seq, team.parent, list(team.tags), reason))

    def enter(self, tag, busy):
        """aggregator.py:284-326; `busy` answers device.stream_busy."""
        pi = self.arrivals % len(self.forming)
        self.arrivals += 1
        team = self.forming[pi]
        if team is None:
            team = _Team(self.next_seq, pi)
            self.next_seq += 1
        slice_id = len(team.tags)
        team.tags.append(tag)
        queried = False
        executor = self.parent_executor[pi]
        if len(team.tags) >= self.max_team:
            if self.forming[pi] is team:
                self.forming[pi] = None
                self.watch[executor].remove(team)
            self._close(team, "cap")
        elif self.forming[pi] is None:
            queried = True
            if not busy():
                self.solo_fast_path += 1
                self._close(team, "solo")
            else:
                self.forming[pi] = team
                self.watch[executor].append(team)
        return pi, slice_id, queried

    def stream_idle(self, executor):
        """aggregator.py:328-332 for every watch on the drained stream."""
        fire, self.watch[executor] = self.watch[executor], []
        for team in fire:
            if team.state == "forming":
                if self.forming[team.parent] is team:
                    self.forming[team.parent] = None
                self._close(team, "drain")


def replay(trace: dict) -> dict:
    """Replay a recorded trace; returns {region: closed-team list}."""
    regions = {
        r["name"]: RegionOracle(r["name"], r["max_team"], r["parents"],
                                trace["executors"])
        for r in trace["regions"]
    }
    for ev in trace["events"]:
        if ev[0] == "arrive":
            _, name, tag, busy = ev
            asked = []

            def answer(busy=busy, asked=asked):
                asked.append(True)
                if busy is None:
                    raise AssertionError("reference did not query busy here")
                return busy
            regions[name].enter(tag, answer)
            if busy is not None and not asked:
                raise AssertionError("reference queried busy, oracle did not")
        else:
            _, stream = ev
            for reg in regions.values():
                reg.stream_idle(stream)
    return {name: reg.closed for name, reg in regions.items()}
