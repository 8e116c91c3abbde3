"""Partition plans and the event-log format (drop-in subset of pipesafe.reduction).

``PartitionPlan`` is the reference's row partition (reduction.py:55-87).  On
the device it drives two things: the PBS_REDUCE_PLAN dot order (one
sequential chain per range, left-to-right combine, reduction.py:282-294) and
the row slabs of the multi-GPU path.  ``EventLog`` keeps the reference's
JSONL schema (reduction.py:136-178) so ``verify_phase_order`` can be re-run
on device-produced schedules.
"""

from __future__ import annotations

import json
import threading
from dataclasses import dataclass

import numpy as np

BATCH_LABELS = ("a", "b", "c", "d", "e", "f", "g", "h", "r")  # reduction.py:32

REDUCE_START = "reduce_start"
REDUCE_END = "reduce_end"
SPMV_START = "spmv_start"
SPMV_END = "spmv_end"
COEFF_READY = "coeff_ready"


@dataclass(frozen=True)
class PartitionPlan:
    """Disjoint contiguous row ranges covering [0, n) (reduction.py:55-87)."""

    n: int
    ranges: tuple[tuple[int, int], ...]

    def __post_init__(self):
        if self.n < 0:
            raise ValueError("negative vector length")
        if not self.ranges:
            raise ValueError("plan needs at least one range")
        pos = 0
        for lo, hi in self.ranges:
            if lo != pos or hi < lo or (hi == lo and self.n > 0):
                raise ValueError(f"ranges must tile [0, {self.n}) in order; got {self.ranges}")
            pos = hi
        if pos != self.n:
            raise ValueError(f"ranges cover [0, {pos}) but n = {self.n}")

    @property
    def worker_count(self) -> int:
        return len(self.ranges)

    @classmethod
    def balanced(cls, n: int, workers: int) -> "PartitionPlan":
        if workers < 1:
            raise ValueError("workers must be >= 1")
        workers = min(workers, max(n, 1))
        bounds = np.linspace(0, n, workers + 1).astype(np.int64)
        return cls(n, tuple((int(bounds[k]), int(bounds[k + 1])) for k in range(workers)))

    def is_balanced(self) -> bool:
        return self == PartitionPlan.balanced(self.n, self.worker_count)


@dataclass(frozen=True)
class ExecutionEvent:
    seq: int
    iter: int
    kind: str
    tag: str | None = None


class EventLog:
    """Append-only record of scheduling events (reduction.py:136-178)."""

    def __init__(self):
        self._lock = threading.Lock()
        self._events: list[ExecutionEvent] = []

    def append(self, iter_index: int, kind: str, tag: str | None = None) -> ExecutionEvent:
        with self._lock:
            ev = ExecutionEvent(len(self._events), iter_index, kind, tag)
            self._events.append(ev)
            return ev

    def events(self) -> list[ExecutionEvent]:
        with self._lock:
            return list(self._events)

    def __len__(self) -> int:
        return len(self._events)

    def write_jsonl(self, path: str) -> None:
        with open(path, "w", encoding="ascii") as fh:
            for ev in self.events():
                fh.write(json.dumps({"seq": ev.seq, "iter": ev.iter, "kind": ev.kind, "tag": ev.tag}))
                fh.write("\n")

    @classmethod
    def read_jsonl(cls, path: str) -> "EventLog":
        log = cls()
        with open(path, "r", encoding="ascii") as fh:
            for line in fh:
                row = json.loads(line)
                log._events.append(ExecutionEvent(row["seq"], row["iter"], row["kind"], row.get("tag")))
        return log


_KINDS = {0: REDUCE_START, 1: REDUCE_END, 2: SPMV_START, 3: SPMV_END, 4: COEFF_READY}
_TAGS = {0: None, 1: "Ax", 2: "Ar", 3: "As", 4: "Aw", 5: "Ao", 6: "Au", 7: "At", 8: "Ay"}


def events_to_log(records) -> EventLog:
    """Device schedule records (iter, kind, tag, t_ms) -> the reference's EventLog.

    seq follows the CUDA-event timestamps (ties keep issue order), so the
    reference's verify_phase_order (reduction.py:486-563) can be re-run on it.
    """
    recs = [(float(t), k, int(i), int(kind), int(tag)) for k, (i, kind, tag, t) in enumerate(records)]
    recs.sort(key=lambda r: (r[0], r[1]))
    log = EventLog()
    for t, _, i, kind, tag in recs:
        log.append(i, _KINDS[kind], _TAGS.get(tag))
    return log


def overlap_report(records) -> dict:
    """Per iteration: the reduction's [start, end] vs the As SpMV's [start, end]
    (CUDA-event ms).  overlapped = the intervals intersect, i.e. the
    all-gather + check really ran while A s was computed."""
    per: dict[int, dict] = {}
    for i, kind, tag, t in records:
        d = per.setdefault(int(i), {})
        if kind == 0:
            d["r0"] = t
        elif kind == 1:
            d["r1"] = t
        elif kind == 2 and int(tag) == 3:
            d["a0"] = t
        elif kind == 3 and int(tag) == 3:
            d["a1"] = t
    out = {}
    for i, d in sorted(per.items()):
        if {"r0", "r1", "a0", "a1"} <= d.keys():
            inter = min(d["r1"], d["a1"]) - max(d["r0"], d["a0"])
            out[i] = {"reduce_ms": d["r1"] - d["r0"], "as_ms": d["a1"] - d["a0"],
                      "overlap_ms": max(inter, 0.0), "overlapped": inter > 0}
    return out
