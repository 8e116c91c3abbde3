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


def stamps_to_records(stamps, spine: str = "As") -> list[tuple[int, int, int, float]]:
    """Device-clock stamps of one partition ([iterations, 8]: As start/end, Aw
    start/end, publish start/end and finalize start/end of check i, ns; -1
    absent) -> schedule records (iter, kind, tag, t) in the reference's
    vocabulary: the reduction of check i starts when its record is published
    and ends (coefficients ready) when its finalize has run; the products are
    the As and Aw SpMVs of iteration i."""
    spine_tag = {"As": 3, "Ar": 2}[spine]  # ssBiCGSafe2's spine product is s = A r
    recs = []
    for i, row in enumerate(np.asarray(stamps)):
        as0, as1, aw0, aw1, pub0, _pub1, _fin0, fin1 = (float(v) for v in row)
        if as0 < 0:
            # no spine product: the record after max_iters, which the reference
            # takes with plan_dot outside the loop (solvers.py:736-739), not as a
            # batch reduction -- its log has no events for it either
            continue
        if pub0 >= 0:
            recs.append((i, 0, 0, pub0))
        if fin1 >= 0:
            recs.append((i, 1, 0, fin1))
            recs.append((i, 4, 0, fin1))
        if as0 >= 0 and as1 >= 0:
            recs.append((i, 2, spine_tag, as0))
            recs.append((i, 3, spine_tag, as1))
        if aw0 >= 0 and aw1 >= 0:
            recs.append((i, 2, 4, aw0))
            recs.append((i, 3, 4, aw1))
    return recs


def events_to_log(records) -> EventLog:
    """Schedule records (iter, kind, tag, t) -> the reference's EventLog.

    seq follows the device timestamps (ties keep record order), so the
    reference's verify_phase_order (reduction.py:486-563) can be re-run on it.
    """
    recs = [(float(t), k, int(i), int(kind), int(tag)) for k, (i, kind, tag, t) in enumerate(records)]
    recs.sort(key=lambda r: (r[0], r[1]))
    log = EventLog()
    for t, _, i, kind, tag in recs:
        log.append(i, _KINDS[kind], _TAGS.get(tag))
    return log


def overlap_report(stamps) -> dict:
    """Per iteration i of one partition's device-clock stamps: the reduction of
    check i ([publish start, finalize end]) against the As SpMV of iteration
    i.  overlapped: the intervals intersect; hidden: the coefficients were
    ready before A s finished, i.e. the reduction cost the iteration nothing."""
    out = {}
    for i, row in enumerate(np.asarray(stamps)):
        as0, as1, _aw0, _aw1, pub0, _pub1, _fin0, fin1 = (float(v) for v in row)
        if min(as0, as1, pub0, fin1) < 0:
            continue
        inter = min(fin1, as1) - max(pub0, as0)
        out[i] = {"reduce_us": (fin1 - pub0) / 1e3, "as_us": (as1 - as0) / 1e3,
                  "overlap_us": max(inter, 0.0) / 1e3, "overlapped": inter > 0, "hidden": fin1 <= as1}
    return out
