"""The reference's own schedule verifier on device-produced evidence.

profiles/r2/evidence/ holds EventLog JSONL files (the reference's schema,
reduction.py:136-178) written by tools/schedule_evidence.py from the
%globaltimer stamps of partitioned solves on a B200: p-BiCGSafe and
ssBiCGSafe2 on config 2, as the one-partition path and as loopback groups of
2 and 4 partitions.  Here the reference's verify_phase_order
(reduction.py:486-563, test_acceptance.py:248-288 criterion 6) is imported
from /root/reference and run on them unchanged: p-BiCGSafe's one reduction
per iteration starts before its As product ends (the overlap), ssBiCGSafe2's
starts only after A r is complete.
"""

import glob
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EVIDENCE = os.path.join(ROOT, "profiles", "r2", "evidence")
REF_SRC = "/root/reference/pkg/src"


def _reference_reduction():
    if not os.path.isdir(REF_SRC):
        pytest.skip("the reference is not in this container")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    try:
        from pipesafe import reduction
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"cannot import the reference: {e}")
    return reduction


def _logs():
    return sorted(glob.glob(os.path.join(EVIDENCE, "eventlog_*.jsonl")))


@pytest.mark.parametrize("path", _logs(), ids=os.path.basename)
def test_reference_verify_phase_order_on_device_log(path):
    red = _reference_reduction()
    method = "ssbicgsafe2" if "ssbicgsafe2" in os.path.basename(path) else "pbicgsafe"
    log = red.EventLog.read_jsonl(path)
    rep = red.verify_phase_order(log, method)
    assert rep.ok, rep.violations[:5]
    assert rep.iterations_checked >= 99


def test_evidence_covers_both_methods_and_partition_counts():
    names = {os.path.basename(p) for p in _logs()}
    for method in ("pbicgsafe", "ssbicgsafe2"):
        for n in (1, 2, 4):
            assert any(nm.startswith(f"eventlog_{method}_n{n}_") for nm in names), (method, n)
    summ = json.load(open(os.path.join(EVIDENCE, "overlap_summary.json")))["results"]
    # device clock: p-BiCGSafe's reduction runs while As computes; ssBiCGSafe2's cannot
    for p, r in summ["pbicgsafe_n2"].items():
        assert r["reduce_overlaps_spine_frac"] >= 0.9, (p, r)
    for p, r in summ["ssbicgsafe2_n2"].items():
        assert r["reduce_overlaps_spine_frac"] == 0.0, (p, r)
