"""Summarise bench JSON lines: python tools/bsum.py file.json ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:  # noqa: BLE001
        print(f"== {f}: {e}")
        continue
    c = d.get("config", {})
    print(f"== {f}: {d['value']:.1f} it/s, {d['ms_per_step']:.2f} ms/solve, {c.get('iterations_per_solve')} it")
    ir = d.get("iteration_roofline", {})
    print("   iteration roofline frac %.3f" % ir.get("frac", float("nan")),
          "own %.3f" % ir["frac_own_schedule"] if "frac_own_schedule" in ir else "")
    print("   kernels", {k: (round(v["avg_us"], 1), round(v["frac"], 3)) for k, v in d.get("kernels", {}).items()
                         if isinstance(v, dict) and "avg_us" in v and "frac" in v})
    o = d.get("overlap")
    if o:
        print("   overlap hidden %.2f reduce %.1f us As %.1f us" % (o["hidden_frac"], o["reduce_us_median"] or 0,
                                                                  o["as_us_median"] or 0))
    if d.get("e2e"):
        print("   e2e %.1f" % d["e2e"]["value"])
