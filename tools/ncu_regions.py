"""Stall samples of a sell/csr pipe kernel by role, from the gzipped `ncu --page source --csv` export:
every mbarrier wait (SYNCS.PHASECHK + its branch) with its samples, and the totals."""
import csv, gzip, sys
rows = list(csv.reader(gzip.open(sys.argv[1], "rt")))
kernel = None; hdr = None; out = {}
for r in rows:
    if not r: continue
    if r[0] == "Kernel Name": kernel = r[1]; hdr = None; continue
    if r[0] == "Address": hdr = r; continue
    if hdr is None: continue
    out.setdefault(kernel, []).append(dict(zip(hdr, r)))
for k, ins in out.items():
    ins = ins[: len(ins) // 2] if len(ins) > 4000 else ins  # the export lists each function twice
    S = lambda d: int(d["Warp Stall Sampling (All Samples)"] or 0)
    X = lambda d: int(d.get("Instructions Executed") or 0)
    tot = sum(S(d) for d in ins)
    print("==", k[:90], "samples", tot, "warp-instructions", sum(X(d) for d in ins))
    for i, d in enumerate(ins):
        if "SYNCS.PHASECHK" in d["Source"] and X(d) > 0:
            s = S(d) + (S(ins[i + 1]) if i + 1 < len(ins) else 0)
            print(f"   wait @{i:5d} exec {X(d):8d} samples {s:5d} ({100*s/max(tot,1):4.1f}%)  {d['Source'].strip()[:70]}")
