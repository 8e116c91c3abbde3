"""Top stalled SASS instructions per kernel from `ncu --page source --csv --print-source sass`."""
import csv
import sys


def main(path, top=25):
    kernel, hdr, rows = None, None, []
    out = {}
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "Kernel Name":
            kernel = r[1]
            hdr = None
            continue
        if r[0] == "Address":
            hdr = r
            continue
        if hdr is None:
            continue
        d = dict(zip(hdr, r))
        out.setdefault(kernel, []).append(d)
    for k, ins in out.items():
        tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in ins)
        print(f"== {k[:110]}  total samples {tot}")
        ins.sort(key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))
        for d in ins[:top]:
            s = int(d["Warp Stall Sampling (All Samples)"] or 0)
            stalls = {h[6:]: int(v) for h, v in d.items() if h.startswith("stall_") and "Not Issued" not in h
                      and v.isdigit() and int(v) > 0.15 * max(s, 1)}
            print(f"{s:7d} {100*s/max(tot,1):5.1f}%  {d['Address'][-5:]} {d['Source'].strip()[:60]:60s} {stalls}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
