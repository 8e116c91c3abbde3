"""Summarise `ncu --page details --csv` exports: one block of key metrics per kernel launch."""
import csv
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Limit Shared Mem",
        "Block Limit Registers", "Grid Size", "Waves Per SM", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active",
        "Issue Slots Busy", "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler"]


def main(paths):
    for path in paths:
        rows = list(csv.reader(open(path)))
        idx = {h: i for i, h in enumerate(rows[0])}
        out = {}
        for r in rows[1:]:
            if len(r) <= idx["Metric Value"]:
                continue
            k = (r[idx["ID"]], r[idx["Kernel Name"]].split("(")[0])
            m = r[idx["Metric Name"]]
            if m in WANT:
                out.setdefault(k, {})[m] = f"{r[idx['Metric Value']]} {r[idx['Metric Unit']]}"
        for k, v in out.items():
            print(path, *k)
            for m in WANT:
                if m in v:
                    print(f"    {m:36s} {v[m]}")


if __name__ == "__main__":
    main(sys.argv[1:])
