"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): total and per kernel/grid.

    python tools/launch_summary.py launches.csv [top]
"""
import collections
import csv
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    rows = [r for r in csv.DictReader(line for line in open(path) if not line.startswith("=="))
            if r.get("Metric Name") == "gpu__time_duration.sum"]
    agg = collections.OrderedDict()
    tot = 0.0
    for r in rows:
        v = float(r["Metric Value"].replace(",", "")) * UNIT[r["Metric Unit"]]
        name = r["Kernel Name"]
        if "frchol_panel" in name:
            k = "frchol_panel_kernel"
        elif "dgemm_tc<128, 32" in name:
            k = "dgemm_tc 128x32 (panel update)"
        else:
            k = name.split("(")[0][:48] + " grid" + r.get("Grid Size", "")
        a = agg.setdefault(k, [0.0, 0])
        a[0] += v
        a[1] += 1
        tot += v
    print(f"total {tot:.1f} us over {len(rows)} launches (serialised, cold L2)")
    for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{v:10.1f} us {100 * v / tot:5.1f}%  n={n:4d}  {k}")


if __name__ == "__main__":
    main()
