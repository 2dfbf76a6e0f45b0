"""Per-launch table from an ncu --csv metrics/sections dump: kernel, grid, duration, DMMA pipe %, achieved
occupancy, registers, bank conflicts, top warp-state metrics (measurement tool).

    python tools/ncu_table.py dump.csv
"""
import csv
import sys
from collections import OrderedDict

WANT = {
    "gpu__time_duration.sum": "us", "Duration": "us",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma%",
    "Achieved Occupancy": "occ%", "Registers Per Thread": "regs",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "bank_confl",
    "Warp Cycles Per Issued Instruction": "cyc/issue", "gpc__cycles_elapsed.avg.per_second": "clk",
    "dram__bytes_read.sum": "dram_rd", "dram__bytes_write.sum": "dram_wr",
}


def main():
    rows = [r for r in csv.DictReader(line for line in open(sys.argv[1]) if line.startswith('"'))]
    launches = OrderedDict()
    for r in rows:
        key = r["ID"]
        d = launches.setdefault(key, {"kernel": r["Kernel Name"], "grid": r.get("Grid Size", "")})
        name = r.get("Metric Name", "")
        if name in WANT:
            v = r["Metric Value"].replace(",", "")
            unit = r.get("Metric Unit", "")
            try:
                x = float(v)
            except ValueError:
                continue
            if WANT[name] == "us":
                x = x / 1e3 if unit in ("nsecond", "ns") else (x * 1e3 if unit in ("msecond", "ms") else x)
            if WANT[name] == "clk" and unit in ("hz",):
                x /= 1e9
            d[WANT[name]] = x
    cols = ["us", "dmma%", "occ%", "regs", "bank_confl", "cyc/issue", "clk", "dram_rd", "dram_wr"]
    print("| kernel | grid | " + " | ".join(cols) + " |")
    print("|---|---|" + "---|" * len(cols))
    for d in launches.values():
        k = d["kernel"].replace("void gi::", "").replace("(int)", "").replace("(bool)", "").split("(gi::")[0]
        vals = []
        for c in cols:
            x = d.get(c)
            vals.append("" if x is None else (f"{x:.1f}" if abs(x) < 1e6 else f"{x:.3g}"))
        print(f"| {k} | {d['grid']} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
