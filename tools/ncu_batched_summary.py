"""Summary of one ncu --set full report of the batched kernel: speed-of-light, occupancy, pipe use, stall
reasons and the per-matrix instruction mix (measurement tool; writes the text that profiles/ keeps).

    python tools/ncu_batched_summary.py report.ncu-rep batch
"""
import collections
import csv
import io
import subprocess
import sys


def page(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, nb = sys.argv[1], int(sys.argv[2])
    raw = page(rep, "--page", "raw")
    d = dict(zip(raw[0], raw[2]))
    u = dict(zip(raw[0], raw[1]))
    f = lambda k: float(d[k].replace(",", ""))
    print(f"# ncu --set full, batched_geninv_kernel, {nb} matrices (C5), {rep.split('/')[-1]}")
    print(f"duration {f('gpu__time_duration.sum'):.3f} {u['gpu__time_duration.sum']}, "
          f"SM clock {f('smsp__cycles_elapsed.avg.per_second'):.3f} {u['smsp__cycles_elapsed.avg.per_second']}")
    for k, name in [("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active %"),
                    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 (SIMT) pipe %"),
                    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (occupancy)"),
                    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
                    ("launch__registers_per_thread", "registers / thread"),
                    ("launch__occupancy_limit_shared_mem", "CTA limit: shared memory"),
                    ("launch__occupancy_limit_registers", "CTA limit: registers"),
                    ("dram__bytes_read.sum", "DRAM bytes read"), ("dram__bytes_write.sum", "DRAM bytes written"),
                    ("smsp__inst_executed.sum", "warp instructions executed")]:
        if k in d:
            print(f"  {name:34s} {f(k):,.2f} {u.get(k, '')}")
    st = [(f(k), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in d
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and d[k]]
    tot = sum(a for a, _ in st)
    print("stall reasons (share of PC samples):")
    for a, k in sorted(st, reverse=True)[:10]:
        print(f"  {k:28s} {a / tot * 100:5.1f} %")
    rows = page(rep, "--page", "source", "--print-source", "sass")
    h = rows[1]
    iS, iE = h.index("Source"), h.index("Instructions Executed")
    mix = collections.Counter()
    for r in rows[2:]:
        if len(r) > iE and r[iE].replace(",", "").isdigit():
            w = r[iS].split()
            op = (w[1] if w and w[0].startswith("@") and len(w) > 1 else (w[0] if w else "?")).split(".")[0]
            mix[op] += int(r[iE].replace(",", ""))
    tot = sum(mix.values())
    print(f"warp instructions per matrix: {tot / nb:,.0f}; mix:")
    for op, c in mix.most_common(14):
        print(f"  {op:10s} {c / nb:8,.0f}  {c / tot * 100:5.1f} %")


if __name__ == "__main__":
    main()
