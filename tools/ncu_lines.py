"""Aggregate an ncu source-page CSV (SASS level) by CUDA source line (file:line) using nvdisasm -g.

    ncu -i rep.ncu-rep --page source --csv > x.csv
    nvcc ... -cubin -o k.cubin file.cu && nvdisasm -g -c k.cubin > k.dis
    python tools/ncu_lines.py x.csv k.dis <kernel-substring> [top]
"""
import csv
import re
import sys


def main():
    csvp, disp, kname = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(csvp)))
    hdr = rows[1]
    data = rows[2:]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iA = hdr.index("Address")
    iE = hdr.index("Instructions Executed")
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    idx = {h: hdr.index(h) for h in stalls}
    off2line = {}
    cur = None
    infn = False
    for l in open(disp):
        if l.startswith("\t.section") or l.startswith(".section"):
            infn = kname in l and ".text." in l
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]+)\*/", l)
        if m and cur is not None:
            off2line[int(m.group(1), 16)] = cur
    addrs = [int(r[iA], 16) for r in data if r[iA].startswith("0x")]
    base = min(addrs)
    agg = {}
    tot = 0.0
    for r in data:
        if not r[iA].startswith("0x"):
            continue
        ln = off2line.get(int(r[iA], 16) - base, ("?", 0))
        v = float(r[iS] or 0)
        tot += v
        a = agg.setdefault(ln, [0.0, 0.0, {}])
        a[0] += v
        a[1] += float(r[iE] or 0)
        for h in stalls:
            a[2][h] = a[2].get(h, 0.0) + float(r[idx[h]] or 0)
    srcs = {}
    print(f"mapped {len(off2line)} offsets; total samples {tot:.0f}")
    for (f, ln), (v, e, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        tops = sorted(st.items(), key=lambda x: -x[1])[:2]
        if f not in srcs:
            try:
                srcs[f] = open(next(p for p in ["paper_0804_4809_b200/csrc/" + f] if p)).read().split("\n")
            except Exception:
                srcs[f] = []
        txt = srcs[f][ln - 1].strip()[:60] if 0 < ln <= len(srcs[f]) else ""
        print(f"{v / tot * 100:5.1f}% {f}:{ln:<4d} exec {e:9.3g} "
              f"{','.join(f'{k[6:]}={w / tot * 100:.1f}' for k, w in tops):34s} {txt}")


if __name__ == "__main__":
    main()
