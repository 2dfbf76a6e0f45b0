"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: time share per kernel."""
import collections
import csv
import io
import sys


def load(path):
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))


def summarise(path, top=30):
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        if "dgemm_tc" in name:
            key = name[name.index("dgemm_tc"):name.index(">") + 1] + " grid" + r["Grid Size"]
        else:
            key = name.split("(")[0][-80:]
        v = float(r["Metric Value"].replace(",", "")) * unit[r["Metric Unit"]]
        agg[key][0] += 1
        agg[key][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"total {tot:.2f} ms over {sum(v[0] for v in agg.values())} launches"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{v[1]:12.3f} ms {100 * v[1] / tot:6.2f}%  n={v[0]:5d}  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
