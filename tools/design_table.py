"""Rewrite the results rows of DESIGN.md §8 from profiles/r02_bench_*.json (the lines tools/bench_all.sh
writes), so the table always quotes the committed bench lines.

    python tools/design_table.py [round]      # default r02
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RND = sys.argv[1] if len(sys.argv) > 1 else "r02"


def L(w):
    return json.load(open(os.path.join(ROOT, "profiles", f"{RND}_bench_{w}_n1.json")))


def clk(d):
    c = d.get("clocks") or {}
    rs = [r for r in c.get("reasons", []) if r]
    return f"{c.get('sm_mhz', 0):.0f} MHz" + (" " + ", ".join(rs) if rs else "")


def t(d):
    ms = d["ms_per_step"]
    return f"{ms / 1e3:.3f} s" if ms >= 1000 else f"{ms:.3f} ms"


def phases(d):
    ph = d["config"].get("phase_ms_rank0") or {}
    if not ph:
        return ""
    f = (lambda v: f"{v:.1f}") if ph["gram_allreduce_ms"] >= 100 else (lambda v: f"{v:.2f}" if v >= 1 else f"{v:.1f}")
    return (f"Gram {f(ph['gram_allreduce_ms'])}, chain {ph['factor_inverse_x_ms']:.2f}, "
            f"a7 {f(ph['output_ms'])} ms; ")


def native(label, w):
    d = L(w)
    r = d["roofline"]
    return (f"| {label} | {t(d)} | {d['value']:,.0f} | {100 * d['config']['pct_fp64_peak']:.1f} % | "
            f"{100 * r['frac']:.1f} % | {d['e2e']['value']:,.0f} | {d['cpu_baseline']['value']:.0f} | "
            f"{phases(d)}{clk(d)}; {d['gpu_launches']} launches |")


def emulated(label, w):
    d = L(w)
    r = d["roofline"]
    return (f"| {label} | {t(d)} | {d['value']:,.0f} | -- | {r['fp64_equivalent_tflops']:.1f} TF FP64-eq. "
            f"({100 * r['frac']:.0f} % of int8 {r['peak']:.0f}) | {d['e2e']['value']:,.0f} | "
            f"{d['cpu_baseline']['value']:.0f} | {phases(d)}{clk(d)}; {d['gpu_launches']} launches |")


def rows():
    out = {
        "| C4 2^21": native("C4 2^21 x 4096 r3584 (seed 5)", "c4"),
        "| C4, Gram + a7 emulated": emulated("C4, Gram + a7 emulated", "c4_emulated"),
        "| C3T 16384": native("C3T 16384 x 4096 r3072", "c3t"),
        "| C3T, emulated": emulated("C3T, emulated", "c3t_emulated"),
        "| C3 4096": native("C3 4096 x 16384 r3072 (T branch)", "c3"),
        "| C3, emulated": emulated("C3, emulated", "c3_emulated"),
        "| C2 4096": native("C2 4096 x 1024", "c2"),
        "| C2, a7 emulated": emulated("C2, a7 emulated", "c2_emulated"),
    }
    d = L("c1")
    out["| C1 64"] = (f"| C1 64 x 48 r32 | {t(d)} | {d['value']:,.0f} | -- | (one kernel) | {d['e2e']['value']:,.0f} | "
                      f"{d['cpu_baseline']['value']:.0f} | one-CTA path; {clk(d)}; {d['gpu_launches']} launches |")
    d = L("c5")
    out["| C5 65,536"] = (f"| C5 65,536 x 96 x 64 | {t(d)} | {d['value']:,.0f} | {100 * d['roofline']['frac']:.1f} % | "
                          f"(one kernel) | {d['e2e']['value']:,.0f} | {d['cpu_baseline']['value']:.0f} | "
                          f"{d['config']['us_per_matrix']:.3f} us/matrix (round 1: 11.59 ms); {clk(d)}; "
                          f"{d['gpu_launches']} launches |")
    d = L("reference")
    out["| reference arm"] = (f"| reference arm (the oracle on a 16384-row sample of C4) | {t(d)} | {d['value']:,.0f} | "
                              f"-- | -- | -- | {d['value']:,.0f} | `profiles/{RND}_bench_reference_n1.json`, "
                              f"{d['cpu_baseline']['cores']} host cores |")
    return out


def main():
    p = os.path.join(ROOT, "DESIGN.md")
    lines = open(p).read().split("\n")
    new = rows()
    n = 0
    for i, ln in enumerate(lines):
        for k, v in new.items():
            if ln.startswith(k):
                if lines[i] != v:
                    n += 1
                lines[i] = v
    open(p, "w").write("\n".join(lines))
    print(f"{n} rows updated")


if __name__ == "__main__":
    main()
