"""Rewrite the results rows of DESIGN.md §8 from profiles/r01_bench_*.json (the lines tools/bench_all.sh
writes), so the table always quotes the committed bench lines.

    python tools/design_table.py
"""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def L(w):
    return json.load(open(os.path.join(ROOT, "profiles", f"r01_bench_{w}_n1.json")))


def row(ln):
    if ln.startswith("| C4 2^21 x 4096 r3584 (seed 5) |"):
        d = L("c4"); ph = d["config"]["phase_ms_rank0"]
        ln = re.sub(r"^\| C4 2\^21 x 4096 r3584 \(seed 5\) \| [^|]+\| [^|]+\| [^|]+\| [^|]+\| [^|]+\| [^|]+\| Gram \d+ ms, "
                    r"factorisation chain [\d.]+ ms",
                    f"| C4 2^21 x 4096 r3584 (seed 5) | {d['ms_per_step'] / 1e3:.3f} s | {d['value']:,.0f} | "
                    f"{100 * d['config']['pct_fp64_peak']:.1f} % | {100 * d['roofline']['frac']:.1f} % | "
                    f"{d['e2e']['value']:,.0f} GFLOP/s | {d['cpu_baseline']['value']:.0f} | Gram "
                    f"{ph['gram_allreduce_ms']:.0f} ms, factorisation chain {ph['factor_inverse_x_ms']:.1f} ms", ln)
        return re.sub(r"output \d+ ms;", f"output {ph['output_ms']:.0f} ms;", ln)
    if ln.startswith("| C4, Gram + a7 emulated"):
        d = L("c4_emulated"); ph = d["config"]["phase_ms_rank0"]; r = d["roofline"]
        return (f"| C4, Gram + a7 emulated (`--emulate`) | {d['ms_per_step'] / 1e3:.3f} s | {d['value']:,.0f} | -- | "
                f"{r['fp64_equivalent_tflops']:.1f} TFLOP/s FP64-eq. ({r['achieved'] / 1e3:.2f} POPS int8 = "
                f"{100 * r['frac']:.0f} % of the sustained int8 peak {r['peak'] / 1e3:.2f}; SM clock "
                f"~{d['clocks']['sm_mhz'] / 1e3:.2f} GHz, power-capped) | {d['e2e']['value']:,.0f} GFLOP/s | "
                f"{d['cpu_baseline']['value']:.0f} | `profiles/r01_bench_c4_emulated_n1.json`; Gram "
                f"{ph['gram_allreduce_ms']:.0f} ms (native 1040), chain {ph['factor_inverse_x_ms']:.0f} ms, a7 "
                f"{ph['output_ms']:.0f} ms (native 1951); `sw_power_cap` |")
    if ln.startswith("| C3T, Gram + a7 emulated |"):
        d = L("c3t_emulated"); ph = d["config"]["phase_ms_rank0"]; r = d["roofline"]
        return (f"| C3T, Gram + a7 emulated | {d['ms_per_step']:.2f} ms | {d['value']:,.0f} | -- | "
                f"{r['fp64_equivalent_tflops']:.1f} TFLOP/s FP64-eq. ({100 * r['frac']:.0f} % of the int8 peak "
                f"{r['peak'] / 1e3:.2f} POPS) | {d['e2e']['value']:,.0f} GFLOP/s | {d['cpu_baseline']['value']:.0f} | "
                f"Gram {ph['gram_allreduce_ms']:.1f} ms (native 8.4), a7 {ph['output_ms']:.1f} ms (native 15.4); "
                f"`profiles/r01_bench_c3t_emulated_n1.json` |")
    if ln.startswith("| C3, Gram + a7 emulated"):
        d = L("c3_emulated"); r = d["roofline"]
        return (f"| C3, Gram + a7 emulated (T branch: a7 = G'X from column digit planes of G) | {d['ms_per_step']:.2f} ms"
                f" | {d['value']:,.0f} | -- | {r['fp64_equivalent_tflops']:.1f} TFLOP/s FP64-eq. ({100 * r['frac']:.0f} % "
                f"of {r['peak'] / 1e3:.2f} POPS) | {d['e2e']['value']:,.0f} GFLOP/s | {d['cpu_baseline']['value']:.0f} | "
                f"`profiles/r01_bench_c3_emulated_n1.json` |")
    if ln.startswith("| C2, a7 emulated"):
        d = L("c2_emulated"); r = d["roofline"]
        return (f"| C2, a7 emulated (Gram on DMMA: s < 3072) | {d['ms_per_step']:.2f} ms | {d['value']:,.0f} | -- | "
                f"{r['fp64_equivalent_tflops']:.1f} TFLOP/s FP64-eq. | {d['e2e']['value']:,.0f} GFLOP/s | "
                f"{d['cpu_baseline']['value']:.0f} | `profiles/r01_bench_c2_emulated_n1.json` |")
    if ln.startswith("| C3T 16384 x 4096 r3072 |"):
        d = L("c3t"); ph = d["config"]["phase_ms_rank0"]
        return (f"| C3T 16384 x 4096 r3072 | {d['ms_per_step']:.2f} ms | {d['value']:,.0f} | "
                f"{100 * d['config']['pct_fp64_peak']:.1f} % | {100 * d['roofline']['frac']:.1f} % | "
                f"{d['e2e']['ms_per_step']:.1f} ms | {d['cpu_baseline']['value']:.0f} | Gram {ph['gram_allreduce_ms']:.2f},"
                f" chain {ph['factor_inverse_x_ms']:.2f} (was 12.6 at the start of the previous session), output "
                f"{ph['output_ms']:.2f} ms |")
    if ln.startswith("| C3 4096 x 16384 r3072 (T branch) |"):
        d = L("c3")
        return (f"| C3 4096 x 16384 r3072 (T branch) | {d['ms_per_step']:.2f} ms | {d['value']:,.0f} | "
                f"{100 * d['config']['pct_fp64_peak']:.1f} % | {100 * d['roofline']['frac']:.1f} % | "
                f"{d['e2e']['ms_per_step']:.1f} ms | {d['cpu_baseline']['value']:.0f} | whole-call geninv_d |")
    if ln.startswith("| C2 4096 x 1024 |"):
        d = L("c2")
        return (f"| C2 4096 x 1024 | {d['ms_per_step']:.2f} ms | {d['value']:,.0f} | {100 * d['config']['pct_fp64_peak']:.1f}"
                f" % | {100 * d['roofline']['frac']:.1f} % | {d['e2e']['ms_per_step']:.2f} ms | "
                f"{d['cpu_baseline']['value']:.0f} | L2 flushed per step; latency-bound chain (64 panels of ~11.5 us + "
                f"gaps): was 2.96 ms at the start of the previous session |")
    if ln.startswith("| C1 64 x 48 r32 |"):
        d = L("c1")
        return re.sub(r"^\| C1 64 x 48 r32 \| [^|]+\| [^|]+\| -- \| -- \| [^|]+\|",
                      f"| C1 64 x 48 r32 | {d['ms_per_step']:.3f} ms | {d['value']:.0f} | -- | -- | "
                      f"{d['e2e']['ms_per_step']:.3f} ms |", ln)
    if ln.startswith("| C5 65,536 x 96 x 64 |"):
        d = L("c5")
        ln = re.sub(r"^\| C5 65,536 x 96 x 64 \| [^|]+\| [^|]+\| [^|]+\|",
                    f"| C5 65,536 x 96 x 64 | {d['ms_per_step']:.2f} ms | {d['value']:,.0f} | "
                    f"{100 * d['roofline']['frac']:.1f} % |", ln)
        return re.sub(r"\| [\d.]+ ms \(PCIe: 3.2 GB each way\)", f"| {d['e2e']['ms_per_step']:.1f} ms (PCIe: 3.2 GB each way)", ln)
    return ln


def main():
    p = os.path.join(ROOT, "DESIGN.md")
    s = open(p).read()
    open(p, "w").write("\n".join(row(ln) for ln in s.split("\n")))


if __name__ == "__main__":
    main()
