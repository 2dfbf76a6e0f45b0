"""bench.py -- geninv FP64 throughput on B200 (the BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4|C3T|C3|C2|C5] [--impl ours|reference]

Default workload: C4, the tall 2,097,152 x 4096 matrix of exact rank 3584
(BASELINE.json configs[3]), rows sharded over the N ranks: each rank forms
its partial Gram G_p'G_p, one NCCL all-reduce sums A, the factorisation and
inverse run replicated, and each rank writes its own column block of G+
(SURVEY §8(e)).  One step = one whole geninv of the workload (a1-a8).
Total work is fixed as N grows ("scaling": "strong").

value      = F_alg / (max-over-ranks device time per step), GFLOP/s, inputs resident in HBM
e2e        = the same through the C ABI with HOST buffers (pinned), copies inside the timed region
roofline   = the dominant kernel (the a7 output product, DMMA) against the measured FP64 DMMA peak
cpu_baseline = the oracle (numpy, paper's algorithm) on a bounded row sample of the same workload

--impl reference times the oracle itself (the deliberately slow CPU reference) on that sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_0804_4809_b200 import inputs as I  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "MEASURED_FP64.json")
SEED = 1


# digit products of the emulated contractions (csrc/emu.cu: 7 digits, groups t + u <= T, T = 9)
_EMU_T = int(os.environ.get("GENINV_EMU_T", "9"))
EMU_PAIRS = sum(1 for t in range(1, 8) for u in range(1, 8) if t + u <= _EMU_T)


def seed_of(cfg) -> int:
    """The seed the parity tests use for this config (inputs.QSEED: the oracle's margins are in Q)."""
    return I.QSEED.get(cfg.name if cfg.name != "C3T" else "C3", SEED)


# --------------------------------------------------------------------------- flop model
def fullrank_direct() -> bool:
    """The library evaluates r = s through L^-1 (DESIGN reading R27) unless GENINV_FULLRANK_DIRECT=0."""
    return os.environ.get("GENINV_FULLRANK_DIRECT", "1") != "0"


def f_alg(s: int, ell: int, piv: np.ndarray, direct: bool = False) -> dict:
    """Algorithmic FP64 flops of one geninv in the evaluation order that runs (SURVEY §8(a) convention: SYRKs
    count one triangle).  direct (r = s, R27): X = L^-T L^-1 as one TRTRI (s^3/3) and one LAUUM (s^3/3) in
    place of L'L, the SPD inverse and K, X."""
    r = len(piv)
    k = np.arange(s)
    rk = np.searchsorted(np.sort(piv), k, side="left")      # columns accepted before column k
    chol = float(np.sum(2.0 * (s - k) * rk + (s - k)))
    if direct and r == s:
        parts = {"gram": float(ell) * s * (s + 1), "chol": chol, "inv": 2.0 * float(s) ** 3 / 3.0,
                 "out": 2.0 * s * s * ell}
    else:
        parts = {
            "gram": float(ell) * s * (s + 1),
            "chol": chol,
            "ltl": float(s) * r * (r + 1),
            "inv": float(r) ** 3,
            "kx": 2.0 * s * r * r + float(s) * (s + 1) * r,
            "out": 2.0 * s * s * ell,
        }
    parts["total"] = sum(parts.values())
    return parts


def fp64_peak():
    try:
        d = json.load(open(FP64_PEAK_FILE))
        return d["dmma_tflops"], "measured (profiles/MEASURED_FP64.json: register-resident DMMA.8x8x4 microbenchmark)"
    except Exception:
        return 37.2, "nominal 148 SM x 128 flop/clk x 1.965 GHz (no measured FP64 peak file)"


def int8_peak(long_step):
    """Dense INT8 tensor peak (TOPS) for the emulated products: the driver-measured bf16 cuBLAS peak
    (MEASURED_PEAKS.json; burst for a short step, sustained for a kernel inside a long step) times
    the nominal INT8 / BF16 ratio 4.5 / 2.25 = 2; else the nominal 4.5 POPS."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        key = "bf16_tflops_sustained" if long_step else "bf16_tflops"
        return 2.0 * d[key], (f"MEASURED_PEAKS.json {key} ({d[key]:.1f} TFLOP/s) x 2, the nominal INT8 / BF16 "
                              f"dense ratio (4.5 / 2.25 POPS); tools/i8gemm.cu, a plain tcgen05 int8 GEMM, reaches 2.4 POPS")
    except Exception:
        return 4500.0, "nominal B200 dense INT8 4.5 POPS (no MEASURED_PEAKS.json)"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t_end = time.time() + 3.0                  # the sampler is running before the region starts
            while not self.lines and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
            self.n0 = len(self.lines)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            n_in = len(self.lines) - getattr(self, "n0", 0)
            if n_in < 1:                               # region shorter than the 200 ms period: one more
                try:                                   # sample right at its end (clocks still at load)
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=10).stdout.strip()
                    if out:
                        self.lines.append(out.splitlines()[-1])
                        self.short = True
                except Exception:
                    pass
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[max(0, getattr(self, "n0", 0) - 1):]:   # from the last sample before the region
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        out = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}
        if getattr(self, "short", False):
            out["note"] = "timed region shorter than the 200 ms sampling period: samples at its start and end"
        return out


# --------------------------------------------------------------------------- distributed
def dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        if world == 1 and n_gpus > 1:
            raise SystemExit(f"--gpus {n_gpus} needs torchrun --nproc-per-node {n_gpus}")
    if world > 1:
        import torch.distributed as dist
        # the one exchange (the all-reduce of A) pinned to one algorithm / protocol: its summation order is
        # then fixed run to run as well as identical on every rank (the replicated factorisation needs
        # bit-identical A); at ~0.1-0.3 ms against seconds of DMMA work the choice costs nothing
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def allsum(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


def allmax(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------- workloads
def workload(name: str):
    if name == "C4":
        return I.CONFIGS["C4"], False, "C4: tall G 2097152 x 4096 fp64, exact rank 3584 (U V, N(0,1)), rows sharded"
    if name == "C3T":
        c = I.CONFIGS["C3"]
        return I.Config("C3T", c.n, c.m, c.rank, ncopy=c.ncopy), True, \
            "C3 transposed: G' of the 4096 x 16384 rank-3072 matrix, i.e. 16384 x 4096 (N branch)"
    if name in ("C1", "C2", "C3", "C5"):
        return I.CONFIGS[name], False, f"{name}: BASELINE.json configs"
    raise SystemExit(f"unknown workload {name}")


def make_rows(cfg, transposed_of_c3, row0, rows, device):
    if transposed_of_c3:
        c3 = I.CONFIGS["C3"]
        G = I.make_single(c3, seed_of(c3), device=device)
        return G.T[row0:row0 + rows].contiguous()
    return I.make_single(cfg, seed_of(cfg), device=device, row0=row0, rows=rows)


# --------------------------------------------------------------------------- the reference arm (oracle)
def oracle_sample(cfg, transposed_of_c3):
    """A bounded sample of the workload for the CPU oracle: its first rows (C4: 16384 of 2^21 rows)."""
    if cfg.name in ("C4",):
        rows = 16384
        G = I.make_single(cfg, seed_of(cfg), rows=rows).numpy()
        return G, f"rows 0..{rows - 1} of the C4 matrix ({rows} x {cfg.n}, same generator, N branch)"
    if transposed_of_c3 or cfg.name == "C3":
        c3 = I.CONFIGS["C3"]
        cols = 4096
        G = I.make_single(c3, seed_of(c3)).numpy()
        G = G.T[:cols] if transposed_of_c3 else G[:, :cols].copy()
        return np.ascontiguousarray(G), f"{cols} of 16384 long-side lines of C3"
    if cfg.name == "C5":
        G = I.make_batch(cfg, seed_of(cfg), 0, 4096).numpy()
        return G, "matrices 0..4095 of the 65536-matrix batch"
    G = I.make_single(cfg, seed_of(cfg)).numpy()
    return G, "the whole matrix"


def run_oracle_once(G):
    from oracle import geninv_oracle as O
    t0 = time.perf_counter()
    if G.ndim == 3:
        Gp, r, _, _ = O.geninv_batched(G)
        dt = time.perf_counter() - t0
        m, n = G.shape[1:]
        s, ell = min(m, n), max(m, n)
        fl = sum(f_alg(s, ell, np.arange(int(rv)))["total"] for rv in r)  # rank-r leading columns (approx.)
        return fl, dt
    R = O.geninv(G)
    dt = time.perf_counter() - t0
    m, n = G.shape
    fl = f_alg(min(m, n), max(m, n), R.chol.piv)["total"]
    return fl, dt


def host_record():
    """The box's host CPU and the oracle's thread settings."""
    rec = {"cpu_model": None, "sockets": None, "cores_per_socket": None, "threads_per_core": None,
           "logical_cpus_usable": cpu_cores(), "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
           "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            v = v.strip()
            if k == "Model name":
                rec["cpu_model"] = v
            elif k == "Socket(s)":
                rec["sockets"] = int(v)
            elif k == "Core(s) per socket":
                rec["cores_per_socket"] = int(v)
            elif k == "Thread(s) per core":
                rec["threads_per_core"] = int(v)
    except Exception:
        pass
    try:
        from threadpoolctl import threadpool_info
        rec["blas"] = [{"api": d.get("internal_api"), "threads": d.get("num_threads")} for d in threadpool_info()
                       if d.get("user_api") == "blas"]
    except Exception:
        rec["blas"] = None
    return rec


def oracle_extra_times(dev):
    """1-thread oracle times for C1 and a 1024-matrix C5 slice, and the all-thread oracle on the FULL C3
    (SURVEY §8(d5)); inputs from the same generator (C3 formed on the device, as the bench's input)."""
    from threadpoolctl import threadpool_limits

    from oracle import geninv_oracle as O
    out = {}
    G1 = I.make_single(I.CONFIGS["C1"], seed_of(I.CONFIGS["C1"])).numpy()
    G5 = I.make_batch(I.CONFIGS["C5"], seed_of(I.CONFIGS["C5"]), 0, 1024).numpy()
    with threadpool_limits(limits=1):
        O.geninv(G1)
        t0 = time.perf_counter()
        for _ in range(20):
            O.geninv(G1)
        out["C1_1thread_ms"] = (time.perf_counter() - t0) / 20 * 1e3
        t0 = time.perf_counter()
        O.geninv_batched(G5)
        out["C5_1024_matrices_1thread_s"] = time.perf_counter() - t0
    c3 = I.CONFIGS["C3"]
    G3 = I.make_single(c3, seed_of(c3), device=dev).cpu().numpy()
    t0 = time.perf_counter()
    O.geninv(G3)
    out["C3_full_all_threads_s"] = time.perf_counter() - t0
    return out


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def reference_arm(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg, tr, desc = workload(args.workload)
    G, sample = oracle_sample(cfg, tr)
    for _ in range(args.warmup):
        run_oracle_once(G)
    fl_tot, dt_tot = 0.0, 0.0
    for _ in range(args.steps):
        fl, dt = run_oracle_once(G)
        fl_tot += fl
        dt_tot += dt
    v = fl_tot / dt_tot / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt_tot / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "sample": sample},
            "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": cpu_cores(), "kind": "oracle", "sample": sample,
                             "host": host_record()},
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--emulate", action="store_true",
                    help="a7 on the INT8 tensor cores (Ozaki-split FP64 emulation, SURVEY f4) instead of DMMA")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)

    from paper_0804_4809_b200.binding import Handle
    from paper_0804_4809_b200.sharded import row_range

    world, rank, local = dist_setup(args.gpus)
    cfg, c3t, desc = workload(args.workload)
    if cfg.batch > 1:
        return bench_batched(args, cfg, desc, world, rank)
    m, n = cfg.m, cfg.n
    tr = int(m < n)
    s, ell = min(m, n), max(m, n)
    colshard = bool(world > 1 and tr)   # wide G (C3): columns sharded, row blocks of G+ 
    dev = torch.device("cuda", local)

    # ---- inputs resident in HBM
    if colshard:
        row0, row1 = row_range(n, world, rank)          # this rank's columns of G
        rows = row1 - row0
        Gfull = make_rows(cfg, c3t, 0, m, dev)
        G = Gfull[:, row0:row1].contiguous()
        del Gfull
        Gp = torch.empty(rows, m, dtype=torch.float64, device=dev)   # row block of G+ (cols_p x m)
    else:
        row0, row1 = row_range(m, world, rank)
        rows = row1 - row0
        G = make_rows(cfg, c3t, row0, rows, dev) if world > 1 or not c3t else make_rows(cfg, c3t, 0, m, dev)
        Gp = torch.empty(n, rows, dtype=torch.float64, device=dev)   # local column block of G+ (n x rows)
    A = torch.zeros(s, s, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    h = Handle(local)
    if args.emulate:
        h.set_emulation(1)
    stream = torch.cuda.current_stream(dev)
    if world > 1:
        import torch.distributed as dist

    trans = 1 if colshard else tr
    comm = None
    if world > 1:
        t_ = torch.ones(1, device=dev)
        dist.all_reduce(t_)                          # creates the NCCL communicator
        comm = dist.distributed_c10d._get_default_group()._get_backend(dev)._comm_ptr()

    # The timed step is the product entry point a user calls: geninv_d (N = 1) or geninv_sharded_d
    # (N > 1: local Gram, ncclAllReduce of A inside the library, replicated factorisation, local block of
    # G+).  The phases and the a7 launch (the roofline kernel) are timed in separate untimed passes below.
    def step():
        if world > 1:
            _, info = h.geninv_sharded_d(comm, G, 1 if colshard else 0, Gp)
        else:
            _, info = h.geninv_d(G, Gp)
        return info

    info = step()
    torch.cuda.synchronize()
    # piv for the flop model (untimed): the full-rank Cholesky of the (all-reduced) Gram
    Aw = torch.zeros(s, s, dtype=torch.float64, device=dev)
    h.geninv_gram_d(G, trans, Aw)
    if world > 1:
        dist.all_reduce(Aw)
    _, piv, _ = h.geninv_frchol_d(Aw)
    piv = piv.cpu().numpy()
    del Aw
    F = f_alg(s, ell, piv, direct=fullrank_direct() and not (s <= 64 and ell <= 128))
    for _ in range(max(0, args.warmup - 1)):
        step()
    # inputs (G and G+) that fit in the 126 MB L2 are flushed between timed steps by writing a 512 MB
    # buffer; the step time is then the sum of per-step event pairs, the flushes outside them
    flush = (m * n * 8 * 2 < 512e6)
    fbuf = torch.empty(64 << 20, dtype=torch.float64, device=dev) if flush else None
    step_ev = []
    barrier(world)
    l0 = h.launch_count
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            if flush:
                fbuf.fill_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                info = step()
                b.record(stream)
                step_ev.append((a, b))
            else:
                info = step()
        t1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = (h.launch_count - l0) * world + (2 * args.steps * world if world > 1 else 0)  # + 2 NCCL all-reduces
    if flush:
        ms = float(sum(a.elapsed_time(b) for a, b in step_ev)) / args.steps
    else:
        ms = t0.elapsed_time(t1) / args.steps
    ms = allmax(ms, world)
    value = F["total"] / (ms * 1e-3) / 1e9
    peak, peak_src = fp64_peak()
    # cross-rank check of the replicated factorisation: every rank's (r, hash of X's bits) must agree
    replicated = None
    if world > 1:
        from paper_0804_4809_b200.sharded import check_replicated, replicated_digest
        if info.order == 0:
            replicated = bool(check_replicated(replicated_digest(h.geninv_copy_x(), info.rank)))
            if not replicated:
                raise SystemExit("replicated factorisation differs between ranks (r or X bits)")
    # dominant kernel: the a7 output product.  geninv_d / geninv_sharded_d launch it inside the call, so the
    # same launch is timed through geninv_apply_d right after the timed region: `steps` launches on the X the
    # timed calls left, each between CUDA events on the launching stream (the L2 flushed before each when the
    # inputs fit in it)
    roof_note = ("geninv_apply_d (the a7 launch geninv_d / geninv_sharded_d make, on the X the timed calls "
                 "left) x steps after the timed region, CUDA events around each on the launching stream")
    ev_out = []
    try:
        for _ in range(args.steps):
            if flush:
                fbuf.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            h.geninv_apply_d(G, trans, Gp)
            e1.record(stream)
            ev_out.append((e0, e1))
        torch.cuda.synchronize()
    except Exception as exc:   # the one-CTA small path (C1) and the low-rank K order keep no X
        ev_out.clear()
        roof_note = f"not separable: {str(exc)[:120]}"
    if ev_out:
        out_ms = float(np.mean([a.elapsed_time(b) for a, b in ev_out]))
        out_ms = allmax(out_ms, world)
        out_flops_launch = 2.0 * s * s * (ell if (tr and not colshard) else rows)   # this rank's long-side lines
        achieved = out_flops_launch / (out_ms * 1e-3) / 1e12
    else:
        out_ms, achieved, out_flops_launch = None, None, None
    # phases (one untimed pass of the split form, CUDA events between the stages; N > 1: torch's all-reduce)
    phases = None
    try:
        for _ in range(2):                           # the first pass captures the chain's CUDA graphs
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            A.zero_()
            torch.cuda.synchronize()
            evs[0].record(stream)
            h.geninv_gram_d(G, trans, A)
            if world > 1:
                dist.all_reduce(A)
            evs[1].record(stream)
            h.geninv_from_gram_d(A)
            evs[2].record(stream)
            h.geninv_apply_d(G, trans, Gp)
            evs[3].record(stream)
            torch.cuda.synchronize()
        phases = dict(zip(["gram_allreduce_ms", "factor_inverse_x_ms", "output_ms"],
                          [round(evs[i].elapsed_time(evs[i + 1]), 3) for i in range(3)]))
    except Exception as exc:
        phases = {"not separable": str(exc)[:120]}
    traffic = None
    try:
        tr_d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr_d.get(f"{args.workload}_out_bytes_per_launch")
    except Exception:
        pass
    rank_ok = info.rank if info is not None else None
    clocks = clk.summary()

    # ---- host copy of this rank's input (untimed), then free the device-resident buffers
    e2e = None
    Gh = None
    if not args.no_e2e:
        try:
            Gh = torch.empty(G.shape, dtype=torch.float64).pin_memory()
            Gh.copy_(G)
        except RuntimeError as e:
            e2e = {"value": None, "unit": "GFLOP/s", "skipped": f"pinned host buffers unavailable: {e}"[:200]}
    gp_shape = tuple(Gp.shape)
    del G, Gp
    torch.cuda.empty_cache()
    if Gh is not None:
        e2e = e2e_run(args, Gh, gp_shape, int(colshard), world, local, F, h, comm)
        del Gh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Gs, sample = oracle_sample(cfg, c3t)
        fl, dt = run_oracle_once(Gs)                      # warm (BLAS threads, page-in)
        fl, dt = run_oracle_once(Gs)
        cpu = {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": sample + f"; oracle = numpy/OpenBLAS geninv of PAPER.md P:105-140, {dt:.2f} s",
               "host": host_record()}
        try:
            cpu["extra_times"] = oracle_extra_times(dev)
        except Exception as exc:
            cpu["extra_times"] = {"skipped": str(exc)[:160]}

    if rank == 0:
        i8_peak, i8_src = int8_peak(ms > 1000.0)
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if not args.emulate else
            (f"f64 (Gram and a7 emulated on INT8 tensor cores: 7 int8 digits per element, {EMU_PAIRS} exact int32 "
             "digit products, FP64 accumulation)" if s >= 3072 else "f64 (a7 emulated on INT8 tensor cores; Gram on DMMA)"),
            "data": "synthetic",
            "config": {"workload": desc, "m": m, "n": n, "rank": rank_ok, "seed": seed_of(cfg),
                       "ms_per_matrix": ms, "parallelism": (f"columns sharded x{world}" if colshard else f"rows sharded x{world}") if world > 1 else "single GPU",
                       "pct_fp64_peak": value / (peak * 1e3),
                       "pct_fp64_peak_nominal_at_run_clock": (value / (148 * 128 * clocks["sm_mhz"] * 1e-3)
                                                             if clocks.get("sm_mhz") else None),
                       "pct_fp64_peak_note": "pct_fp64_peak: the measured DMMA peak (profiles/MEASURED_FP64.json); "
                                             "nominal: 148 SM x 128 flop/clk x the SM clock sampled during the run; "
                                             "no vendor FP64 figure is available offline",
                       "flops_per_step": F["total"],
                       "phase_ms_rank0": phases,
                       "flops_breakdown": {k: v for k, v in F.items() if k != "total"},
                       "l2": "inputs (G 64 GiB) far larger than the 126 MB L2; no flush needed"
                       if cfg.name == "C4" else ("L2 flushed before every timed step (512 MB write); step time = "
                                                 "sum of per-step CUDA event pairs") if flush else
                       "inputs (G + G+) larger than 512 MB, 4x the L2; no flush needed"},
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": launches,
            "replicated_check": replicated,
            "roofline": ({"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                          "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                          "kernel": "dgemm_tc<128,128,64,32,6,K-major,K-major> (a7 G+ = X G')",
                          "flops_per_launch": out_flops_launch, "ms_per_launch": out_ms,
                          "measured": roof_note, "peak_source": peak_src} if not args.emulate else
                         {"bound": "tensor", "achieved": achieved * EMU_PAIRS if achieved else None, "peak": i8_peak,
                          "unit": "TOPS (int8)", "frac": achieved * EMU_PAIRS / i8_peak if achieved else None,
                          "traffic": None,
                          "kernel": f"emu_split(_cols) + emu_gemm_kernel (a7 G+ = X G' / G' X as {EMU_PAIRS} int8 digit products, tcgen05.mma.kind::i8)",
                          "fp64_equivalent_tflops": achieved, "flops_per_launch": out_flops_launch,
                          "ms_per_launch": out_ms, "measured": roof_note + "; the a7 step = digit split of X and G + "
                          "the emulated products", "peak_source": i8_src}),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def e2e_run(args, Gh, gp_shape, trans, world, local, F, h, comm=None):
    """Same metric through the C ABI with HOST buffers (pinned): the H2D copy of this rank's G and the
    D2H copy of its block of G+ are inside the timed region, every step."""
    dev = torch.device("cuda", local)
    try:
        Gph = torch.empty(gp_shape, dtype=torch.float64).pin_memory()
    except RuntimeError as e:
        return {"value": None, "unit": "GFLOP/s", "skipped": f"pinned host buffers unavailable: {e}"[:200]}
    stream = torch.cuda.current_stream(dev)
    if world > 1:
        import torch.distributed as dist
        Gd = torch.empty(Gh.shape, dtype=torch.float64, device=dev)
        Gpd = torch.empty(gp_shape, dtype=torch.float64, device=dev)

        def step():
            Gd.copy_(Gh, non_blocking=True)
            h.geninv_sharded_d(comm, Gd, trans, Gpd)
            Gph.copy_(Gpd, non_blocking=True)
            torch.cuda.synchronize()
    else:
        def step():
            h.geninv_host_d(Gh, Gph)
    for _ in range(max(1, min(args.warmup, 2))):
        step()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / args.steps * 1e3
    barrier(world)
    ms = allmax(wall, world)
    nbytes_in = int(Gh.numel()) * 8 * world
    nbytes_out = int(np.prod(gp_shape)) * 8 * world
    return {"value": F["total"] / (ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": nbytes_in, "d2h_bytes_per_step": nbytes_out,
            "api": "geninv_host_d (pinned host G and G+)" if world == 1 else
            "pinned H2D of the local rows + geninv_sharded_d + D2H of the local block of G+"}


def bench_batched(args, cfg, desc, world, rank):
    from paper_0804_4809_b200.binding import Handle
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    from paper_0804_4809_b200.sharded import batch_range
    b0, b1 = batch_range(cfg.batch, world, rank)    # independent matrices: no exchange
    nb = b1 - b0
    G = I.make_batch(cfg, seed_of(cfg), b0, nb, device=dev)
    Gp = torch.empty(nb, cfg.n, cfg.m, dtype=torch.float64, device=dev)
    rk = torch.empty(nb, dtype=torch.int32, device=dev)
    h = Handle(local)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        h.geninv_batched_d(G, Gp, rk)
    barrier(world)
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            h.geninv_batched_d(G, Gp, rk)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = allmax(e0.elapsed_time(e1) / args.steps, world)
    s, ell = min(cfg.m, cfg.n), max(cfg.m, cfg.n)
    ranks = rk.cpu().numpy()
    F = allsum(sum(f_alg(s, ell, np.arange(int(r)))["total"] for r in ranks), world)
    peak, src = fp64_peak()
    value = F / (ms * 1e-3) / 1e9
    # e2e: every step copies this rank's G from pinned host memory, runs geninv_batched_d and reads G+ and
    # the ranks back into pinned host memory (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        Gh = torch.empty(G.shape, dtype=torch.float64).pin_memory()
        Gh.copy_(G)
        Gph = torch.empty(Gp.shape, dtype=torch.float64).pin_memory()
        rkh = torch.empty(rk.shape, dtype=torch.int32).pin_memory()
        torch.cuda.synchronize()
        barrier(world)
        # 8 chunks round-robin over 3 streams: the H2D copy of one chunk, the kernel of another and the
        # D2H copy of a third overlap (PCIe is full duplex)
        nch, streams = 8, [torch.cuda.Stream(dev) for _ in range(3)]
        bounds = [nb * c // nch for c in range(nch + 1)]
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for st_ in streams:
            st_.wait_event(a0)
        for _ in range(args.steps):
            for c in range(nch):
                lo, hi = bounds[c], bounds[c + 1]
                st_ = streams[c % 3]
                with torch.cuda.stream(st_):
                    G[lo:hi].copy_(Gh[lo:hi], non_blocking=True)
                    h.use_stream(st_)
                    h.geninv_batched_d(G[lo:hi], Gp[lo:hi], rk[lo:hi])
                    Gph[lo:hi].copy_(Gp[lo:hi], non_blocking=True)
                    rkh[lo:hi].copy_(rk[lo:hi], non_blocking=True)
        for st_ in streams:
            stream.wait_stream(st_)
        a1.record(stream)
        torch.cuda.synchronize()
        h.use_stream(stream)
        ems = allmax(a0.elapsed_time(a1) / args.steps, world)
        e2e = {"value": F / (ems * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ems,
               "h2d_bytes_per_step": int(allsum(Gh.numel() * 8, world)),
               "d2h_bytes_per_step": int(allsum(Gph.numel() * 8 + rkh.numel() * 4, world)),
               "api": "geninv_batched_d on 8 batch chunks over 3 streams, pinned host G / G+ / rank copies"}
        del Gh, Gph, rkh
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Gs, sample = oracle_sample(cfg, False)
        fl, dt = run_oracle_once(Gs)
        fl, dt = run_oracle_once(Gs)
        cpu = {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": sample + f"; oracle = numpy batched geninv (P:105-140 per matrix), {dt:.2f} s",
               "host": host_record()}
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                          "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic",
                          "config": {"workload": desc, "batch": cfg.batch, "us_per_matrix": ms * 1e3 / cfg.batch,
                                     "hbm_gbs": 2 * cfg.batch * cfg.m * cfg.n * 8 / (ms * 1e-3) / 1e9},
                          "clocks": clk.summary(),
                          "e2e": e2e,
                          "roofline": {"bound": "tensor", "achieved": value / 1e3, "peak": peak, "unit": "TFLOP/s",
                                       "frac": value / 1e3 / peak, "traffic": None, "peak_source": src,
                                       "kernel": "batched_geninv_kernel (one launch per step: the whole path)"},
                          "cpu_baseline": cpu,
                          "gpu_launches": args.steps}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
