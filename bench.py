"""bench.py — throughput of the τ(F_α)-preconditioned Krylov hot path on B200.

Contract: `python bench.py --gpus N --steps K --warmup W`
prints ONE JSON line on rank 0.

Workload (BASELINE.json metric "preconditioned Krylov iters/sec
(matvec+τ-solve), % HBM roofline, 2D n=1023"): BASELINE config 5 at n = 1023
— the 2D constant-coefficient FDE A = νI + I⊗(T_α+T_αᵀ) + (T_β+T_βᵀ)⊗I,
α = β = 1.5, ν = h^α/Δt with h = Δt = 1/(n+1), preconditioned by
τ(F) = (S⊗S)diag(p_α(θ_i)+p_β(θ_j))(S⊗S), RHS U[0,1) from seed 0 (DESIGN.md
§3 input recipe). A "step" is one complete fde_pcg solve from x0 = 0 to
‖r‖ ≤ 1e-10‖b‖ through the C ABI (every §8(a) row: matvec, τ-solve, dots,
axpys and on-device convergence control); `value` is PCG iterations per
second summed over all ranks (each rank solves its own replica: "replicas
only"). L2 is flushed (a 512 MiB write) before every step,
outside the timed events.

`--impl reference` times the oracle (oracle/, dense fp64 CPU) on the same
workload instead: rank 0 only, a bounded number of PCG iterations per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "preconditioned Krylov iters/sec (matvec+τ-solve), % HBM roofline, 2D n=1023"
UNIT = "PCG iters/s"
FP64_DERIVED_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # SMs x FP64 FMA/clk x 2 x max clock = 37.2
FLUSH_BYTES = 512 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fde", choices=["fde", "reference"])
    ap.add_argument("--n", type=int, default=1023)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the n=2047 and cfg4 sub-records")
    return ap.parse_args()


def workload(args):
    p = W.config(5, n=args.n, batch=args.batch)
    desc = {"workload": "BASELINE cfg5 2D const-coef FDE, n=%d per dim (N=%d), alpha=beta=1.5, "
                        "PCG + tau(F) to rtol 1e-10, x0=0, full solve per step" % (p.n, p.N),
            "n": p.n, "N": p.N, "batch": p.batch, "rhs": "U[0,1) seed 0",
            "l2": "flushed (512 MiB write) before every step, outside the timed events"}
    return p, desc


# ----------------------------------------------------------------- algorithmic counts
def unit_alg(p) -> tuple:
    """Algorithmic (bytes, flops) of ONE unit W = matvec + τ-solve over the
    whole batch: bytes = the compulsory fp64 I/O
    (read x, write y, read r, write z: 32 B/element; + fields for variable
    coefficients: 2D +32, 1D +16; +8 for the 1/D field of TAU_D); flops = the
    standard FFT count per line (a real FFT of length L = 2.5·L·log2 L):
    constant-symmetric Toeplitz 10·m·log2(2m) + 2m + 2n, variable
    15·m·log2(2m) + 12m + 5n, DST-I 2.5·m·log2(2m); 2D = both directions'
    matvec lines + four DST passes."""
    n, m = p.n, p.n + 1
    lg = np.log2(2 * m)
    var = p.dp_field is not None
    b_el = 32 + ((32 if p.dims == 2 else 16) if var else 0) + (8 if p.prec == W.PREC_TAU_D else 0)
    t_line = (15 * m * lg + 12 * m + 5 * n) if var else (10 * m * lg + 2 * m + 2 * n)
    d_line = 2.5 * m * lg
    lines = n if p.dims == 2 else 1
    dirs = 2 if p.dims == 2 else 1
    flops = p.batch * lines * dirs * (t_line + 2 * d_line)
    return b_el * p.batch * p.N, flops


def roofline(p, us: float, peaks: dict, kernel: str, traffic) -> dict:
    """Binding roofline of one unit's work done in `us` µs:
    t_HBM = bytes/HBM peak, t_FP64 = flops/FP64 peak; the bound is the larger
    of the two, frac = max(t_HBM, t_FP64)/us; both fractions are reported."""
    by, fl = unit_alg(p)
    t_h = by / (peaks["hbm_gbs"] * 1e9) * 1e6
    t_f = fl / (peaks["fp64_tflops"] * 1e12) * 1e6
    gbs = by / (us * 1e-6) / 1e9
    tfl = fl / (us * 1e-6) / 1e12
    hbm = {"achieved_gbs": round(gbs, 1), "peak_gbs": peaks["hbm_gbs"], "frac": round(t_h / us, 4),
           "bytes_per_unit": int(by), "bytes_per_element": round(by / (p.batch * p.N), 2)}
    fp = {"achieved_tflops": round(tfl, 3), "peak_tflops": round(peaks["fp64_tflops"], 3), "frac": round(t_f / us, 4),
          "flops_per_unit": int(fl), "flops_per_element": round(fl / (p.batch * p.N), 1)}
    if t_f >= t_h:
        out = {"bound": "alu", "achieved": fp["achieved_tflops"], "peak": fp["peak_tflops"], "unit": "TFLOP/s",
               "frac": fp["frac"], "peak_source": peaks["fp64_src"]}
    else:
        out = {"bound": "hbm", "achieved": hbm["achieved_gbs"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
               "frac": hbm["frac"], "peak_source": peaks["hbm_src"]}
    out.update({"traffic": traffic, "kernel": kernel, "us": round(us, 3), "hbm": hbm, "fp64": fp})
    return out


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.splitlines():
            f = [v.strip() for v in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        busy = [v for v in sm if smax and v > 0.3 * smax] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- CPU oracle sample
def oracle_pcg_sample(p, iters: int):
    """The oracle (dense fp64 CPU, as it stands) running `iters` PCG iterations
    of the same system on RHS 0. Returns (seconds, iterations, threads)."""
    import oracle as O
    s = O.System(2, p.n, p.alpha, p.beta, p.nu, p.dp, p.dm, p.ep, p.em)
    Pinv = lambda v: s.prec_solve(v, O.PREC_TAU, p.cx, p.cy)
    s.S  # build the dense sine matrix outside the timing (setup, like fde_create)
    t0 = time.perf_counter()
    _, k, _, _ = O.pcg(s.matvec, Pinv, p.rhs[0], 1e-300, iters)
    dt = time.perf_counter() - t0
    return dt, k, blas_threads()


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:
        return 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    p, desc = workload(args)
    per_step = 8
    for _ in range(args.warmup):
        oracle_pcg_sample(p, 1)
    tot_t, tot_it, thr = 0.0, 0, 1
    for _ in range(args.steps):
        dt, k, thr = oracle_pcg_sample(p, per_step)
        tot_t += dt
        tot_it += k
    v = tot_it / tot_t
    sample = "%d PCG iterations per step (dense oracle: 4 n^3 matvec + 4 n^3 tau matmuls each), RHS 0" % per_step
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": desc,
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": thr, "kind": "oracle", "sample": sample,
                            "cpu": cpu_model()},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------- multi-rank
def reduce_over_ranks(ms: float, iters: int, device):
    """Replicas only: the job's time is the MAX of the ranks'
    device times, its work the SUM of their iterations. Collective on the
    default process group (NCCL on the GPU box; gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    k = torch.tensor([float(iters)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(k, op=dist.ReduceOp.SUM)
    return float(t.item()), int(k.item())


# ----------------------------------------------------------------- product arm
def time_solves(torch, h, p, b, x, stream, flush, steps: int, warmup: int, solver: str = "pcg"):
    """`warmup` untimed solves, then `steps` solves each bracketed by CUDA
    events on the handle's stream, L2 flushed before each (outside the
    events). Returns (total ms, total iterations over all RHS)."""
    def one():
        if solver == "pcg":
            return h.pcg(b, x, p.rtol, p.maxit)
        return h.gmres(b, x, p.rtol, p.restart, p.maxit)
    for _ in range(warmup):
        one()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    iters = 0
    for i in range(steps):
        flush.fill_(i & 0xff)
        ev[i][0].record(stream)
        st, stats = one()
        ev[i][1].record(stream)
        iters += sum(s_["iters"] for s_ in stats)
        assert all(s_["converged"] for s_ in stats), stats
    torch.cuda.synchronize()
    return sum(a.elapsed_time(c) for a, c in ev), iters


def live_iteration(h, p, b, torch, solver="pcg", peaks=None):
    """Device time of every kernel of one loop body (a PCG iteration / a
    GMRES(30) cycle) on a mid-solve state, bracketed by CUDA events on the
    solve's stream (fde_profile_solve: warm, the solvers' own launches)."""
    xs = torch.zeros_like(b)
    live, _ = h.profile_solve(b, xs, solver, p.rtol, 10 if solver == "pcg" else 30, restart=p.restart)
    tot = sum(t for _, t in live)
    agg = {}
    for name, us in live:
        agg[name] = agg.get(name, 0.0) + us
    return live, tot, agg


def sub_record(torch, fde, args, cfg: int, n: int, solver: str, dev, stream, flush, peaks, steps=3, warmup=2):
    """A second driver-timed workload on the same JSON line:
    the same solve contract (device-timed, L2 flushed) plus its loop body's
    kernels and the dominant kernel's binding roofline."""
    p = W.config(cfg, n=n)
    h = fde.Fde.from_problem(p, stream=stream.cuda_stream)
    b = torch.from_numpy(p.rhs.copy()).to(dev)
    x = torch.zeros_like(b)
    ms, iters = time_solves(torch, h, p, b, x, stream, flush, steps, warmup, solver)
    live, tot, agg = live_iteration(h, p, b, torch, solver)
    rec = {"workload": "BASELINE cfg%d, n=%d (N=%d), %s" % (cfg, n, p.N,
                                                          "PCG + tau(F) to 1e-10" if solver == "pcg"
                                                          else "GMRES(30) right-prec. mean-coef tau to 1e-10"),
           "value": iters / (ms / 1e3), "unit": "PCG iters/s" if solver == "pcg" else "GMRES iters/s",
           "ms_per_step": ms / steps, "iters_per_solve": iters / steps, "steps": steps, "warmup": warmup,
           "us_per_iter": round(ms * 1e3 / max(iters, 1), 3),
           "loop_body_kernels_us": {k: round(v, 2) for k, v in agg.items()}}
    if solver == "pcg":
        top = max(live, key=lambda kv: kv[1])
        rec["roofline"] = roofline(p, top[1], peaks, top[0], TRAFFIC.get("%s@%d" % (top[0], n)))
        rec["roofline_iteration"] = roofline(p, tot, peaks, "one PCG iteration", None)
    else:
        # one GMRES(30) cycle applies the unit (matvec + tau-solve) once per Arnoldi step
        steps_in_cycle = p.restart
        rec["roofline_step"] = roofline(p, tot / steps_in_cycle, peaks, "one Arnoldi step (cycle/30)", None)
    h.close()
    return rec


def run_fde(args, rank, world, local_rank):
    import torch
    from paper_1912_13304_b200 import fde

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream(dev)
    p, desc = workload(args)
    h = fde.Fde.from_problem(p, stream=stream.cuda_stream)
    b = torch.from_numpy(p.rhs.copy()).to(dev)
    x = torch.zeros_like(b)
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
    peaks = measured_peaks(fde)

    for _ in range(args.warmup):
        h.pcg(b, x, p.rtol, p.maxit)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()

    clk = ClockSampler(local_rank)
    clk.start()
    time.sleep(0.2)
    l0 = h.kernel_launches()
    ms, iters = time_solves(torch, h, p, b, x, stream, flush, args.steps, 0)
    launches = h.kernel_launches() - l0
    clocks = clk.stop()
    if world > 1:
        ms, iters = reduce_over_ranks(ms, iters, dev)
    value = iters / (ms / 1e3)

    # e2e: the same solve through the C ABI from pinned HOST buffers
    bh = torch.empty(b.shape, dtype=torch.float64, pin_memory=True)
    bh.copy_(b.cpu())
    xh = torch.zeros(b.shape, dtype=torch.float64, pin_memory=True)
    bn, xn = bh.numpy(), xh.numpy()
    h.pcg(bn, xn, p.rtol, p.maxit)
    e_ms, e_it = 0.0, 0
    for i in range(args.steps):
        flush.fill_(i & 0xff)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st, stats = h.pcg(bn, xn, p.rtol, p.maxit)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms += e0.elapsed_time(e1)
        e_it += sum(s_["iters"] for s_ in stats)
    if world > 1:
        e_ms, e_it = reduce_over_ranks(e_ms, e_it, dev)
    e2e = {"value": e_it / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(bn.nbytes),
           "d2h_bytes_per_step": int(xn.nbytes), "path": "fde_pcg with pinned host b, x (library-staged copies)"}

    # roofline: the dominant kernel of one PCG iteration timed live
    # (CUDA events on the solve's stream, warm), against the unit's ALGORITHMIC
    # bytes (32 B/element) and flops (standard FFT count); binding = max
    live, iter_us, agg = live_iteration(h, p, b, torch)
    top_name, top_us = max(live, key=lambda kv: kv[1])
    roof = roofline(p, top_us, peaks, top_name, TRAFFIC.get("%s@%d" % (top_name, p.n)))
    roof["share_of_iteration"] = round(top_us / iter_us, 4)
    # the whole iteration as the solve runs it: device-timed solve / iterations
    # (the in-graph kernels plus the solve's setup, amortised)
    roof["per_iteration"] = roofline(p, ms * 1e3 / max(iters, 1) * world, peaks,
                                     "one PCG iteration (timed solve / iterations)", None)
    iteration = {"us_kernels": round(iter_us, 3), "us_per_iter_timed": round(ms * 1e3 / max(iters, 1) * world, 3),
                 "kernels": [{"name": nm, "us": round(us, 3), "share": round(us / iter_us, 4)} for nm, us in live],
                 "mode": "one PCG iteration on a mid-solve state (after 10), kernels bracketed by CUDA events, warm"}
    # the unit W = fde_matvec + fde_tau_apply (the standard-basis operations of the ABI):
    # warm = back-to-back launches, cold = L2 flushed before every launch
    y = torch.empty_like(b)
    z = torch.empty_like(b)
    prof = h.profile_unit(b, y, z, reps=20, flush=None)
    prof_cold = h.profile_unit(b, y, z, reps=10, flush=flush)
    unit_us = sum(t for _, t in prof)
    unit = {"us": round(unit_us, 3), "kernels": {nm: round(us, 3) for nm, us in prof},
            "mode": "warm L2 (back-to-back launches)",
            "cold_us": {nm: round(us, 3) for nm, us in prof_cold}, "cold_total_us": round(sum(t for _, t in prof_cold), 3),
            "roofline": roofline(p, unit_us, peaks, "fde_matvec + fde_tau_apply (warm)", None)}
    h.close()

    extra = {}
    if not args.no_sub and rank == 0:
        extra["n2047"] = sub_record(torch, fde, args, 5, 2047, "pcg", dev, stream, flush, peaks)
        extra["cfg4"] = sub_record(torch, fde, args, 4, 1023, "gmres", dev, stream, flush, peaks, steps=2, warmup=1)

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": desc,
           "iters_per_solve": iters / (args.steps * world), "clocks": clocks, "e2e": e2e,
           "gpu_launches": int(launches), "roofline": roof, "iteration": iteration, "unit_w": unit,
           "peaks": {k: v for k, v in peaks.items()}}
    out.update(extra)
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(p)
    return out


def cpu_baseline(p) -> dict:
    """The oracle (dense fp64 CPU, as it stands) on a bounded sample of the
    same workload: PCG iterations of the same system on RHS 0, with all host
    cores (BLAS threads = os.cpu_count()) and with one thread."""
    ncpu = os.cpu_count() or 1
    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    dt, k, thr = oracle_pcg_sample(p, 40)
    rec = {"value": k / dt, "unit": UNIT, "cores": thr, "os_cpu_count": ncpu, "kind": "oracle",
           "sample": "%d PCG iterations of the same system (RHS 0) by the dense fp64 oracle, %d BLAS threads"
                     % (k, thr), "cpu": cpu_model(), "seconds": round(dt, 2)}
    if threadpool_limits is not None:
        with threadpool_limits(limits=1):
            dt1, k1, _ = oracle_pcg_sample(p, 3)
        rec["single_thread"] = {"value": k1 / dt1, "unit": UNIT, "cores": 1, "seconds": round(dt1, 2),
                                "sample": "%d PCG iterations, BLAS limited to 1 thread" % k1}
    return rec


def measured_peaks(fde=None):
    """Roofline denominators: HBM = MEASURED_PEAKS.json (driver-measured copy
    bandwidth); FP64 = measured on this GPU by fde_measure_fp64_peak (DFMA
    chains over every SM), else the derived 148 SMs x 64 FMA/clk x 2 x 1.965 GHz."""
    out = {}
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        out.update(hbm_gbs=float(d["hbm_gbs"]), hbm_src="MEASURED_PEAKS.json hbm_gbs (measured copy)")
    except Exception:
        out.update(hbm_gbs=6650.0, hbm_src="fallback 6.65 TB/s (B200_PROFILING.md)")
    out.update(fp64_tflops=FP64_DERIVED_TFLOPS, fp64_src="derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz")
    if fde is not None:
        try:
            v = fde.measure_fp64_peak(5)
            if v > 1.0:
                out.update(fp64_tflops=v, fp64_src="measured on this GPU: fde_measure_fp64_peak (DFMA chains, best of 5)")
        except Exception as e:  # pragma: no cover
            out["fp64_err"] = str(e)
    return out


def ncu_traffic():
    """Per-launch dram bytes of each kernel from the committed ncu --set full
    capture (profiles/traffic.json, written by tools/ncu_summary.py), if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(path))
    except Exception:
        return {}


TRAFFIC = ncu_traffic()


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = run_fde(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
