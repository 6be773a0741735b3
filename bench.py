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
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # SMs x FP64 FMA/clk x 2 x max clock = 37.2
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
    return ap.parse_args()


def workload(args):
    p = W.config(5, n=args.n, batch=args.batch)
    desc = {"workload": "BASELINE cfg5 2D const-coef FDE, n=%d per dim (N=%d), alpha=beta=1.5, "
                        "PCG + tau(F) to rtol 1e-10, x0=0, full solve per step" % (p.n, p.N),
            "n": p.n, "N": p.N, "batch": p.batch, "rhs": "U[0,1) seed 0",
            "l2": "flushed (512 MiB write) before every step, outside the timed events"}
    return p, desc


# ----------------------------------------------------------------- algorithmic counts
def unit_counts(name: str, p) -> tuple:
    """Algorithmic (bytes, flops) per launch of one kernel of the unit
    W = matvec + τ-solve (DESIGN.md §6 / SURVEY §8(d)): bytes = compulsory
    fp64 I/O of the kernel, flops = standard FFT count (a real FFT of length L
    costs 2.5·L·log2 L) plus the pointwise work."""
    n, m = p.n, p.n + 1
    L = 2 * m
    lg = np.log2(L)
    lines = p.batch * (n if p.dims == 2 else 1)
    el = p.batch * p.N
    if name.startswith("toeplitz"):
        var = name.endswith("_var")
        col = "_cols" in name
        b = (24 if col else 16) + (16 if var else 0)
        f_line = (15 * m * lg + 12 * m + 5 * n) if var else (10 * m * lg + 2 * m + 2 * n)
        return b * el, f_line * lines
    if name.startswith("dst"):
        return 16 * el, 2.5 * m * lg * lines + (n * lines)
    if name.startswith("tau"):
        return 16 * el, 2 * 2.5 * m * lg * lines + 3 * n * lines
    if name == "copy":
        return 16 * el, 0
    if name.startswith("sine_op"):
        # sine-domain operator line pass: DST, Toeplitz, DST on each
        # line; rows: read r, p, write p, w; cols: read p, w, write q; 1D: read r, p,
        # write p, q; concurrent body (rc): rows AND columns, each reading r, p_old and
        # writing its w; the row units also write p_new and apply the lagged x += αp
        b = {"sine_op_rows": 32, "sine_op_cols": 24, "sine_op_1d": 32, "sine_op_rc": 72}[name]
        f_line = 2 * 2.5 * m * lg + (10 * m * lg + 2 * m + 2 * n) + 3 * n
        return b * el, f_line * lines * (2 if name == "sine_op_rc" else 1)
    if name == "sine_xr":
        return 48 * el, 8 * el   # read x, p, r, q; write x, r
    if name == "sine_xr_rc":
        return 32 * el, 7 * el   # read r, w_r, w_c; write r (p and the lagged x are written by the row units)
    if name.startswith("pcg_"):
        return 48 * el, 6 * el
    raise KeyError(name)


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

    def step():
        return h.pcg(b, x, p.rtol, p.maxit)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()

    clk = ClockSampler(local_rank)
    clk.start()
    time.sleep(0.2)
    l0 = h.kernel_launches()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    iters = 0
    for i in range(args.steps):
        flush.fill_(i & 0xff)
        ev[i][0].record(stream)
        st, stats = step()
        ev[i][1].record(stream)
        iters += sum(s["iters"] for s in stats)
        assert all(s["converged"] for s in stats), stats
    torch.cuda.synchronize()
    launches = h.kernel_launches() - l0
    clocks = clk.stop()
    ms = sum(a.elapsed_time(c) for a, c in ev)
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
        e_it += sum(s["iters"] for s in stats)
    if world > 1:
        e_ms, e_it = reduce_over_ranks(e_ms, e_it, dev)
    e2e = {"value": e_it / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(bn.nbytes),
           "d2h_bytes_per_step": int(xn.nbytes), "path": "fde_pcg with pinned host b, x (library-staged copies)"}

    # roofline: per-kernel device time of one unit W (matvec + τ-solve), L2 flushed before every launch
    y = torch.empty_like(b)
    z = torch.empty_like(b)
    # live: device time of every kernel of the last PCG iteration of a solve, from
    # CUDA event nodes captured into the solve's loop-body graph (warm, exactly
    # the kernels and launch configuration of the timed region)
    xs = torch.zeros_like(b)
    live, _ = h.profile_solve(b, xs, "pcg", p.rtol, 10)
    iter_us = sum(t for _, t in live)
    kern = []
    for name, us in live:
        by, fl = unit_counts(name, p)
        t_h = by / (MEASURED["hbm_gbs"] * 1e9) * 1e6
        t_f = fl / (FP64_PEAK_TFLOPS * 1e12) * 1e6
        kern.append({"name": name, "us": round(us, 3), "share": round(us / iter_us, 4), "bytes": int(by),
                     "flops": int(fl), "hbm_frac": round(t_h / us, 4), "fp64_frac": round(t_f / us, 4)})
    iteration = {"us_kernels": round(iter_us, 3), "us_per_iter_timed": round(ms * 1e3 / max(iters, 1) * world, 3),
                 "kernels": kern, "mode": "one PCG iteration on a mid-solve state (after 10), kernels bracketed by CUDA events, warm"}
    # the unit W = fde_matvec + fde_tau_apply (the standard-domain operations of the ABI):
    # warm = back-to-back launches, cold = L2 flushed before every launch
    prof = h.profile_unit(b, y, z, reps=20, flush=None)
    prof_cold = h.profile_unit(b, y, z, reps=10, flush=flush)
    unit_us = sum(t for _, t in prof)
    ukern = []
    for name, us in prof:
        by, fl = unit_counts(name, p)
        t_h = by / (MEASURED["hbm_gbs"] * 1e9) * 1e6
        t_f = fl / (FP64_PEAK_TFLOPS * 1e12) * 1e6
        ukern.append({"name": name, "us": round(us, 3), "share": round(us / unit_us, 4), "bytes": int(by),
                      "flops": int(fl), "hbm_frac": round(t_h / us, 4), "fp64_frac": round(t_f / us, 4)})
    top = max(kern, key=lambda k: k["us"])
    hbm_gbs = top["bytes"] / (top["us"] * 1e-6) / 1e9
    tfl = top["flops"] / (top["us"] * 1e-6) / 1e12
    if top["fp64_frac"] >= top["hbm_frac"]:
        roof = {"bound": "alu", "achieved": round(tfl, 3), "peak": round(FP64_PEAK_TFLOPS, 2), "unit": "TFLOP/s",
                "frac": round(tfl / FP64_PEAK_TFLOPS, 4),
                "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (DESIGN.md §6)"}
    else:
        roof = {"bound": "hbm", "achieved": round(hbm_gbs, 1), "peak": MEASURED["hbm_gbs"], "unit": "GB/s",
                "frac": round(hbm_gbs / MEASURED["hbm_gbs"], 4), "peak_source": MEASURED["src"]}
    roof.update({"kernel": top["name"], "traffic": TRAFFIC.get(top["name"]),
                 "hbm": {"achieved_gbs": round(hbm_gbs, 1), "frac": round(hbm_gbs / MEASURED["hbm_gbs"], 4)},
                 "fp64": {"achieved_tflops": round(tfl, 3), "frac": round(tfl / FP64_PEAK_TFLOPS, 4)}})
    unit_bytes = sum(k["bytes"] for k in ukern)
    unit_flops = sum(k["flops"] for k in ukern)
    unit_roof = max(unit_bytes / (MEASURED["hbm_gbs"] * 1e9), unit_flops / (FP64_PEAK_TFLOPS * 1e12)) * 1e6
    unit = {"us": round(unit_us, 3), "kernels": ukern, "mode": "warm L2 (back-to-back launches)",
            "cold_us": {nm: round(us, 3) for nm, us in prof_cold}, "cold_total_us": round(sum(t for _, t in prof_cold), 3),
            "hbm_frac": round(unit_bytes / (MEASURED["hbm_gbs"] * 1e9) * 1e6 / unit_us, 4),
            "binding_roofline_frac": round(unit_roof / unit_us, 4)}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": desc,
           "iters_per_solve": iters / (args.steps * world), "clocks": clocks, "e2e": e2e,
           "gpu_launches": int(launches), "roofline": roof, "iteration": iteration, "unit_w": unit}
    if rank == 0 and not args.no_cpu_baseline:
        it = 40
        dt, k, thr = oracle_pcg_sample(p, it)
        out["cpu_baseline"] = {"value": k / dt, "unit": UNIT, "cores": thr, "kind": "oracle",
                               "sample": "%d PCG iterations of the same system (RHS 0) by the dense fp64 oracle" % k,
                               "cpu": cpu_model(), "seconds": round(dt, 2)}
    h.close()
    return out


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "MEASURED_PEAKS.json hbm_gbs (measured copy)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "src": "fallback 6.65 TB/s (B200_PROFILING.md)"}


def ncu_traffic():
    """Per-launch dram bytes of each kernel from the committed ncu --set full
    capture (profiles/traffic.json, written by tools/ncu_summary.py), if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(path))
    except Exception:
        return {}


MEASURED = measured_peaks()
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
