"""Throughput of every BASELINE config on one B200 (evidence beside bench.py's
headline line): full solves through the C ABI, device time by CUDA events on
the handle's stream (L2 flushed before each solve), Krylov iterations per
second (RHS-iterations for batch > 1), plus the live per-kernel profile of one
loop body (fde_profile_solve). Writes one JSON object per line to stdout.

usage: python tools/sweep.py [--quick]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1912_13304_b200 import fde  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true")
ap.add_argument("--only", default="")
args = ap.parse_args()

CASES = [  # (cfg, n, batch)
    (1, None, 1), (2, None, 1), (3, None, 1), (4, None, 1),
    (5, 255, 1), (5, 511, 1), (5, 1023, 1), (5, 2047, 1), (5, 4095, 1),
    (5, 255, 8), (5, 511, 8), (5, 1023, 8), (5, 2047, 8), (5, 4095, 2),
]
if args.quick:
    CASES = [(1, None, 1), (3, None, 1), (4, None, 1), (5, 1023, 1), (5, 1023, 8)]
if args.only:
    CASES = [c for c in CASES if str(c[0]) in args.only.split(",")]

dev = torch.device("cuda:0")
stream = torch.cuda.current_stream(dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def solve(h, p, b, x):
    if p.solver == "pcg":
        return h.pcg(b, x, p.rtol, p.maxit)
    return h.gmres(b, x, p.rtol, p.restart, p.maxit)


for cfg, n, batch in CASES:
    p = W.config(cfg, n=n, batch=batch)
    t0 = time.time()
    h = fde.Fde.from_problem(p, stream=stream.cuda_stream)
    b = torch.from_numpy(p.rhs.copy()).to(dev)
    x = torch.zeros_like(b)
    for _ in range(2):
        solve(h, p, b, x)
    reps = 3
    ms, its = 0.0, 0
    for i in range(reps):
        flush.fill_(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st, stats = solve(h, p, b, x)
        e1.record(stream)
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
        its += sum(s["iters"] for s in stats)
    xs = torch.zeros_like(b)
    live, _ = h.profile_solve(b, xs, p.solver, p.rtol, 10 if p.solver == "pcg" else p.restart, p.restart)
    agg = {}
    for name, us in live:
        agg[name] = agg.get(name, 0.0) + us
    out = {"cfg": cfg, "n": p.n, "N": p.N, "batch": batch, "solver": p.solver, "prec": p.prec,
           "iters_per_solve": its / reps / batch, "ms_per_solve": ms / reps,
           "iters_per_s": its / (ms / 1e3), "us_per_iter": ms * 1e3 / (its / batch),
           "loop_body_kernels_us": {k: round(v, 2) for k, v in agg.items()},
           "loop_body": "one PCG iteration" if p.solver == "pcg" else "one GMRES(%d) cycle" % p.restart,
           "converged": all(s["converged"] for s in stats), "wall_s": round(time.time() - t0, 1)}
    print(json.dumps(out), flush=True)
    h.close()
    del b, x, xs
    torch.cuda.empty_cache()
