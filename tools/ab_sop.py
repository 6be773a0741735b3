"""A/B timing of the sine-domain PCG bodies at cfg 5 sizes: per-kernel device
times of one iteration (fde_profile_solve) and full-solve iters/s, for the
environment given on the command line (e.g. FDE_SOP=0)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1912_13304_b200 import fde  # noqa: E402


def run(n, batch, reps=5):
    p = W.config(5, n=n, batch=batch)
    h = fde.Fde.from_problem(p)
    b = torch.from_numpy(p.rhs.copy()).cuda()
    x = torch.zeros_like(b)
    for _ in range(2):
        st, stats = h.pcg(b, x, p.rtol, p.maxit)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    its = 0
    for _ in range(reps):
        st, stats = h.pcg(b, x, p.rtol, p.maxit)
        its += sum(s["iters"] for s in stats)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    live, _ = h.profile_solve(b, torch.zeros_like(b), "pcg", p.rtol, 10)
    h.close()
    return {"n": n, "batch": batch, "iters": stats[0]["iters"], "us_per_iter": round(ms * 1e3 / its * batch, 2),
            "kernels": {k: round(v, 2) for k, v in live}}


if __name__ == "__main__":
    tag = os.environ.get("FDE_SOP", "1")
    for n, batch in ((255, 1), (511, 1), (1023, 1), (1023, 2), (1023, 8), (2047, 1)):
        r = run(n, batch)
        r["FDE_SOP"] = tag
        print(json.dumps(r), flush=True)
