"""Run `reps` units W = fde_matvec + fde_tau_apply of a BASELINE config on
cuda:0 (the short command the ncu captures profile)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1912_13304_b200 import fde  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=5)
ap.add_argument("--n", type=int, default=1023)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--pcg", action="store_true", help="also run one fde_pcg solve")
ap.add_argument("--gmres", type=int, default=0, help="also run one fde_gmres solve with this maxit")
a = ap.parse_args()
p = W.config(a.cfg, n=a.n, batch=a.batch)
h = fde.Fde.from_problem(p, stream=torch.cuda.current_stream().cuda_stream)
x = torch.from_numpy(p.rhs.copy()).cuda()
y = torch.empty_like(x)
z = torch.empty_like(x)
for _ in range(a.reps):
    h.matvec(x, y)
    h.tau_apply(x, z)
if a.pcg:
    xs = torch.zeros_like(x)
    print(h.pcg(x, xs, p.rtol, p.maxit))
if a.gmres:
    xs = torch.zeros_like(x)
    print(h.gmres(x, xs, p.rtol, p.restart, a.gmres))
torch.cuda.synchronize()
print("ok", float(y.norm()), float(z.norm()))
