"""Small end-to-end exercise of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run): FFT and direct paths,
1D and 2D, constant and variable coefficients, every preconditioner kind,
PCG (sine and standard bodies) and GMRES (right and left)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1912_13304_b200 import fde  # noqa: E402

dev = torch.device("cuda:0")
cases = [(1, 31, 2, W.PREC_TAU, "pcg"), (2, 63, 1, W.PREC_TAU_D, "gmres"), (3, 31, 2, W.PREC_TAU, "pcg"),
         (4, 63, 1, W.PREC_TAU, "gmres"), (4, 31, 1, W.PREC_TAU_DSYM, "gmres"), (3, 16, 1, W.PREC_TAU, "pcg"),
         (4, 17, 1, W.PREC_TAU_D, "gmres"), (1, 15, 1, W.PREC_NONE, "pcg")]
for cfg, n, batch, prec, solver in cases:
    p = W.config(cfg, n=n, batch=batch, prec=prec)
    h = fde.Fde.from_problem(p)
    b = torch.from_numpy(p.rhs.copy()).to(dev)
    y, z, x = torch.empty_like(b), torch.empty_like(b), torch.zeros_like(b)
    h.matvec(b, y)
    h.tau_apply(b, z)
    if solver == "pcg":
        h.pcg(b, x, 1e-8, 40)
    else:
        h.gmres(b, x, 1e-8, 10, 40)
        h.gmres(b, x, 1e-6, 10, 20, left=True)
    torch.cuda.synchronize()
    h.close()
    print("ok", cfg, n, batch, prec, solver, flush=True)
print("sanitize run done")
