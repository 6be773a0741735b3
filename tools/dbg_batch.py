import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_1912_13304_b200 import fde
for n in (511, 1023):
    p = W.config(5, n=n, batch=2)
    h = fde.Fde.from_problem(p)
    b = torch.from_numpy(p.rhs.copy()).cuda(); x = torch.zeros_like(b)
    st, stats = h.pcg(b, x, p.rtol, 200)
    print(n, "batch2", st, [(s["iters"], s["converged"], s["rel_res"]) for s in stats])
    h.close()
    for k in range(2):
        q = W.config(5, n=n, batch=1); q.rhs = p.rhs[k:k+1].copy()
        h = fde.Fde.from_problem(q)
        b = torch.from_numpy(q.rhs.copy()).cuda(); x1 = torch.zeros_like(b)
        st, stats = h.pcg(b, x1, q.rtol, 200)
        print(n, "single", k, st, [(s["iters"], s["converged"], s["rel_res"]) for s in stats],
              float((x1[0] - x[k]).norm() / x1[0].norm()))
        h.close()
