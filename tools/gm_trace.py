"""Timeline of one DCGS2 Arnoldi step's orthogonalisation kernels (trace
build -DFDE_SOP_TRACE=1 via FDE_LIB): pass A blocks (start, end of the
element loop), the last block's partial sums and Givens step, pass B blocks
(start, end), for step j = 20 of the last cycle of a cfg-4 GMRES solve."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1912_13304_b200 import fde  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1023
p = W.config(4, n=n)
h = fde.Fde.from_problem(p)
b = torch.from_numpy(p.rhs.copy()).cuda()
x = torch.zeros_like(b)
h.gmres(b, x, p.rtol, p.restart, 60)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
assert fde.lib.fde_debug_xr_trace(buf, 4096) == 0
a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
t = a[:4000].reshape(1000, 4)
A = t[t[:, 0] > 0]
B = t[t[:, 2] > 0]
t0 = A[:, 0].min()
r = lambda v: [round(float((v.min() - t0) / 1e3), 2), round(float((v.mean() - t0) / 1e3), 2),
               round(float((v.max() - t0) / 1e3), 2)]
out = {"n": n, "A_blocks": int(len(A)), "A_start": r(A[:, 0]), "A_loop_end": r(A[:, 1]),
       "A_last_in": round(float((a[4000] - t0) / 1e3), 2), "A_finalized": round(float((a[4001] - t0) / 1e3), 2),
       "A_step_done": round(float((a[4002] - t0) / 1e3), 2),
       "B_blocks": int(len(B)), "B_start": r(B[:, 2]), "B_end": r(B[:, 3])}
print(json.dumps(out))
h.close()
